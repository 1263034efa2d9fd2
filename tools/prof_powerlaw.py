"""Profiling driver: power-law 4M (config #3) SpMV in a given format, 3 launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402

fmt = sys.argv[1] if len(sys.argv) > 1 else "csr"
dev = sp.create_device("cuda", 0)
a = gen.powerlaw_csr(dev)
m = {"csr": a, "vector": a.with_kernel("vector"), "coo": None, "hybrid": None}.get(fmt)
if fmt == "coo":
    m = sp.coo_from_csr(a)
elif fmt == "hybrid":
    m = sp.hybrid_from_csr(a)
elif fmt == "sellp":
    m = sp.sellp_from_csr(a)
b = sp.dense_from_array(dev, torch.tensor(np.random.default_rng(0).random(a.rows)))
x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
for _ in range(3):
    m.apply(b, x)
torch.cuda.synchronize()
