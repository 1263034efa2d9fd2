"""A/B of the CSR SpMV kernels on the config-#3 power-law matrix (fp64 / fp32), us per SpMV."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402
from tools.sweep_configs import timed_spmv  # noqa: E402

dev = sp.create_device("cuda", 0)
for prec in (sp.Precision.double, sp.Precision.single):
    a = gen.powerlaw_csr(dev, precision=prec)
    b = sp.dense_from_array(dev, torch.tensor(np.random.default_rng(0).random(a.rows).astype(prec.dtype)))
    x = sp.dense_create(dev, a.rows, 1, prec, 0.0)
    res = {k: timed_spmv(a.with_kernel(k), b, x) for k in ("tile", "merge")}
    print(prec.value, os.environ.get("SPARSEB200_TILE_C", "2048"),
          " ".join(f"{k}={v:.1f}us" for k, v in res.items()), flush=True)
    del a
    torch.cuda.empty_cache()
