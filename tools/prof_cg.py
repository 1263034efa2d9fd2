"""Profiling driver: 5 standalone SpMVs then one Jacobi-CG solve, fp64 Poisson 128^3.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/prof_cg.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 128
fmt = sys.argv[2] if len(sys.argv) > 2 else "csr"
dev = sp.create_device("cuda", 0)
a = gen.poisson3d(dev, p)
if fmt == "sellp":
    a = sp.sellp_from_csr(a)
elif fmt == "ell":
    a = sp.ell_from_csr(a)
b = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 1.0)
x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
for _ in range(5):
    a.apply(b, x)
torch.cuda.synchronize()
csr = gen.poisson3d(dev, p)
m = sp.jacobi_create(csr)
log = sp.Cg(a, criteria=[sp.Iteration(100000), sp.ResidualNorm(1e-8)], preconditioner=m).solve(b, x)
torch.cuda.synchronize()
print("iterations", log.iterations)
