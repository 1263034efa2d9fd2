"""Profiling driver for the config #4 iteration kernels: one GMRES(30) cycle and ten
BiCGSTAB iterations (Jacobi, fp64 3-D convection-diffusion p^3), then five iterations of
the fused-direction CG graph loop at q^3 (config #5 shape on one GPU).  Run with
SPARSEB200_GRAPH=0 (host-polled loops: ncu cannot profile kernel nodes of graphs with
conditional nodes; the kernels and their order are the graph loop's).

    SPARSEB200_GRAPH=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --csv --log-file gpurun_out/krylov.csv python tools/prof_krylov.py 256 512
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 256
q = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dev = sp.create_device("cuda", 0)
a = gen.convdiff3d(dev, p)
m = sp.jacobi_create(a)
for name, cls, kw, its in (("gmres30", sp.Gmres, {"krylov_dim": 30}, 30), ("bicgstab", sp.Bicgstab, {}, 10)):
    b = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 1.0)
    x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
    log = cls(a, criteria=[sp.Iteration(its)], preconditioner=m, **kw).solve(b, x)
    torch.cuda.synchronize()
    print(name, "iterations", log.iterations, flush=True)
del a, m
torch.cuda.empty_cache()
if q:
    a = gen.poisson3d(dev, q)
    m = sp.jacobi_create(a)
    b = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 1.0)
    x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
    log = sp.Cg(a, criteria=[sp.Iteration(5)], preconditioner=m).solve(b, x)
    torch.cuda.synchronize()
    print("cg", q, "iterations", log.iterations, flush=True)
