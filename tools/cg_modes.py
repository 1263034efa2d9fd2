"""Per-iteration time of the CG loop shapes (sb_set_cg_fused 0 / 1 / 3) over grid sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08230_b200 import _lib, gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402

sizes = [int(v) for v in (sys.argv[1:] or ["96", "128", "160", "192", "224", "256"])]
dev = sp.create_device("cuda", 0)
for p in sizes:
    a = gen.poisson3d(dev, p)
    s = sp.Cg(a, criteria=[sp.Iteration(100000), sp.ResidualNorm(1e-8)], preconditioner=sp.jacobi_create(a))
    b = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 1.0)
    x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
    row = []
    for mode in (0, 1, 3):
        _lib.fn("sb_set_cg_fused")(mode)
        for _ in range(2):
            x.values.zero_()
            s.solve(b, x)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its = 0
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            x.values.zero_()
            its += s.solve(b, x).iterations
        e1.record()
        torch.cuda.synchronize()
        row.append(f"mode{mode} {e0.elapsed_time(e1) / its * 1e3:7.2f}us")
    print(f"p={p:4d} n={a.rows:9d} iters={its // 3:5d}  " + "  ".join(row), flush=True)
    del a, s, b, x
    torch.cuda.empty_cache()
