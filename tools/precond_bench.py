"""ILU(0) / IC(0) / SpTRSV timings and preconditioned-solver comparisons (device)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3  # ms (host wall, includes syncs)


dev = sp.create_device("cuda", 0)
out = {}
p = int(sys.argv[1]) if len(sys.argv) > 1 else 128
a = gen.poisson3d(dev, p)
n = a.rows
out["ilu0_ms"] = timed(lambda: sp.ilu0_factorize(a), 3)
out["ic0_ms"] = timed(lambda: sp.ic0_factorize(a), 3)
f = sp.ilu0_factorize(a)
g = sp.ic0_factorize(a)
b = sp.dense_create(dev, n, 1, sp.Precision.double, 1.0)
y = sp.dense_create(dev, n, 1, sp.Precision.double, 0.0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, mat in (("trsv_lower_unit", lambda: sp.solve_lower_tri(f.l, b, y, unit_diag=True), f.l),
                      ("trsv_upper", lambda: sp.solve_upper_tri(f.u, b, y), f.u)):
    ms = timed(fn, 10)  # includes the structure check + host sync per call
    byt = 12 * mat.nnz + 4 * (n + 1) + 16 * n
    out[name] = {"ms_incl_check": ms, "bytes": byt, "gbs_incl_check": byt / ms / 1e6}
for label, m in (("jacobi", sp.jacobi_create(a)), ("ic0", g), ("ilu0", f)):
    x = sp.dense_create(dev, n, 1, sp.Precision.double, 0.0)
    s = sp.Cg(a, criteria=[sp.Iteration(100000), sp.ResidualNorm(1e-8)], preconditioner=m)
    s.solve(b, x)
    x.values.zero_()
    torch.cuda.synchronize()
    e0.record()
    log = s.solve(b, x)
    e1.record()
    torch.cuda.synchronize()
    out[f"cg_{label}"] = {"iterations": log.iterations, "ms": e0.elapsed_time(e1)}
c = gen.convdiff3d(dev, 64)
bc = sp.dense_create(dev, c.rows, 1, sp.Precision.double, 1.0)
for label, m in (("jacobi", sp.jacobi_create(c)), ("ilu0", sp.ilu0_factorize(c))):
    x = sp.dense_create(dev, c.rows, 1, sp.Precision.double, 0.0)
    s = sp.Gmres(c, criteria=[sp.Iteration(5000), sp.ResidualNorm(1e-8)], krylov_dim=30, preconditioner=m)
    s.solve(bc, x)
    x.values.zero_()
    torch.cuda.synchronize()
    e0.record()
    log = s.solve(bc, x)
    e1.record()
    torch.cuda.synchronize()
    out[f"gmres30_convdiff64_{label}"] = {"iterations": log.iterations, "ms": e0.elapsed_time(e1)}
print(json.dumps(out))
