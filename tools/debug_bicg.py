import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2510_08230_b200 import gen
from paper_2510_08230_b200 import sparseops as sp
p = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dev = sp.create_device("cuda", 0)
a = gen.convdiff3d(dev, p)
m = sp.jacobi_create(a)
for fmt in ("csr", "strict"):
    mat = a if fmt == "csr" else a.with_kernel("strict")
    b = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 1.0)
    x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
    try:
        log = sp.Bicgstab(mat, criteria=[sp.Iteration(5000), sp.ResidualNorm(1e-8)], preconditioner=m).solve(b, x)
        print(fmt, "ok", log.iterations, log.residual_history[-3:])
    except sp.errors.BreakdownError as e:
        h = e.log.residual_history
        print(fmt, "breakdown", e.iteration, len(h), h[:3], h[-6:], "x finite:", bool(np.isfinite(x.numpy()).all()))
