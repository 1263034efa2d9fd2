"""Debug: graph vs polled CG loop with a nonzero initial guess (fresh process order)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2510_08230_b200 import _lib, gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402
from tests.gpu_util import host, vec  # noqa: E402

order = sys.argv[1] if len(sys.argv) > 1 else "gp"
dev = sp.create_device("cuda", 0)
a = gen.stencil_csr(dev, 18, dim=3)
rng = np.random.default_rng(5)
b = rng.random(a.rows)
x0 = rng.random(a.rows)
for its in (1, 2, 7):
    for g in order:
        _lib.fn("sb_set_graph_mode")(1 if g == "g" else 0)
        x = vec(dev, x0)
        lg = sp.Cg(a, criteria=[sp.Iteration(its)], preconditioner=sp.jacobi_create(a)).solve(vec(dev, b), x)
        xh = host(x)
        print(order, g, its, lg.iterations, lg.residual_history[:3], float(np.abs(xh).sum()), xh[:3])
