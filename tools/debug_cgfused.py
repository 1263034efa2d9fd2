"""Debug: CG loop modes (sb_set_cg_fused 0/1/2) on the fused-direction test's cases."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2510_08230_b200 import _lib, gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402
from tests.gpu_util import host, vec  # noqa: E402

dev = sp.create_device("cuda", 0)
a = gen.stencil_csr(dev, 18, dim=3)
rng = np.random.default_rng(5)
b = rng.random(a.rows)
x0 = rng.random(a.rows)
mats = [a, a.with_kernel("strict"), a.with_kernel("vector"), sp.ell_from_csr(a), sp.sellp_from_csr(a),
        sp.coo_from_csr(a)]
cases = [([sp.Iteration(2000), sp.ResidualNorm(1e-7)], True, None), ([sp.Iteration(7)], True, x0),
         ([sp.Iteration(8)], False, None), ([sp.Iteration(2000), sp.ResidualNorm(1e-6)], False, x0)]
from oracle import sbref  # noqa: E402
rp, ci_, v = (t.cpu().numpy() for t in (a.row_ptrs, a.col_idxs, a.values))
inv = sbref.jacobi_create(rp, ci_, v)[0]
lg, xo = sbref.solve("cg", rp, ci_, v, b, x0=x0, inv_diag=inv, max_iters=7, threads=1)
print("oracle case 1", lg.iterations, lg.residual_history[:3], float(np.abs(xo).sum()))
for ci, (crit, pre, xi) in enumerate(cases):
    for k, mat in enumerate(mats):
        res = []
        for graph in (1, 0):
            for mode in (0, 1, 2):
                _lib.fn("sb_set_cg_fused")(mode)
                _lib.fn("sb_set_graph_mode")(graph)
                x = vec(dev, np.zeros(a.rows) if xi is None else xi)
                try:
                  lg = sp.Cg(mat, criteria=crit, preconditioner=sp.jacobi_create(a) if pre else None).solve(vec(dev, b), x)
                  res.append((graph, mode, lg.iterations, lg.residual_history[:3], float(np.abs(host(x)).sum())))
                except sp.errors.BreakdownError as e:
                  res.append((graph, mode, "breakdown", e.iteration))
        same = all(r[2:] == res[0][2:] for r in res)
        print("case", ci, "mat", k, "OK" if same else "MISMATCH")
        if not same or ci == 1:
            for r in res:
                print("   ", r)
