"""CG 128^3 per-iteration time (CUDA events), for A/B of solver variants via env vars."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dev = sp.create_device("cuda", 0)
a = gen.poisson3d(dev, p)
R = int(os.environ.get("SB_R", "0"))
if R:
    st = a.row_stats()
    plan = a.plan()
    plan.block_rows = R
    plan.nnz_cap = st.max_block_nnz[{64: 1, 128: 2, 256: 3}[R]]
    plan.nnz_cap256 = 0 if R != 128 else plan.nnz_cap256
s = sp.Cg(a, criteria=[sp.Iteration(100000), sp.ResidualNorm(1e-8)], preconditioner=sp.jacobi_create(a))
b = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 1.0)
x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
for _ in range(3):
    x.values.zero_()
    log = s.solve(b, x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
its = 0
for _ in range(5):
    x.values.zero_()
    its += s.solve(b, x).iterations
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"fused={os.environ.get('SPARSEB200_CG_FUSED', '1')} R={R} p={p} iters={log.iterations} "
      f"solve={ms / 5:.3f} ms  per-iter={ms / its * 1e3:.2f} us")
try:
    import ctypes
    print("  L2 persist attr:", torch.cuda.get_device_properties(0).L2_cache_size // (1 << 20), "MB L2")
except Exception:
    pass
