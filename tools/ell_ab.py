"""128^3 ELL / SELL-P / Hybrid SpMV times (us, back to back), fp32 and fp64, for env A/B."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402
from tools.sweep_configs import timed_spmv  # noqa: E402

dev = sp.create_device("cuda", 0)
out = []
for prec in (sp.Precision.single, sp.Precision.double):
    a = gen.poisson3d(dev, 128, precision=prec)
    b = sp.dense_create(dev, a.rows, 1, prec, 1.0)
    x = sp.dense_create(dev, a.rows, 1, prec, 0.0)
    for name, m in (("ell", sp.ell_from_csr(a)), ("hybrid", sp.hybrid_from_csr(a))):
        us = min(timed_spmv(m, b, x) for _ in range(3))
        out.append(f"{name}_{prec.name} {us:.2f}")
print(" ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SPARSEB200_")), "|", "  ".join(out))
