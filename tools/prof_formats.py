"""Profiling driver: ELL / SELL-P(64) / SELL-P(32) / CSR / COO SpMV on the 3-D Poisson 128^3
matrix, fp64 and fp32, three applies each (ncu -k regex selects the kernels).

    ncu --set full -k regex:"ell_kernel|sellp" -s 2 -c 12 -o gpurun_out/formats python tools/prof_formats.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dev = sp.create_device("cuda", 0)
for prec in (sp.Precision.double, sp.Precision.single):
    a = gen.poisson3d(dev, p, precision=prec)
    b = sp.dense_create(dev, a.rows, 1, prec, 1.0)
    x = sp.dense_create(dev, a.rows, 1, prec, 0.0)
    for name, m in (("ell", sp.ell_from_csr(a)), ("sellp64", sp.sellp_from_csr(a, 64)),
                    ("sellp32", sp.sellp_from_csr(a, 32)), ("csr", a), ("coo", sp.coo_from_csr(a))):
        for _ in range(3):
            m.apply(b, x)
        torch.cuda.synchronize()
        print(prec.name, name, "done", flush=True)
