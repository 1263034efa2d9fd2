"""Stream-SpMV block-rows sweep for fp32 / fp64 on 3-D Poisson 128^3 and 2-D Poisson 1000^2
(L2 flushed before each launch for the 80 MB 2-D matrix)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402
from tools.sweep_configs import timed_spmv  # noqa: E402

dev = sp.create_device("cuda", 0)
flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 1 GB
for name, mk, fl in (("poisson3d_128", lambda pr: gen.poisson3d(dev, 128, precision=pr), None),
                     ("poisson2d_1000", lambda pr: gen.poisson2d(dev, 1000, precision=pr), flush)):
    for prec in (sp.Precision.single, sp.Precision.double):
        base = mk(prec)
        st = base.row_stats()
        vb = prec.itemsize
        byt = (vb + 4) * base.nnz + 4 * (base.rows + 1) + 2 * vb * base.rows
        row = []
        for R, q in ((256, 3), (128, 2), (64, 1)):
            a = base.with_kernel("stream")
            plan = a.plan()
            plan.block_rows = R
            plan.nnz_cap = st.max_block_nnz[q]
            b = sp.dense_create(dev, a.rows, 1, prec, 1.0)
            x = sp.dense_create(dev, a.rows, 1, prec, 0.0)
            us = timed_spmv(a, b, x, flush=fl)
            row.append(f"R={R}: {us:7.2f}us ({byt / us / 1e3 / 6543.1:.3f})")
        print(name, prec.value, " ".join(row), flush=True)
