"""Stream-SpMV tuning sweep: block rows R x matrix size; CUDA-event timing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402

dev = sp.create_device("cuda", 0)
for p in (128, 256):
    base = gen.poisson3d(dev, p)
    st = base.row_stats()
    for R, q, ns in ((256, 3, 2), (128, 2, 2), (64, 1, 2)):
        a = base.with_kernel("stream")
        plan = a.plan()
        plan.block_rows = R
        plan.nnz_cap = st.max_block_nnz[q]
        b = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 1.0)
        x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
        for _ in range(5):
            a.apply(b, x)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(50):
            a.apply(b, x)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 50 * 1e3
        byt = 12 * a.nnz + 4 * (a.rows + 1) + 16 * a.rows
        print(f"p={p} R={R} stages={ns}: {us:8.2f} us  {byt / us / 1e3:8.1f} GB/s  frac {byt / us / 1e3 / 6543.1:.3f}")
