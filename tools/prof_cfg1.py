"""One flushed config-#1 stream SpMV (2-D Poisson 1000^2 fp64) and one fp32 128^3 SpMV, for
ncu --set full (kernel filter csr_stream_kernel; launch 4 = config #1, 8 = fp32 128^3)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402

dev = sp.create_device("cuda", 0)
flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float64, device="cuda")
for mk, prec in ((lambda pr: gen.poisson2d(dev, 1000, precision=pr), sp.Precision.double),
                 (lambda pr: gen.poisson3d(dev, 128, precision=pr), sp.Precision.single)):
    a = mk(prec).with_kernel("stream")
    b = sp.dense_create(dev, a.cols, 1, prec, 1.0)
    x = sp.dense_create(dev, a.rows, 1, prec, 0.0)
    for _ in range(4):
        flush.sum()
        a.apply(b, x)
    torch.cuda.synchronize()
print("ok")
