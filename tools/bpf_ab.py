"""Standalone stream-SpMV times (us) for the b L2-hint A/B (SPARSEB200_STREAM_BPF_MB):
config #1 (2-D Poisson 1000^2 fp64, L2 flushed before every launch) and 3-D Poisson 128^3
fp64 / fp32 (back to back, larger than L2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402
from tools.sweep_configs import timed_spmv  # noqa: E402

dev = sp.create_device("cuda", 0)
flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 1 GB
out = []
for name, mk, fl, prec in (("cfg1_2d1000_f64", lambda pr: gen.poisson2d(dev, 1000, precision=pr), flush, sp.Precision.double),
                           ("cfg1_2d1000_f32", lambda pr: gen.poisson2d(dev, 1000, precision=pr), flush, sp.Precision.single),
                           ("3d128_f64", lambda pr: gen.poisson3d(dev, 128, precision=pr), None, sp.Precision.double),
                           ("3d128_f32", lambda pr: gen.poisson3d(dev, 128, precision=pr), None, sp.Precision.single)):
    a = mk(prec).with_kernel("stream")
    b = sp.dense_create(dev, a.cols, 1, prec, 1.0)
    x = sp.dense_create(dev, a.rows, 1, prec, 0.0)
    us = min(timed_spmv(a, b, x, reps=30, flush=fl) for _ in range(3))
    out.append(f"{name} {us:.2f}")
print(f"bpf_mb={os.environ.get('SPARSEB200_STREAM_BPF_MB', '0')}: " + "  ".join(out))
