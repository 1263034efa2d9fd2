"""Arrival-time analysis of the persistent CG grid barriers (fp64 Poisson p^3).

    SPARSEB200_CG_PROFILE=1 SPARSEB200_CG_PROFILE_DUMP=/tmp/st.bin python tools/cg_arrivals.py [p]

Reads the raw stamps the library dumps (barriers 10..27: per-CTA arrival times, CTA 0's
release times, the SM of every CTA) and prints, per barrier, the arrival spread
percentiles and whether the late CTAs are the same ones every time (per-SM / per-CTA
correlation), to tell hardware-rate variation from work imbalance.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dump = os.environ.get("SPARSEB200_CG_PROFILE_DUMP", "/tmp/st.bin")
dev = sp.create_device("cuda", 0)
a = gen.poisson3d(dev, p)
m = sp.jacobi_create(a)
b = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 1.0)
for rep in range(2):
    x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
    log = sp.Cg(a, criteria=[sp.Iteration(100000), sp.ResidualNorm(1e-8)], preconditioner=m).solve(b, x)
torch.cuda.synchronize()
st = np.fromfile(dump, dtype=np.uint64).astype(np.int64)
G = st.size // 20
arr = st[: 18 * G].reshape(18, G)
rel = st[18 * G: 18 * G + 18]
sm = st[19 * G: 20 * G]
nblk = (a.rows + 255) // 256
blocks = np.array([len(range(i, nblk, G)) for i in range(G)])
print(f"p={p} iterations={log.iterations} G={G} blocks/CTA min {blocks.min()} max {blocks.max()}")
late_rank = np.zeros(G)
for e in range(18):
    t = arr[e] - arr[e].min()
    late_rank += np.argsort(np.argsort(t)) / G
    q = np.percentile(t, [10, 50, 90, 99, 100]) * 1e-3
    print(f"barrier {10 + e} ({'pq' if e % 2 == 0 else 'rz'}): arrival spread p10 {q[0]:.2f} p50 {q[1]:.2f} "
          f"p90 {q[2]:.2f} p99 {q[3]:.2f} max {q[4]:.2f} us; wake {(rel[e] - arr[e].max()) * 1e-3:.2f} us; "
          f"corr(blocks) {np.corrcoef(t, blocks)[0, 1]:+.2f}")
late_rank /= 18
by_sm = {}
for i in range(G):
    by_sm.setdefault(int(sm[i]), []).append(late_rank[i])
sm_rank = np.array([np.mean(v) for k, v in sorted(by_sm.items())])
print(f"mean lateness rank per CTA: std {late_rank.std():.3f} (0.29 = random); per SM std {sm_rank.std():.3f}")
order = np.argsort(sm_rank)
keys = sorted(by_sm)
print("latest SMs:", [(keys[i], round(sm_rank[i], 2)) for i in order[-8:]])
print("earliest SMs:", [(keys[i], round(sm_rank[i], 2)) for i in order[:8]])
# same-CTA persistence: correlation of arrival order between consecutive same-kind barriers
cs = [np.corrcoef(arr[e] - arr[e].min(), arr[e + 2] - arr[e + 2].min())[0, 1] for e in range(16)]
print("corr of arrival times barrier e vs e+2:", np.round(cs, 2))
