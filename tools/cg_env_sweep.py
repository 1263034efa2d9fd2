"""Per-iteration time of the Jacobi-CG solve (fp64 Poisson p^3) under environment settings.

    python tools/cg_env_sweep.py 128 "" "SPARSEB200_CG_L2=1" "SPARSEB200_CG_L2=3" ...

Each setting runs in its own process (the library reads its knobs once); the solve is
timed with CUDA events over 5 solves after 2 warm-ups, like bench.py's step.
"""
import os
import subprocess
import sys

CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
from paper_2510_08230_b200 import gen
from paper_2510_08230_b200 import sparseops as sp
p = %d
dev = sp.create_device("cuda", 0)
a = gen.poisson3d(dev, p)
s = sp.Cg(a, criteria=[sp.Iteration(100000), sp.ResidualNorm(1e-8)], preconditioner=sp.jacobi_create(a))
b = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 1.0)
x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
for _ in range(2):
    x.values.zero_(); s.solve(b, x)
best = 1e9
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its = 0
    torch.cuda.synchronize(); e0.record()
    for _ in range(5):
        x.values.zero_(); its += s.solve(b, x).iterations
    e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / its * 1e3)
print(f"RESULT {its // 5} {best:.2f}")
'''

repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
p = int(sys.argv[1])
for setting in sys.argv[2:] or [""]:
    env = dict(os.environ)
    for kv in setting.split():
        k, v = kv.split("=", 1)
        env[k] = v
    out = subprocess.run([sys.executable, "-c", CHILD % (repo, p)], env=env, capture_output=True, text=True)
    res = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
    if res:
        _, its, us = res[0].split()
        print(f"{setting or '(default)':50s} iterations {its}  {us} us/iteration", flush=True)
    else:
        print(f"{setting or '(default)':50s} FAILED\n{out.stderr[-2000:]}", flush=True)
