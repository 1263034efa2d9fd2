"""Benchmark: Jacobi-preconditioned CG, fp64, 3-D 7-point Poisson 128^3 (BASELINE config #2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one full solve (b = 1, x0 = 0, rtol 1e-8 -> ~319 iterations) through the
device solver.  `value` = CG iterations per second over all ranks with every input
resident in HBM (device-timed with CUDA events, max over ranks); `e2e` = the same
metric through the public frontend API (pysparseops) with host buffers: each step
copies b and x0 from pinned host memory, solves, and copies x back.

`roofline` is for the dominant kernel, the CSR SpMV (TMA-staged stream kernel) that
runs once per CG iteration: algorithmic bytes per launch (12*nnz +
4*(n+1) + 8n + 8n = 216,924,164 B at 128^3) / its CUDA-event launch duration,
against the measured HBM copy bandwidth in MEASURED_PEAKS.json.  `cpu_baseline` is
the oracle port (oracle/sbref.cpp) of the reference's CG on this host's cores for a
bounded sample of iterations.

Multi-GPU (N > 1; under torchrun, or `--gpus N` alone, which re-launches itself through
torch.distributed.run with N ranks): the SAME global system is row-partitioned across
the N GPUs (paper_2510_08230_b200.dist: NCCL halo exchange overlapped with the interior
SpMV, ncclAllReduce of the local dots, the graph-loop DistCg of csrc/dist_krylov.cu) ->
strong scaling; `value` stays global CG iterations per second.  The default workload is
cg128 at EVERY N, so the driver's 1/2/4/8 series is one problem (strong scaling of
config #2; latency-bound beyond 2-4 GPUs at 2.1M rows).  `--workload cg512` selects
BASELINE config #5 (Poisson 512^3, 134M rows), the north_star strong-scaling problem.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "SpMV GB/s & % HBM roofline; CG solve time/iters/s, Poisson-3D fp64, 1/2/4/8 GPU"
WORKLOADS = {"cg128": 128, "cg512": 512}
P = 128
RTOL = 1e-8


def _peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks",
               0x1: "gpu_idle"}

    def __init__(self, index):
        self.samples, self.reasons = [], set()
        self.stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.nv:
            self.stop.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _max_over_ranks(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_baseline_sample(iters=60):
    """Oracle port of the reference's Jacobi-CG (oracle/sbref.cpp) on all host threads,
    fixed-iteration sample at 128^3 -> iterations/s."""
    import numpy as np

    from oracle import fixtures, sbref

    rp, ci, v = fixtures.stencil_csr(P, dim=3)
    inv, _ = sbref.jacobi_create(rp, ci, v)
    b = np.ones(rp.size - 1)
    threads = len(os.sched_getaffinity(0))
    sbref.solve("cg", rp, ci, v, b, inv_diag=inv, max_iters=2, threads=threads)  # warm
    t0 = time.perf_counter()
    log, _ = sbref.solve("cg", rp, ci, v, b, inv_diag=inv, max_iters=iters, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": log.iterations / dt, "unit": "CG iters/s", "cores": threads, "kind": "port",
            "sample": f"{log.iterations} fixed Jacobi-CG iterations, fp64 Poisson 128^3, "
                      f"oracle/sbref.cpp (C++ restatement of the reference), {dt:.2f} s"}


def reference_numba_sample(iters=20):
    """The reference ITSELF (sparseops, pure Python + numba, installed unmodified into
    baseline/_ref by `pip install --no-deps --target baseline/_ref`) running its own
    Jacobi-CG (solvers.py:188-224) on the `omp` device with every host thread
    (BASELINE.md §4): a fixed-iteration sample at 128^3 -> iterations/s.  None when the
    install is absent.  Matrix construction and jacobi_create are outside the timing."""
    path = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "sparseops")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_sparseops")
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import sparseops as ref  # the reference (top-level name; ours is paper_2510_08230_b200.sparseops)
    except Exception:
        return None
    from oracle import fixtures

    threads = len(os.sched_getaffinity(0))
    n, ri, ci, v = fixtures.stencil3d_triplets(P)
    dev = ref.create_device("omp", threads=threads)
    t0 = time.perf_counter()
    a = ref.csr_from_coo(ref.coo_from_arrays(dev, n, n, ri, ci, v, ref.Precision.double, ref.IndexWidth.i32))
    m = ref.jacobi_create(a)
    setup = time.perf_counter() - t0
    b = ref.dense_create(dev, n, 1, ref.Precision.double, 1.0)
    x = ref.dense_create(dev, n, 1, ref.Precision.double, 0.0)
    ref.Cg(a, criteria=[ref.Iteration(2)], preconditioner=m).solve(b, x)  # numba JIT warm-up
    x = ref.dense_create(dev, n, 1, ref.Precision.double, 0.0)
    t0 = time.perf_counter()
    log = ref.Cg(a, criteria=[ref.Iteration(iters)], preconditioner=m).solve(b, x)
    dt = time.perf_counter() - t0
    return {"value": log.iterations / dt, "unit": "CG iters/s", "cores": threads, "kind": "reference",
            "sample": f"{log.iterations} fixed Jacobi-CG iterations, fp64 Poisson 128^3, the reference "
                      f"sparseops (numba) on omp[{threads}] from baseline/_ref, {dt:.2f} s "
                      f"(setup incl. jacobi_create {setup:.1f} s, untimed)"}


def run_reference(args):
    world, rank, _ = _dist()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rank != 0:
            dist.barrier()
            return
    for _ in range(args.warmup):
        cpu_baseline_sample(10)
    vals = [cpu_baseline_sample(30)["value"] for _ in range(args.steps)]
    base = cpu_baseline_sample(30)
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "CG iters/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 30 * 1000.0 / v, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "Jacobi-CG fp64 3-D 7-pt Poisson 128^3, rtol 1e-8 "
                                   "(fixed-iteration CPU sample of 30 iterations per step)"},
            "cpu_baseline": {**base, "value": v},
            "reference_numba": reference_numba_sample(),
            "e2e": {"value": v, "unit": "CG iters/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _spmv_roofline(a, dev, stream, torch, sp):
    """Average CUDA-event duration of the dominant kernel (the CSR SpMV of the iteration)
    over 50 back-to-back launches on the solver's stream."""
    n, nnz = a.rows, a.nnz
    p_vec = sp.dense_create(dev, a.cols, 1, sp.Precision.double, 1.0)
    q_vec = sp.dense_create(dev, n, 1, sp.Precision.double, 0.0)
    for _ in range(5):
        a.apply(p_vec, q_vec)
    reps = 50
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s0.record(stream)
    for _ in range(reps):
        a.apply(p_vec, q_vec)
    s1.record(stream)
    torch.cuda.synchronize()
    spmv_ms = s0.elapsed_time(s1) / reps
    spmv_bytes = a.precision.itemsize * (nnz + n + a.cols) + a.index_width.itemsize * (nnz + n + 1)
    peak, peak_kind = _peaks()
    achieved = spmv_bytes / (spmv_ms / 1e3) / 1e9
    traffic = None
    for name in ("r2_spmv_traffic.json", "r1_spmv_traffic.json"):  # newest committed capture first
        try:  # DRAM bytes per launch from the committed ncu --set full capture of this kernel
            with open(os.path.join(REPO, "profiles", name)) as fh:
                t = json.load(fh)
            if t["algorithmic_bytes"] == spmv_bytes:
                traffic = t["traffic"]
                break
        except Exception:
            pass
    return spmv_ms, spmv_bytes, {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "kernel": f"csr_{a.kernel}_kernel<double,int>",
        "alg_bytes_per_launch": spmv_bytes, "peak_source": peak_kind}


def _persistent_traffic(iter_bytes):
    """DRAM bytes per CG iteration of the persistent kernel from the committed ncu
    --set full capture (profiles/), if it was taken for this byte model."""
    for name in ("r2_cg_persistent_traffic.json", "r1_cg_persistent_traffic.json"):
        try:
            with open(os.path.join(REPO, "profiles", name)) as fh:
                t = json.load(fh)
            if t["algorithmic_bytes_per_iteration"] == iter_bytes:
                return t["traffic_per_iteration"]
        except Exception:
            pass
    return None


def run_ours(args):
    import torch

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    if world > 1 or args.partitioned:
        import torch.distributed as dist
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return run_partitioned(args, world, rank, local)

    from paper_2510_08230_b200 import gen
    from paper_2510_08230_b200 import pysparseops as pg
    from paper_2510_08230_b200 import sparseops as sp

    p = WORKLOADS[args.workload]
    dev = sp.create_device("cuda", local)
    stream = torch.cuda.current_stream()
    a = gen.poisson3d(dev, p)
    n, nnz = a.rows, a.nnz
    m = sp.jacobi_create(a)
    solver = sp.Cg(a, criteria=[sp.Iteration(100000), sp.ResidualNorm(RTOL)], preconditioner=m)
    b = sp.dense_create(dev, n, 1, sp.Precision.double, 1.0)
    x = sp.dense_create(dev, n, 1, sp.Precision.double, 0.0)

    def step():
        x.values.zero_()
        return solver.solve(b, x)

    for _ in range(max(args.warmup, 1)):
        log = step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            log = step()
            iters += log.iterations
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    value = iters / (ms / 1000.0)

    from paper_2510_08230_b200 import _lib
    loop = int(_lib.fn("sb_cg_last_loop")())  # 3 persistent kernel, 1 fused graph, 0 three-kernel
    spmv_ms, spmv_bytes, spmv_roof = _spmv_roofline(a, dev, stream, torch, sp)
    peak = spmv_roof["peak"]
    # algorithmic bytes of one iteration (SURVEY.md 8d / DESIGN.md 3): matrix once, plus
    # 12 vector passes for the fused loops (gather z, p_old; write q, p; read p, q, x, r, M;
    # write x, r, z), 13 for the three-kernel loop
    a_bytes = 12 * nnz + 4 * (n + 1)
    cg_iter_bytes = a_bytes + (13 if loop == 0 else 12) * 8 * n
    cg_iter_ms = ms / max(iters, 1)
    if loop == 3:
        # dominant kernel = the persistent CG kernel (one launch per solve, >99% of the
        # step); its duration is taken as the whole solve (setup SpMV + init included)
        achieved = cg_iter_bytes / (cg_iter_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": _persistent_traffic(cg_iter_bytes),
                    "kernel": f"cg_persistent_kernel<double,int,{int(_lib.fn('sb_cg_last_block_rows')())}>",
                    "alg_bytes_per_launch": cg_iter_bytes * log.iterations,
                    "launch_us": ms / args.steps * 1e3, "peak_source": spmv_roof["peak_source"],
                    "note": "bytes per launch = iterations x (matrix + 12 vector passes); "
                            "traffic per iteration from the committed ncu capture"}
        launches = args.steps * 3
    else:
        roofline = spmv_roof
        launches = args.steps * (2 + (4 * ((log.iterations + 1) // 2) if loop == 1 else 3 * log.iterations))

    # ---- e2e: public frontend API with host buffers (pinned), copies inside the region
    pdev = pg.device("cuda", local)
    bh = torch.ones(n, dtype=torch.float64).pin_memory()
    x0h = torch.zeros(n, dtype=torch.float64).pin_memory()
    xh = torch.empty(n, dtype=torch.float64).pin_memory()
    cg = pg.solver.cg(pdev, a, pg.preconditioner.Jacobi(pdev, a), max_iters=100000,
                      reduction_factor=RTOL)

    def e2e_step():
        bt = pg.as_tensor(bh.to(dev.torch, non_blocking=True), device=pdev)
        xt = pg.as_tensor(x0h.to(dev.torch, non_blocking=True), device=pdev)
        logger, res = cg.apply(bt, xt)
        xh.copy_(res.values, non_blocking=True)
        return logger

    for _ in range(max(args.warmup, 1)):
        e2e_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_iters = 0
    e0.record(stream)
    for _ in range(args.steps):
        e_iters += e2e_step().iterations
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_value = e_iters / (e0.elapsed_time(e1) / 1e3)
    assert abs(float(xh[n // 2]) - float(x.values[n // 2])) <= 1e-6 * abs(float(x.values[n // 2]))

    cpu = cpu_baseline_sample() if not args.no_cpu and p == 128 else None
    cpu_ref = reference_numba_sample() if not args.no_cpu and p == 128 else None
    line = {
        "metric": METRIC, "value": value, "unit": "CG iters/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (device-generated 7-point Poisson stencil, b = 1, x0 = 0)",
        "config": {"workload": f"Jacobi-CG fp64 3-D 7-pt Poisson {p}^3 (n={n:,}, nnz={nnz:,}), "
                               f"rtol 1e-8, CSR",
                   "parallelism": "single GPU",
                   "l2": "inputs larger than L2 (CG working set >= 284 MB vs 126 MB L2); no flush"},
        "iterations_per_solve": log.iterations,
        "solve_ms": ms / args.steps,
        "cg_iteration": {"ms": cg_iter_ms, "alg_bytes": cg_iter_bytes,
                         "gbs": cg_iter_bytes / (cg_iter_ms / 1e3) / 1e9,
                         "frac_of_hbm": cg_iter_bytes / (cg_iter_ms / 1e3) / 1e9 / peak},
        "cg_loop": {3: "persistent cooperative kernel", 1: "graph loop, fused direction",
                    0: "graph loop, three kernels"}.get(loop, str(loop)),
        "spmv": {"kernel": a.kernel, "us": spmv_ms * 1e3, "gbs": spmv_roof["achieved"],
                 "gflops": 2 * nnz / (spmv_ms / 1e3) / 1e9, "roofline_frac": spmv_roof["frac"],
                 "traffic": spmv_roof["traffic"]},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "cpu_baseline_reference_numba": cpu_ref,
        "e2e": {"value": e2e_value, "unit": "CG iters/s", "h2d_bytes_per_step": 2 * 8 * n,
                "d2h_bytes_per_step": 8 * n + 64},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line))


def run_partitioned(args, world, rank, local):
    """Strong scaling: the same global Poisson system row-partitioned over `world` GPUs."""
    import torch
    import torch.distributed as dist

    from paper_2510_08230_b200 import dist as D
    from paper_2510_08230_b200 import sparseops as sp

    p = WORKLOADS[args.workload]
    dev = sp.create_device("cuda", local)
    stream = torch.cuda.current_stream()
    comm = D.NcclComm(rank, world)
    part = D.stencil_partition(dev, p, rank, world)
    nl = part.n_local
    solver = D.DistCg(part, [sp.Iteration(100000), sp.ResidualNorm(RTOL)], comm=comm)
    b = sp.dense_create(dev, nl, 1, sp.Precision.double, 1.0)
    x = sp.dense_create(dev, nl, 1, sp.Precision.double, 0.0)

    def step():
        x.values.zero_()
        return solver.solve(b, x)

    for _ in range(max(args.warmup, 1)):
        log = step()
    torch.cuda.synchronize()
    dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            log = step()
            iters += log.iterations
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = _max_over_ranks(ev0.elapsed_time(ev1), world)
    dist.barrier()
    value = iters / (ms / 1000.0)  # global system: iterations are not multiplied by ranks

    _, _, roofline = _spmv_roofline(part.matrix, dev, stream, torch, sp)

    # e2e: host slabs of b and x0 -> device, solve, x slab back
    bh = torch.ones(nl, dtype=torch.float64).pin_memory()
    x0h = torch.zeros(nl, dtype=torch.float64).pin_memory()
    xh = torch.empty(nl, dtype=torch.float64).pin_memory()

    def e2e_step():
        bt = sp.dense_from_array(dev, bh.to(dev.torch, non_blocking=True))
        xt = sp.dense_from_array(dev, x0h.to(dev.torch, non_blocking=True))
        lg = solver.solve(bt, xt)
        xh.copy_(xt.values, non_blocking=True)
        return lg

    e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_iters = 0
    e0.record(stream)
    for _ in range(args.steps):
        e_iters += e2e_step().iterations
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = _max_over_ranks(e0.elapsed_time(e1), world)
    comm.close()
    if rank == 0:
        n = p ** 3
        line = {
            "metric": METRIC, "value": value, "unit": "CG iters/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-generated 7-point Poisson stencil slabs, b = 1, x0 = 0)",
            "config": {"workload": f"row-partitioned Jacobi-CG fp64 3-D 7-pt Poisson {p}^3 "
                                   f"(n={n:,}), rtol 1e-8, CSR slabs",
                       "parallelism": f"row partition over {world} GPUs, NCCL halo + allreduce",
                       "l2": "inputs larger than L2 per rank at 512^3; no flush"},
            "iterations_per_solve": log.iterations, "solve_ms": ms / args.steps,
            "roofline": roofline, "cpu_baseline": None,
            "e2e": {"value": e_iters / (e_ms / 1e3), "unit": "CG iters/s",
                    "h2d_bytes_per_step": 2 * 8 * nl, "d2h_bytes_per_step": 8 * nl},
            "gpu_launches": args.steps * (8 + 10 * log.iterations),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line))
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the row-partitioned NCCL solver even on one GPU")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cg128",
                    help="cg128 = BASELINE config #2 (default); cg512 = config #5")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        run_ours(args)


def spawn_ranks(args):
    """`bench.py --gpus N` without a launcher: re-run this script under
    torch.distributed.run with N ranks on this node (rendezvous on 127.0.0.1); rank 0's
    JSON line passes through on stdout."""
    import socket
    import subprocess

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    main()
