"""Measurements for BASELINE configs #1, #3 and #4 (the headline #2 is bench.py).

    python tools/sweep_configs.py [--skip-cpu] > gpurun_out/sweep.json

#1  CSR SpMV fp64, 2-D Poisson 1000^2 (80 MB: fits the 126 MB L2, so every timed launch
    is preceded by a 256 MB L2-flush write, outside the timed events)
#3  SpMV format sweep on the 4M-row power-law matrix (fp64 and fp32): CSR (plan: nnz
    tiles; merge path beside it), COO, SELL-P(64), Hybrid(q0.8); ELL is infeasible (560 GB) and reported as such.
    GB/s on each format's own bytes and "useful" GB/s on the CSR bytes
#4  GMRES(30) and BiCGSTAB with Jacobi, fp64 3-D convection-diffusion 256^3, rtol 1e-8
CPU baselines: the oracle port (oracle/sbref.cpp) on 1 and all host threads.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_08230_b200 import gen  # noqa: E402
from paper_2510_08230_b200 import sparseops as sp  # noqa: E402

PEAK = 6543.1


def timed_spmv(mat, b, x, reps=20, flush=None):
    """Average launch time.  Without a flush: `reps` back-to-back launches between two
    events (the matrix is larger than L2).  With a flush: a 256 MB read before every
    launch, whose runtime hides the host enqueue latency of the timed launch."""
    for _ in range(3):
        mat.apply(b, x)
    torch.cuda.synchronize()
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            mat.apply(b, x)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3  # us
    total = 0.0
    for _ in range(reps):
        flush.sum()  # read-only sweep: L2 refilled with clean lines
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mat.apply(b, x)
        e1.record()
        torch.cuda.synchronize()
        total += e0.elapsed_time(e1)
    return total / reps * 1e3  # us


def fmt_bytes(mat, vb, ib):
    n = mat.rows
    if isinstance(mat, sp.CsrMatrix):
        return (vb + ib) * mat.nnz + ib * (n + 1) + 2 * vb * n
    if isinstance(mat, sp.CooMatrix):
        if mat.kernel_request == "auto":  # row-pointer index + CSR kernels: row_idxs never read
            return (vb + ib) * mat.nnz + ib * (n + 1) + 2 * vb * n
        return (vb + 2 * ib) * mat.nnz + 2 * vb * n
    if isinstance(mat, sp.SellpMatrix):
        return (vb + ib) * mat.stored + ib * (2 * mat.num_slices + 1) + 2 * vb * n
    if isinstance(mat, sp.HybridMatrix):
        return (vb + ib) * mat.ell.stored + (vb + 2 * ib) * mat.coo.nnz + 2 * vb * n
    if isinstance(mat, sp.EllMatrix):
        return (vb + ib) * mat.stored + 2 * vb * n
    raise TypeError(mat)


def cpu_spmv(rp, ci, v, b, threads, reps=5):
    from oracle import sbref
    sbref.csr_spmv(rp, ci, v, b, threads=threads)
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        sbref.csr_spmv(rp, ci, v, b, threads=threads)
        ts.append(time.perf_counter() - t)
    return float(np.median(ts))


def config1(dev, out, args, threads, flush):
    a = gen.poisson2d(dev, 1000)
    b = sp.dense_from_array(dev, torch.tensor(np.random.default_rng(0).random(a.rows)))
    x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
    us = timed_spmv(a, b, x, flush=flush)
    byt = fmt_bytes(a, 8, 4)
    rec = {"kernel": a.kernel, "us": us, "gbs": byt / us / 1e3, "frac": byt / us / 1e3 / PEAK,
           "gflops": 2 * a.nnz / us / 1e3, "bytes": byt,
           "l2": "flushed (1 GB read) before every launch"}
    if not args.skip_cpu:
        rp, ci, v = (t.cpu().numpy() for t in (a.row_ptrs, a.col_idxs, a.values))
        bv = b.numpy()[:, 0]
        rec["cpu_1thread_s"] = cpu_spmv(rp, ci, v, bv, 1)
        rec[f"cpu_{threads}threads_s"] = cpu_spmv(rp, ci, v, bv, threads)
    out["config1_poisson2d_1000_csr_f64"] = rec
    print(json.dumps({"config1": rec}), file=sys.stderr)


def config2(dev, out, args, threads, flush):
    """Poisson 128^3 format sweep (north_star: CSR and SELL-P >= 75% of the roofline)."""
    fsweep = {}
    for vdt, prec in ((np.float64, sp.Precision.double), (np.float32, sp.Precision.single)):
        a = gen.poisson3d(dev, 128, precision=prec)
        vb = prec.itemsize
        b = sp.dense_create(dev, a.rows, 1, prec, 1.0)
        x = sp.dense_create(dev, a.rows, 1, prec, 0.0)
        res = {}
        for name, m in {"csr": a, "coo": sp.coo_from_csr(a),
                        "coo_segmented": sp.coo_from_csr(a).with_kernel("segmented"), "ell": sp.ell_from_csr(a),
                        "sellp64": sp.sellp_from_csr(a, 64), "sellp32": sp.sellp_from_csr(a, 32),
                        "hybrid": sp.hybrid_from_csr(a)}.items():
            us = timed_spmv(m, b, x)
            byt = fmt_bytes(m, vb, 4)
            res[name] = {"us": us, "format_bytes": byt, "gbs": byt / us / 1e3,
                         "frac": byt / us / 1e3 / PEAK}
        fsweep[np.dtype(vdt).name] = res
        print(json.dumps({"config2_formats": np.dtype(vdt).name, "res": res}), file=sys.stderr)
    out["config2_poisson128_formats"] = fsweep


def config3(dev, out, args, threads, flush):
    sweep = {}
    for vdt, prec in ((np.float64, sp.Precision.double), (np.float32, sp.Precision.single)):
        a = gen.powerlaw_csr(dev, precision=prec)
        vb = prec.itemsize
        csr_bytes = fmt_bytes(a, vb, 4)
        bv = np.random.default_rng(0).random(a.rows).astype(vdt)
        b = sp.dense_from_array(dev, torch.tensor(bv))
        x = sp.dense_create(dev, a.rows, 1, prec, 0.0)
        mats = {"csr": a, "csr_merge": a.with_kernel("merge"), "csr_vector": a.with_kernel("vector"),
                "coo": sp.coo_from_csr(a), "coo_segmented": sp.coo_from_csr(a).with_kernel("segmented"),
                "sellp64": sp.sellp_from_csr(a, 64),
                "sellp64_sigma8192": sp.sellp_from_csr(a, 64, sigma=8192), "hybrid": sp.hybrid_from_csr(a)}
        res = {}
        for name, m in mats.items():
            us = timed_spmv(m, b, x)
            byt = fmt_bytes(m, vb, 4)
            res[name] = {"us": us, "format_bytes": byt, "gbs": byt / us / 1e3,
                         "frac": byt / us / 1e3 / PEAK, "useful_gbs": csr_bytes / us / 1e3,
                         "gflops": 2 * a.nnz / us / 1e3}
            if name == "csr":
                res[name]["kernel"] = a.kernel
            if name == "hybrid":
                res[name]["ell_width"] = m.ell.width
        res["ell"] = {"feasible": False, "reason": "max row length 11,668 -> 4M x 11,668 padded "
                      f"entries = {4e6 * 11668 * (vb + 4) / 1e9:.0f} GB"}
        if not args.skip_cpu:
            rp, ci, v = (t.cpu().numpy() for t in (a.row_ptrs, a.col_idxs, a.values))
            res["cpu_csr_1thread_s"] = cpu_spmv(rp, ci, v, bv, 1, reps=3)
            res[f"cpu_csr_{threads}threads_s"] = cpu_spmv(rp, ci, v, bv, threads, reps=3)
        sweep[np.dtype(vdt).name] = res
        print(json.dumps({"config3": np.dtype(vdt).name, "res": res}), file=sys.stderr)
        del mats, a
        torch.cuda.empty_cache()
    out["config3_powerlaw_4M"] = sweep


def config4(dev, out, args, threads, flush):
    a = gen.convdiff3d(dev, 256)
    m = sp.jacobi_create(a)
    solves = {}
    for name, cls, kw in (("gmres30", sp.Gmres, {"krylov_dim": 30}), ("bicgstab", sp.Bicgstab, {})):
        s = cls(a, criteria=[sp.Iteration(5000), sp.ResidualNorm(1e-8)], preconditioner=m, **kw)
        b = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 1.0)
        x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
        try:
            s.solve(b, x)  # warm (graph capture)
            x.values.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            log = s.solve(b, x)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            solves[name] = {"iterations": log.iterations, "converged": log.converged,
                            "final_residual": log.residual_history[-1], "solve_ms": ms,
                            "ms_per_iteration": ms / max(log.iterations, 1)}
        except (sp.errors.BreakdownError, sp.errors.NumericFailureError) as exc:
            h = exc.log.residual_history
            solves[name] = {"error": f"{exc.kind} at iteration {getattr(exc, 'iteration', '?')}",
                            "max_residual": max(h) if h else None}
        print(json.dumps({"config4": name, "res": solves[name]}), file=sys.stderr)
    out["config4_convdiff256_f64"] = solves


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--only", default="1,2,3,4", help="comma list of configs to run")
    args = ap.parse_args()
    dev = sp.create_device("cuda", 0)
    threads = len(os.sched_getaffinity(0))
    out = {"host_threads": threads}
    flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 1 GB (~170 us of reads: hides host launch latency)
    for c in args.only.split(","):
        {"1": config1, "2": config2, "3": config3, "4": config4}[c.strip()](dev, out, args, threads, flush)
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
