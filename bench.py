#!/usr/bin/env python
"""Benchmark: ILU(0)-PCG solve of BASELINE config 3 (2-D N=2048, 4.19M unknowns,
T=12, rtol 1e-10) on the B200 path -- the largest single-GPU configuration --
with the reference CPU path timed beside it.

One "step" = one full ``pcg_solve`` (setup: GPU assembly of M + ILU(0)
factorisation; loop: sweeps + matvec + vector updates until rtol), the load
vector resident in HBM.  ``value`` = DOF solved per second over the whole job
(K^d unknowns x solves / s, summed over ranks).  ``e2e`` runs the same solve
through the public numpy API (host F in, host x out, copies inside the timed
region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--workload cfg3] [--N n] [--T t] [--stages] [--no-cpu-baseline]

CPU reference (``cpu_baseline`` and ``--impl reference``): the oracle port of
the reference algorithm (numpy/OpenBLAS transforms on all host cores, C ILU(0)
and sweeps single-threaded like the reference's numba kernels).  A full cfg-3
solve does not fit a CPU host's memory or time budget (the reference's
assemble_M alone needs far more than 62 GB), so each CPU step
is a bounded sample of the same workload: one full solve of the cfg-3
coefficient recipe at N = 192 (T = 12, rtol 1e-10), reported in the same
DOF/s unit.  CPU cost per DOF grows with N (the dense transforms are O(N) per
DOF and the iteration count rises), so the proxy overstates the CPU rate and
the GPU/CPU ratio is conservative.  The reference arm also times one
full-size cfg-3 matvec (apply_system) as a side figure.

Under torchrun (N > 1) every rank solves its own replica (the 2-D configs do
not shard): scaling "weak", time = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG solve s & fast-matvec DOF/s (fp64) at 2D/3D N; % HBM/FP64 roofline"
CPU_PROXY_N = 192          # bounded CPU sample of the workload (see module docstring)
PROFILE_TAG = "r02"        # committed ncu captures: profiles/<tag>_<workload>_<kernel>_full.csv


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--N", type=int, default=None)
    ap.add_argument("--T", type=int, default=None)
    ap.add_argument("--stages", action="store_true", help="print a per-stage breakdown")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def build_workload(name, N=None, T=None):
    from paper_2004_13961_b200 import workloads as wl
    kw = {}
    if N:
        kw["N"] = N
    if T is not None and name != "cfg1":
        kw["T"] = T
    w = wl.CONFIGS[name](**kw)
    F = wl.mass_contract_series(w.fhat) if w.fhat is not None else None
    return w, F


def workload_label(w):
    return f"{w.name}: {w.dim}-D N={w.N} T={w.T} rtol={w.rtol} ILU(0)-PCG"


# ---------------------------------------------------------------- clocks

class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------- helpers

def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0}, "fallback"


def dgemm_tflops(torch):
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    del a, b
    return 2.0 * n ** 3 / best / 1e12


def ncu_traffic(workload, kernel, per_call=1):
    """DRAM bytes (read + write) per call of `kernel` from the committed ncu
    --set full capture profiles/<tag>_<workload>_<kernel>_full.csv (mean over the
    captured launches, times `per_call` launches per call), or None."""
    import csv
    path = os.path.join(ROOT, "profiles", f"{PROFILE_TAG}_{workload}_{kernel}_full.csv")
    try:
        with open(path) as f:
            rows = list(csv.reader(ln for ln in f if not ln.startswith("#")))
    except OSError:
        return None
    if len(rows) < 3:
        return None
    recs = [dict(zip(rows[0], r)) for r in rows[2:]]
    try:
        per = [float(r["dram__bytes_read.sum"]) + float(r["dram__bytes_write.sum"]) for r in recs]
    except (KeyError, ValueError):
        return None
    return sum(per) / len(per) * per_call if per else None


def ilu_updates_per_row(dim, r):
    """In-pattern IKJ updates of an interior row."""
    W = 2 * r + 1
    if dim != 2:
        return None
    upd = 0
    for oy in range(-r, 1):
        for ox in range(-r, r + 1):
            if oy == 0 and ox >= 0:
                break
            for ty in range(oy, min(r, oy + r) + 1):
                for tx in range(max(-r, ox - r), min(r, ox + r) + 1):
                    if ty == oy and tx <= ox:
                        continue
                    upd += 1
    return upd


def matvec_flops(d, P, K):
    """F_alg: minimal sum-factorised flops with the exact parity split."""
    if d == 1:
        return 4.0 * P * K
    if d == 2:
        return P * K * (4.0 * K + 6.0 * P)
    return P * K * (4.0 * K * K + 6.0 * P * K + 8.0 * P * P)


def time_events(torch, fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / 1e3 / reps


# ---------------------------------------------------------------- arms

def run_b200(args, ws, rank, local):
    import torch
    torch.cuda.set_device(local)
    import torch.distributed as dist
    from paper_2004_13961_b200 import (ProblemSpec, SolverConfig, SpectralCoeffs, TransformPlan,
                                       pcg_solve)
    from paper_2004_13961_b200 import _lib, device
    from paper_2004_13961_b200.operator import apply_flat
    from paper_2004_13961_b200.pcg import pcg_solve_device, setup_preconditioner
    from paper_2004_13961_b200.precond import assemble_M
    from paper_2004_13961_b200.sparse import ilu0

    w, F = build_workload(args.workload, args.N, args.T)
    spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha, rhs=w.rhs_field)
    plan = TransformPlan(w.N + 1)
    if F is None:
        from paper_2004_13961_b200.operator import assemble_rhs
        F = assemble_rhs(spec, plan).data
    cfg = SolverConfig(epsilon=w.rtol, preconditioner=(w.T, w.T))
    n = w.dofs
    lib = _lib.load()
    f_dev = device.to_device(np.asarray(F).flatten(order="F"))
    spec.device_operator(plan)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2

    for _ in range(args.warmup):
        x, rep = pcg_solve_device(spec, cfg, plan, f_dev)
        del x
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    times = []
    launches = 0
    iters = None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            l0 = lib.lp_kernel_launches()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            x, rep = pcg_solve_device(spec, cfg, plan, f_dev)
            e.record()
            e.synchronize()
            times.append(s.elapsed_time(e) / 1e3)
            launches += lib.lp_kernel_launches() - l0
            iters = rep["iterations"]
            del x
    torch.cuda.synchronize()
    total = float(np.sum(times))
    if ws > 1:
        t = torch.tensor([total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    value = ws * args.steps * n / total

    # ---- e2e through the public numpy API (host F in, host x out, every step)
    Fh = SpectralCoeffs(np.asarray(F))
    e2e_times = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xh, rh = pcg_solve(spec, cfg, plan, Fh)
        e2e_times.append(time.perf_counter() - t0)
        del xh
    e2e_t = float(np.mean(e2e_times))
    if ws > 1:
        t = torch.tensor([e2e_t], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e = {"value": ws * n / e2e_t, "unit": "DOF/s", "h2d_bytes_per_step": 8 * n,
           "d2h_bytes_per_step": 8 * n, "seconds_per_solve": e2e_t}

    # ---- stage breakdown (device events, same objects)
    peaks, peaks_kind = measured_peaks()
    fp64 = dgemm_tflops(torch)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    flush.zero_()
    torch.cuda.synchronize()
    ev[0].record()
    m = assemble_M(spec, w.T, w.T, plan)
    ev[1].record()
    fac = ilu0(m)
    ev[2].record()
    ev[2].synchronize()
    t_asm = ev[0].elapsed_time(ev[1]) / 1e3
    t_fac = ev[1].elapsed_time(ev[2]) / 1e3
    nnz = m.nnz
    r = torch.randn(n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    h = fac._handle

    def sweep():
        lib.lp_precond_apply(h, r.data_ptr(), z.data_ptr(), _lib.stream_ptr())

    t_sweep = time_events(torch, sweep, 10)

    def mv():
        apply_flat(spec, plan, 3, r)

    t_mv = time_events(torch, mv, 20)
    P, K = w.P, w.K
    F_alg = matvec_flops(w.dim, P, K)
    B_sw = 8.0 * nnz + 32.0 * n
    sw_gbs = B_sw / t_sweep / 1e9
    mv_tf = F_alg / t_mv / 1e12
    solve_s = total / args.steps
    stages = {"assemble_s": t_asm, "ilu0_s": t_fac, "precond_apply_s": t_sweep, "matvec_s": t_mv,
              "iterations": iters, "loop_s_per_iter": (solve_s - t_asm - t_fac) / max(iters, 1),
              "nnz_M": nnz}
    share = {"ilu0": t_fac, "sweeps": t_sweep * iters, "matvec": t_mv * iters}
    dom = max(share, key=share.get)
    sweep_kernel = "box_sweep3d_kernel" if w.dim == 3 else "box_sweep_kernel"
    roof_sweep = {"kernel": f"{sweep_kernel} fwd+bwd (precond_apply)", "bound": "hbm",
                  "achieved": sw_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                  "frac": sw_gbs / peaks["hbm_gbs"],
                  "traffic": ncu_traffic(w.name, "sweep", 2),
                  "algorithmic_bytes": B_sw, "peak_source": peaks_kind,
                  "seconds": t_sweep, "share_of_step": t_sweep * iters / solve_s}
    roof_mv = {"kernel": f"line_transform_kernel x{2 * w.dim} (apply_system)", "bound": "fp64",
               "achieved": mv_tf, "peak": fp64, "unit": "TFLOP/s", "frac": mv_tf / fp64,
               "traffic": ncu_traffic(w.name, "matvec", 2 * w.dim), "algorithmic_flops": F_alg,
               "peak_source": "cuBLAS DGEMM 8192^3 measured in this run",
               "seconds": t_mv, "share_of_step": t_mv * iters / solve_s}
    upd = ilu_updates_per_row(w.dim, w.T + 2)
    F_ilu = 2.0 * upd * n if upd else None
    ilu_tf = F_ilu / t_fac / 1e12 if F_ilu else None
    roof_fac = {"kernel": "ilu2d_kernel (2-D block wavefront)" if w.dim == 2 else "box_ilu0_3d_kernel",
                "bound": "fp64 (separately rounded mul + sub, bitwise reference order: vector pipe, no "
                         "FMA and no tensor cores -- its own ceiling is 18.6 TFLOP/s, measured by "
                         "scripts/micro/fp64_tput.cu; frac is against the DGEMM peak)",
                "achieved": ilu_tf, "peak": fp64, "unit": "TFLOP/s",
                "frac": ilu_tf / fp64 if ilu_tf else None,
                "traffic": ncu_traffic(w.name, "ilu", 1), "algorithmic_flops": F_ilu,
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run",
                "seconds": t_fac, "share_of_step": t_fac / solve_s}
    del fac, m
    roof = {"sweeps": roof_sweep, "matvec": roof_mv, "ilu0": roof_fac}[dom]
    result = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY 8(d))",
        "config": {"workload": workload_label(w), "dofs": n,
                   "parallelism": f"replicas{ws}" if ws > 1 else "single",
                   "l2": "flushed (256 MB write) before every step; factors 28 GB >> L2"},
        "solve_s": solve_s, "iterations": iters,
        "gpu_launches": launches,
        "e2e": e2e,
        "roofline": roof,
        "roofline_all": {"sweeps": roof_sweep, "matvec": roof_mv, "ilu0": roof_fac},
        "matvec_dof_per_s": n / t_mv,
        "fp64_dgemm_tflops": fp64,
        "stages": stages,
        "clocks": clk.summary(),
    }
    return result, w


def cpu_port_solves(steps, N=CPU_PROXY_N, workload="cfg3"):
    """The reference algorithm on the host (oracle port), on the bounded sample:
    full solves of the workload's coefficient recipe at size N.  Returns
    (seconds per solve list, iterations, dofs)."""
    from oracle import legpcg_port as orc
    from types import SimpleNamespace
    w, F = build_workload(workload, N)
    spec = SimpleNamespace(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha, rhs=w.rhs_field,
                           axis_betas=None)
    times, it = [], None
    for _ in range(steps):
        t0 = time.perf_counter()
        _, rep = orc.pcg_solve(spec, F, epsilon=w.rtol, preconditioner=(w.T, w.T))
        times.append(time.perf_counter() - t0)
        it = rep["iterations"]
    return times, it, w.dofs


def cpu_full_matvec_s(workload):
    """One full-size apply_system on the host (oracle port, OpenBLAS on all cores)."""
    from oracle import legpcg_port as orc
    from types import SimpleNamespace
    w, _ = build_workload(workload)
    spec = SimpleNamespace(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha, rhs=w.rhs_field,
                           axis_betas=None)
    u = np.random.default_rng(7).standard_normal((w.K,) * w.dim)
    plan = orc.Plan(w.N + 1)
    orc.apply_system(spec, plan, u)
    t0 = time.perf_counter()
    orc.apply_system(spec, plan, u)
    return time.perf_counter() - t0


def sample_text(workload, N, it, t):
    w, _ = build_workload(workload, N)
    head = (f"full ILU(0)-PCG solve of the {workload} coefficient recipe at N={N} "
            f"(T={w.T}, rtol {w.rtol:g}, {it} iterations, {t:.1f} s): oracle port of the reference, "
            "numpy/OpenBLAS on all host cores + single-threaded C ILU(0)/sweeps")
    if N == {"cfg1": 128, "cfg2": 256, "cfg3": 2048, "cfg4": 128, "cfg5": 512}.get(workload):
        return head + "; this is the full-size workload"
    return (head + f"; the full-size {workload} solve does not fit a CPU host (SURVEY 8(c)), so this "
            "bounded sample stands in for it (CPU cost per DOF grows with N: conservative)")


def run_reference(args, ws, rank):
    if rank != 0:
        return
    w, _ = build_workload(args.workload, args.N, args.T)
    N = CPU_PROXY_N if w.name == "cfg3" and not args.N else w.N
    warm = min(args.warmup, 1)
    if warm:
        cpu_port_solves(warm, N, w.name)
    times, it, dofs = cpu_port_solves(args.steps, N, w.name)
    total = float(np.sum(times))
    v = args.steps * dofs / total
    cores = os.cpu_count()
    extra = {}
    try:
        extra["full_size_matvec_s"] = cpu_full_matvec_s(w.name)
    except MemoryError:
        extra["full_size_matvec_s"] = None
    out = {"metric": METRIC, "impl": "reference", "value": v, "unit": "DOF/s", "n_gpus": ws,
           "steps": args.steps, "warmup": warm, "ms_per_step": 1e3 * total / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded, SURVEY 8(d))",
           "config": {"workload": workload_label(w), "dofs": w.dofs, "cpu_sample_N": N,
                      "cpu_sample_dofs": dofs},
           "iterations": it,
           "cpu_baseline": {"value": v, "unit": "DOF/s", "cores": cores, "kind": "port",
                            "sample": sample_text(w.name, N, it, float(np.mean(times)))},
           "e2e": {"value": v, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           **extra}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    ws, rank, local = dist_info()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    result, w = run_b200(args, ws, rank, local)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        N = CPU_PROXY_N if w.name == "cfg3" and not args.N else w.N
        times, it, dofs = cpu_port_solves(1, N, w.name)
        result["cpu_baseline"] = {"value": dofs / times[0], "unit": "DOF/s",
                                  "cores": os.cpu_count(), "kind": "port",
                                  "sample": sample_text(w.name, N, it, times[0])}
    if args.stages and rank == 0:
        print(json.dumps(result["stages"]), file=sys.stderr)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


if __name__ == "__main__":
    main()
