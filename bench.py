#!/usr/bin/env python
"""Benchmark: ILU(0)-PCG solve of BASELINE config 2 (2-D N=256, T=10, rtol 1e-10)
on the B200 path, with the reference CPU path timed beside it.

One "step" = one full ``pcg_solve`` (setup: GPU assembly of M + ILU(0)
factorisation; loop: sweeps + matvec + vector updates until rtol), inputs
resident in HBM.  ``value`` = DOF solved per second over the whole job
(K^d unknowns x solves / s, summed over ranks).  ``e2e`` runs the same solve
through the public numpy API (host F in, host x out).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--workload cfg2] [--stages] [--no-cpu-baseline]

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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg2")
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


def build_workload(args):
    from paper_2004_13961_b200 import workloads as wl
    kw = {}
    if args.N:
        kw["N"] = args.N
    if args.T is not None and args.workload != "cfg1":
        kw["T"] = args.T
    w = wl.CONFIGS[args.workload](**kw)
    if w.fhat is not None:
        F = wl.mass_contract_series(w.fhat)
    else:
        F = None
    return w, F


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


PROFILE_TAG = "r01e"   # cfg-2 sweep/ILU/matvec captures (profiles/r01e_*_full.csv)


def _ncu_rows(name):
    """Rows (dicts) of a committed ncu --set full summary: profiles/<tag>_<name>_full.csv."""
    import csv
    path = os.path.join(ROOT, "profiles", f"{PROFILE_TAG}_{name}_full.csv")
    try:
        with open(path) as f:
            lines = [ln for ln in f if not ln.startswith("#")]
    except OSError:
        return []
    rows = list(csv.reader(lines))
    if len(rows) < 3:
        return []
    return [dict(zip(rows[0], r)) for r in rows[2:]]


def ncu_traffic(name, kernel, per_call=1):
    """DRAM bytes (read + write) per call of `kernel` from the committed capture (cfg 2),
    summed over `per_call` consecutive launches (a precond_apply is 2 sweep launches)."""
    rows = [r for r in _ncu_rows(name) if kernel in r.get("Kernel Name", "")]
    if not rows:
        return None
    try:
        per = [float(r["dram__bytes_read.sum"]) + float(r["dram__bytes_write.sum"]) for r in rows]
    except (KeyError, ValueError):
        return None
    return sum(per) / len(per) * per_call


def sweep_traffic(workload):
    """DRAM bytes of one precond_apply (fwd + bwd box_sweep_kernel) from the committed capture."""
    return ncu_traffic("sweep", "box_sweep_kernel", 2) if workload == "cfg2" else None


def flush_l2(torch, buf):
    buf.zero_()


def ilu_flops(w):
    """F_ilu = 2 x (in-pattern IKJ updates), interior-row count x rows (SURVEY 8(d):
    73,008 / 132,300 updates per interior row for r = 12 / 14 in 2-D)."""
    r = w.T + 2
    if w.dim == 2:
        W = 2 * r + 1
        # updates of an interior row: pivots (ox, oy) < 0, targets in both boxes past k
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
        return 2.0 * upd * w.dofs
    return None


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

    w, F = build_workload(args)
    spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha, rhs=w.rhs_field)
    plan = TransformPlan(w.N + 1)
    if F is None:
        from paper_2004_13961_b200.operator import assemble_rhs
        F = assemble_rhs(spec, plan).data
    cfg = SolverConfig(epsilon=w.rtol, preconditioner=(w.T, w.T))
    n = w.dofs
    f_dev = device.to_device(np.asarray(F).flatten(order="F"))
    spec.device_operator(plan)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2

    for _ in range(args.warmup):
        x, rep = pcg_solve_device(spec, cfg, plan, f_dev)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    times = []
    launches = 0
    iters = None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush_l2(torch, flush)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            x, rep = pcg_solve_device(spec, cfg, plan, f_dev)
            e.record()
            e.synchronize()
            times.append(s.elapsed_time(e) / 1e3)
            launches += rep["kernel_launches"]
            iters = rep["iterations"]
    torch.cuda.synchronize()
    total = float(np.sum(times))
    if ws > 1:
        t = torch.tensor([total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    # setup launches (assembly 3 + factor 1 + tickets) are counted by the library too
    value = ws * args.steps * n / total

    # ---- e2e through the public numpy API (host F in, host x out)
    e2e_steps = max(1, min(args.steps, 3))
    Fh = SpectralCoeffs(np.asarray(F))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        xh, rh = pcg_solve(spec, cfg, plan, Fh)
    torch.cuda.synchronize()
    e2e_t = (time.perf_counter() - t0) / e2e_steps
    e2e = {"value": n / e2e_t, "unit": "DOF/s", "h2d_bytes_per_step": 8 * n,
           "d2h_bytes_per_step": 8 * n, "seconds_per_solve": e2e_t}

    # ---- stage breakdown (same objects, device resident)
    peaks, peaks_kind = measured_peaks()
    fp64 = dgemm_tflops(torch)
    t_setup0 = time.perf_counter()
    factors = setup_preconditioner(spec, cfg, plan)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup0
    from paper_2004_13961_b200.precond import assemble_M
    from paper_2004_13961_b200.sparse import ilu0
    # warm (the timed solves above already loaded every module); device events
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    ev[0].record()
    m = assemble_M(spec, w.T, w.T, plan)
    ev[1].record()
    ev[1].synchronize()
    t_asm = ev[0].elapsed_time(ev[1]) / 1e3
    fac_tmp = ilu0(m)          # first factorisation allocates the factor buffer
    torch.cuda.synchronize()
    ev[1].record()
    fac_tmp = ilu0(m)          # timed: copy of M + factorisation, buffers resident
    ev[2].record()
    ev[2].synchronize()
    t_fac = ev[1].elapsed_time(ev[2]) / 1e3
    del fac_tmp
    nnz = m.nnz
    r = torch.randn(n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    lib = _lib.load()
    h = factors._handle

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
    loop_per_iter = (np.mean(times) - t_setup) / max(iters, 1)
    stages = {"setup_s": t_setup, "assemble_s": t_asm, "ilu0_s": t_fac,
              "precond_apply_s": t_sweep, "matvec_s": t_mv, "iterations": iters,
              "loop_s_per_iter": loop_per_iter, "nnz_M": nnz}
    share = {"ilu0": t_fac, "sweeps": t_sweep * iters, "matvec": t_mv * iters}
    dom = max(share, key=share.get)
    sweep_kernel = "box_sweep3d_kernel" if w.dim == 3 else "box_sweep_kernel"
    roof_sweep = {"kernel": f"{sweep_kernel} fwd+bwd (precond_apply)", "bound": "hbm",
                  "achieved": sw_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                  "frac": sw_gbs / peaks["hbm_gbs"], "traffic": sweep_traffic(w.name),
                  "algorithmic_bytes": B_sw, "peak_source": peaks_kind}
    roof_mv = {"kernel": f"line_transform_kernel x{2 * w.dim} (apply_system)", "bound": "fp64",
               "achieved": mv_tf, "peak": fp64, "unit": "TFLOP/s", "frac": mv_tf / fp64,
               "traffic": None, "algorithmic_flops": F_alg,
               "peak_source": "cuBLAS DGEMM 8192^3 measured in this run"}
    F_ilu = ilu_flops(w)
    ilu_tf = F_ilu / t_fac / 1e12 if F_ilu else None
    roof_fac = {"kernel": "box_ilu0_tasks (2-D task graph)" if w.dim == 2 else "box_ilu0_3d_kernel",
                "bound": "latency (row-to-row dependency chain); fp64 rate shown",
                "achieved": ilu_tf, "peak": fp64, "unit": "TFLOP/s", "frac": ilu_tf / fp64 if ilu_tf else None,
                "traffic": ncu_traffic("ilu", "box_ilu0_tasks") if w.name == "cfg2" else None,
                "algorithmic_flops": F_ilu, "seconds": t_fac}
    roof = {"sweeps": roof_sweep, "matvec": roof_mv, "ilu0": roof_fac}[dom]
    result = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY 8(d))",
        "config": {"workload": f"{w.name}: {w.dim}-D N={w.N} T={w.T} rtol={w.rtol} ILU(0)-PCG",
                   "dofs": n, "parallelism": f"replicas{ws}" if ws > 1 else "single",
                   "l2": "flushed (256 MB write) before every step"},
        "solve_s": total / args.steps, "iterations": iters,
        "gpu_launches": launches,
        "e2e": e2e,
        "roofline": roof,
        "roofline_all": {"sweeps": roof_sweep, "matvec": roof_mv, "ilu0": roof_fac},
        "matvec_dof_per_s": n / t_mv,
        "fp64_dgemm_tflops": fp64,
        "stages": stages,
        "clocks": clk.summary(),
    }
    return result, w, F


def cpu_reference_solve(w, F, steps):
    """The reference algorithm on the host (oracle port: numpy/OpenBLAS + C ILU)."""
    from oracle import legpcg_port as orc
    from types import SimpleNamespace
    spec = SimpleNamespace(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha, rhs=w.rhs_field,
                           axis_betas=None)
    times = []
    it = None
    for _ in range(steps):
        t0 = time.perf_counter()
        _, rep = orc.pcg_solve(spec, F, epsilon=w.rtol, preconditioner=(w.T, w.T))
        times.append(time.perf_counter() - t0)
        it = rep["iterations"]
    return times, it


def main():
    args = parse()
    ws, rank, local = dist_info()
    if args.impl == "reference":
        if rank != 0:
            return
        w, F = build_workload(args)
        steps = max(1, min(args.steps, 3))
        warm = min(args.warmup, 1)
        if warm:
            cpu_reference_solve(w, F, warm)
        times, it = cpu_reference_solve(w, F, steps)
        total = float(np.sum(times))
        v = steps * w.dofs / total
        cores = os.cpu_count()
        out = {"metric": METRIC, "impl": "reference", "value": v, "unit": "DOF/s", "n_gpus": ws,
               "steps": steps, "warmup": warm, "ms_per_step": 1e3 * total / steps,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded, SURVEY 8(d))",
               "config": {"workload": f"{w.name}: {w.dim}-D N={w.N} T={w.T} rtol={w.rtol} "
                                      "ILU(0)-PCG", "dofs": w.dofs},
               "iterations": it,
               "cpu_baseline": {"value": v, "unit": "DOF/s", "cores": cores, "kind": "port",
                                "sample": f"{steps} full solve(s) of {w.name} (oracle port of "
                                          "the reference: numpy/OpenBLAS transforms on all "
                                          "cores, single-core C ILU(0)/sweeps)"},
               "e2e": {"value": v, "unit": "DOF/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    result, w, F = run_b200(args, ws, rank, local)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        times, it = cpu_reference_solve(w, F, 1)
        result["cpu_baseline"] = {"value": w.dofs / times[0], "unit": "DOF/s",
                                  "cores": os.cpu_count(), "kind": "port",
                                  "sample": f"1 full solve of {w.name} ({it} iterations, "
                                            f"{times[0]:.1f} s): oracle port, numpy/OpenBLAS "
                                            "on all cores + single-core C ILU(0)"}
    if args.stages and rank == 0:
        print(json.dumps(result["stages"]), file=sys.stderr)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result))


if __name__ == "__main__":
    main()
