#!/usr/bin/env python
"""Benchmark of the shift-invert quadratic eigensolve hot path (arXiv 2112.14064).

Arms:
  default (B200)        librq_b200.so on cuda:LOCAL_RANK through the C-ABI.
  --impl reference      the reference's CPU path: oracle/_ref/liboracle_ref.so
                        (reference kern:: kernels compiled from /root/reference +
                        the SPEC restatement), else the oracle port; 1 thread
                        (the reference has no threading); rank 0 only.

One step = one numeric multifrontal LU of Q(sigma) of the configured pencil
(BASELINE metric "FP64 LU-factor GFLOP/s"); the same line reports the time to
nev eigenpairs (factor + Krylov-Schur to converged pairs) and the per-kernel
rooflines. Multi-GPU: replicas only - every rank factors its
own copy, value = sum of per-rank work / max-over-ranks time.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 LU-factor GFLOP/s + time to nev eigenpairs, as % of FP64/HBM roofline"
SIGMA = -0.5
NEV = {"cfg1": 10, "cfg2_riga": 20, "cfg2_iga": 20, "cfg3_riga": 50, "cfg3_iga": 50,
       "cfg4_riga": 100, "cfg4_iga": 100}
FP64_PEAK_TFLOPS = 37.2   # measured DMMA m16n8k4 issue rate, profiles/fp64_peak_r01.jsonl
FP64_DFMA_TFLOPS = 36.7   # measured DFMA rate (same file)
KINDS = ["scatter_original", "extend_add", "front_lu_smem", "panel_lu", "panel_apply+rowperm",
         "schur_dmma", "factor_dag"]


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev=0):
        self.dev, self.samples, self.stop = dev, [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    return rank, ws, local


def allreduce_max(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def host_info():
    """nproc and CPU model of the box the CPU baseline ran on."""
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "pinned_core": 0}


def pin_core0():
    """The reference path is single-threaded (taskset -c 0)."""
    try:
        os.sched_setaffinity(0, {0})
    except (AttributeError, OSError):
        pass


def cpu_factor_sample(P, kind, budget_s):
    """Oracle factorization timed on the host (1 thread, pinned), bounded sample."""
    import oracle
    old = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    pin_core0()
    Q = P.q_values(SIGMA)
    ts = []
    t_end = time.perf_counter() + budget_s
    while True:
        t0 = time.perf_counter()
        f = oracle.Factor(P.n, P.rowptr, P.col, Q, P.box, P.elems, kind=kind)
        ts.append(time.perf_counter() - t0)
        del f
        if time.perf_counter() > t_end or len(ts) >= 50:
            break
    if old is not None:
        os.sched_setaffinity(0, old)
    return ts


def run_reference(args):
    rank, ws, _ = dist_init()
    if rank != 0:
        return
    pin_core0()
    import oracle
    import paper_2112_14064_b200 as rq
    kind = "reference" if oracle.ref() is not None else "port"
    P = rq.baseline_config(args.config)
    o = rq.nested_dissection_order(P)
    flu = o.stats["flops_lu"]
    Q = P.q_values(SIGMA)
    for _ in range(args.warmup):
        oracle.Factor(P.n, P.rowptr, P.col, Q, P.box, P.elems, kind=kind)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.Factor(P.n, P.rowptr, P.col, Q, P.box, P.elems, kind=kind)
        ts.append(time.perf_counter() - t0)
    sec = sum(ts) / len(ts)
    gf = flu / sec / 1e9
    tnev = None
    if args.nev_cpu:
        t0 = time.perf_counter()
        E = oracle.Eig(P, SIGMA, kind=kind)
        E.solve_quadratic(NEV.get(args.config, 20), tol=1e-10, max_restarts=args.max_restarts)
        tnev = (time.perf_counter() - t0) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gf, 4), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128 (reference cdouble; real-flop count F_LU)",
        "data": "synthetic (deterministic BASELINE assembly)",
        "config": {"workload": args.config, "sigma": SIGMA, "nev": NEV.get(args.config, 20),
                   "n": P.n, "nnz": P.nnz, "flops_lu_real": flu, "parallelism": "1 host thread"},
        "time_to_nev_ms": tnev,
        "cpu_baseline": {"value": round(gf, 4), "unit": "GFLOP/s", "cores": 1, "kind": kind,
                         "sample": f"{args.steps} full factorizations of {args.config}",
                         "host": host_info()},
        "e2e": {"value": round(gf, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args):
    rank, ws, local = dist_init()
    import numpy as np

    import paper_2112_14064_b200 as rq
    from paper_2112_14064_b200 import _lib
    import ctypes as C
    _lib.check(_lib.lib.rq_set_device(local))
    peaks = measured_peaks()
    P = rq.baseline_config(args.config)
    nev = args.nev or NEV.get(args.config, 20)
    o = rq.nested_dissection_order(P)
    st = o.stats
    flu = st["flops_lu"]
    op = rq.build_operator(P, SIGMA, o)
    fh = _lib.lib.rq_operator_factor(op._h)

    def time_what(what, iters, param=0):
        ms = C.c_double()
        _lib.check(_lib.lib.rq_operator_time(op._h, what, iters, param, C.byref(ms)))
        return ms.value

    # ---- device-resident steps: numeric factorization (graph replay), L2 flushed between steps
    time_what(5 | 0x100, max(args.warmup, 3))
    barrier(ws)
    with ClockSampler(local) as clk:
        ms_step = time_what(5 | 0x100, args.steps)
    ms_max = allreduce_max(ms_step, ws)
    value = ws * flu / (ms_max * 1e6)  # GFLOP/s, whole job

    # ---- time to nev eigenpairs (device-resident pencil; factor + Krylov-Schur)
    t_nev = []
    info = {}
    for _ in range(max(1, args.nev_runs)):
        t0 = time.perf_counter()
        pairs = op.solve_quadratic(nev, eps=1e-10, seed=0, max_restarts=args.max_restarts,
                                   raise_partial=False)
        t_nev.append((time.perf_counter() - t0) * 1e3 + op.factor_info()["factor_ms"])
        info = op.last_info
    resid_max = max(p.residual for p in pairs)

    # ---- per-kernel profile of one factorization (un-graphed, events per launch)
    ms_k = np.zeros(7)
    cnt_k = np.zeros(7, np.int64)
    work_k = np.zeros(7)
    _lib.check(_lib.lib.rq_factor_profile(fh, ms_k, cnt_k, work_k))
    dom = int(np.argmax(ms_k))
    # ---- memory-bound kernels of the Krylov step
    t_solve = time_what(1 | 0x100, 20)
    t_spmv = time_what(2 | 0x100, 50)
    m = 2 * nev + 1
    t_gemv = time_what(3 | 0x100, 20, m)
    solve_bytes = st["trisolve_bytes"]
    spmv_bytes = 20.0 * P.nnz + 8.0 * (P.n + 1) + 24.0 * P.n
    gemv_bytes = 8.0 * 2 * P.n * m
    hbm = peaks.get("hbm_gbs", 6650.0)

    # ---- e2e through the public API with host buffers (pinned), H2D + D2H inside
    Q = P.q_values(SIGMA)
    try:
        import torch
        pin = torch.empty(P.nnz, dtype=torch.float64, pin_memory=True)
        pin.copy_(torch.from_numpy(Q))
        Qh = pin.numpy()
    except Exception:  # noqa: BLE001
        Qh = np.ascontiguousarray(Q)
    fac = rq.lu_factorize((P.rowptr, P.col, Qh), o)
    for _ in range(max(args.warmup, 3)):
        fac.refactor(Qh)
    barrier(ws)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fac.refactor(Qh)   # H2D of Q(sigma) values, factor, D2H of the pivot/singular flags
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    e2e_ms = allreduce_max(e2e_ms, ws)
    launches = fac.info()["launches"]
    # e2e time to nev from host arrays: operator creation (H2D of K, C, M, Q, factor) + eigs
    t0 = time.perf_counter()
    op2 = rq.build_operator(P, SIGMA, o)
    op2.solve_quadratic(nev, eps=1e-10, seed=0, max_restarts=args.max_restarts, raise_partial=False)
    e2e_nev_ms = (time.perf_counter() - t0) * 1e3
    del op2

    # ---- large config (rank 0, N = 1): the regime of the north-star targets
    #      (large-front Schur updates on FP64 tensor cores, HBM-bound sweeps)
    large = None
    if rank == 0 and ws == 1 and args.large:
        PL = rq.baseline_config(args.large)
        oL = rq.nested_dissection_order(PL)
        stL = oL.stats
        opL = rq.build_operator(PL, SIGMA, oL)

        def time_large(what, iters, param=0):
            ms = C.c_double()
            _lib.check(_lib.lib.rq_operator_time(opL._h, what, iters, param, C.byref(ms)))
            return ms.value
        time_large(5 | 0x100, 2)
        f_ms = time_large(5 | 0x100, 3)
        s_ms = time_large(1 | 0x100, 5)
        sp_ms = time_large(2 | 0x100, 10)
        kL = 2 * NEV.get(args.large, 100) + 1
        gt_ms = time_large(3 | 0x100, 5, kL)
        gn_ms = time_large(4 | 0x100, 5, kL)
        gf_l = stL["flops_lu"] / (f_ms * 1e6)
        sb = stL["trisolve_bytes"]
        spb = 20.0 * PL.nnz + 8.0 * (PL.n + 1) + 24.0 * PL.n
        gb = 8.0 * 2 * PL.n * kL
        large = {
            "workload": args.large, "n": PL.n, "nnz": PL.nnz, "flops_lu": stL["flops_lu"],
            "max_front": int(stL["max_front"]),
            "factor": {"ms": round(f_ms, 3), "gflops": round(gf_l, 1),
                       "frac_fp64": round(gf_l / 1e3 / FP64_PEAK_TFLOPS, 4)},
            "trisolve": {"ms": round(s_ms, 4), "gbs": round(sb / (s_ms * 1e6), 1),
                         "frac_hbm": round(sb / (s_ms * 1e6) / hbm, 4)},
            "spmv_fused_cm": {"ms": round(sp_ms, 4), "gbs": round(spb / (sp_ms * 1e6), 1),
                              "frac_hbm": round(spb / (sp_ms * 1e6) / hbm, 4)},
            "cgs_gemv_t": {"k": kL, "ms": round(gt_ms, 4), "gbs": round(gb / (gt_ms * 1e6), 1),
                           "frac_hbm": round(gb / (gt_ms * 1e6) / hbm, 4)},
            "cgs_gemv_n": {"k": kL, "ms": round(gn_ms, 4), "gbs": round(gb / (gn_ms * 1e6), 1),
                           "frac_hbm": round(gb / (gn_ms * 1e6) / hbm, 4)},
            "l2": "scrubbed (256 MiB) before every timed call",
        }
        del opL
        # the large-front Schur update alone (north-star FP64 tensor target):
        # the factorization's own UPDCB code over every contribution-block tile
        # of the largest front, on a throwaway factorization (it overwrites
        # that front's contribution block)
        try:
            fL = rq.lu_factorize((PL.rowptr, PL.col, PL.q_values(SIGMA)), oL)
            ub = np.zeros(6)
            _lib.check(_lib.lib.rq_factor_bench_updcb(fL._h, -1, 5, ub))
            tf = ub[1] / (ub[0] * 1e9)
            large["schur_update_top_front"] = {
                "kernel": "updcb (factor_dag UPDCB task code, plain grid)", "front": int(ub[2]), "K": int(ub[4]),
                "tiles": int(ub[3]), "ms": round(ub[0], 4), "tflops": round(tf, 2),
                "frac_fp64": round(tf / FP64_PEAK_TFLOPS, 4)}
            del fL
        except Exception as e:  # noqa: BLE001
            large["schur_update_top_front"] = {"error": str(e)[:200]}

    # ---- CPU baseline (rank 0, N = 1 only): bounded oracle factorization sample
    cpu = None
    if rank == 0 and ws == 1 and args.cpu_sample_s > 0:
        import oracle
        kind = "reference" if oracle.ref() is not None else "port"
        ts = cpu_factor_sample(P, kind, args.cpu_sample_s)
        cpu = {"value": round(flu / (sum(ts) / len(ts)) / 1e9, 4), "unit": "GFLOP/s", "cores": 1,
               "kind": kind, "sample": f"{len(ts)} full factorizations of {args.config} "
                                       f"({sum(ts):.1f} s, complex cdouble arithmetic: 4x the real work)",
               "host": host_info()}

    # DRAM bytes per launch of the dominant kernel from a committed ncu --set
    # full capture (profiles/ncu_traffic.json, written by tools/ncu_summary.py)
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            kname = {"factor_dag": "factor_dag_kernel"}.get(KINDS[dom], KINDS[dom])
            ent = json.load(open(tpath)).get(args.config, {}).get(kname)
            if ent:
                traffic, traffic_src = ent["dram_bytes_per_launch"], ent["source"]
        except Exception:  # noqa: BLE001
            traffic = None
    bound = "tensor" if KINDS[dom] == "schur_dmma" else ("hbm" if dom in (0, 1) else "tensor")
    if dom in (0, 1):
        ach = work_k[dom] / (ms_k[dom] * 1e6)  # GB/s
        roof = {"bound": "hbm", "achieved": round(ach, 2), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 5), "traffic": traffic}
    else:
        peak = FP64_PEAK_TFLOPS if KINDS[dom] in ("schur_dmma", "factor_dag") else FP64_DFMA_TFLOPS
        ach = work_k[dom] / (ms_k[dom] * 1e9)  # TFLOP/s
        roof = {"bound": bound, "achieved": round(ach, 4), "peak": peak, "unit": "TFLOP/s",
                "frac": round(ach / peak, 5), "traffic": traffic}
    if traffic_src:
        roof["traffic_unit"] = "bytes/launch"
        roof["traffic_source"] = traffic_src
    roof.update({"kernel": KINDS[dom], "launches_per_step": int(cnt_k[dom]),
                 "share_of_step": round(float(ms_k[dom] / ms_k.sum()), 4),
                 "peak_source": "hbm: MEASURED_PEAKS.json; fp64: measured tools/fp64_peak.cu "
                                "(MEASURED_PEAKS.json has no FP64 entry)"})
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic BASELINE assembly; no dataset)",
        "config": {"workload": args.config, "sigma": SIGMA, "nev": nev, "m": m, "n": P.n,
                   "nnz": P.nnz, "flops_lu_real": flu, "nnz_l_stored": st["nnz_l"],
                   "max_front": st["max_front"], "nfronts": st["nfronts"],
                   "parallelism": f"replicas x{ws}", "l2": "flushed (256 MiB scrub) before every timed step"},
        "factor_frac_fp64": round(value / ws / (FP64_PEAK_TFLOPS * 1e3), 5),
        "time_to_nev_ms": round(min(t_nev), 3), "time_to_nev_runs_ms": [round(t, 2) for t in t_nev],
        "eigs_residual_max": resid_max,
        "eigs": {k: info.get(k) for k in ("restarts", "guard_passes", "n_fb", "n_mv", "n_vv",
                                          "launches", "restart_defect")},
        "kernels": {
            "factor_profile_ms": {KINDS[i]: round(float(ms_k[i]), 4) for i in range(7)},
            "trisolve": {"ms": round(t_solve, 5), "gbs": round(solve_bytes / t_solve / 1e6, 1),
                         "frac_hbm": round(solve_bytes / t_solve / 1e6 / hbm, 4)},
            "spmv_fused_cm": {"ms": round(t_spmv, 5), "gbs": round(spmv_bytes / t_spmv / 1e6, 1),
                              "frac_hbm": round(spmv_bytes / t_spmv / 1e6 / hbm, 4)},
            "cgs_gemv_t": {"ms": round(t_gemv, 5), "k": m, "gbs": round(gemv_bytes / t_gemv / 1e6, 1),
                           "frac_hbm": round(gemv_bytes / t_gemv / 1e6 / hbm, 4)},
        },
        "roofline": roof,
        "large_config": large,
        "cpu_baseline": cpu,
        "e2e": {"value": round(ws * flu / (e2e_ms * 1e6), 3), "unit": "GFLOP/s",
                "h2d_bytes_per_step": 8 * P.nnz, "d2h_bytes_per_step": 16,
                "time_to_nev_ms_from_host": round(e2e_nev_ms, 3)},
        "gpu_launches": int(launches * args.steps),
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg2_riga", choices=sorted(NEV))
    ap.add_argument("--nev", type=int, default=0)
    ap.add_argument("--nev-runs", type=int, default=3)
    ap.add_argument("--max-restarts", type=int, default=1000)
    ap.add_argument("--cpu-sample-s", type=float, default=10.0)
    ap.add_argument("--nev-cpu", type=int, default=1)
    ap.add_argument("--large", default="cfg4_riga",
                    help="secondary large config for the large-front / HBM roofline section ('' to skip)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
