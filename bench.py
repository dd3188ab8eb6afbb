#!/usr/bin/env python
"""Benchmark of the pass-efficient randomized SVD hot path on B200 (BASELINE.json metric
"A-view HBM GB/s (fraction of roofline) and rank-k SVD time per view budget").

A STEP is one pass of the whole hot path over one synthetic matrix.
Default workload (N = 1): BASELINE C4, the largest single-GPU config — fp64 50000 x 200000 (80 GB),
X diag(i^-1.5) Y^T (rank 500) + 1e-8 G, k = 100, p = 20 — with BASELINE C4's three runs:
    rsvd_block_krylov v = 3                            (3 views, Alg. 9 == Alg. 2 at v = 3)
    rsvd_single_pass l2 = 240                          (1 view, Alg. 7)
    rsvd_subspace v = 3, input = A^T, RSVD_SQUARED     (3 views, the A^T A normal-matrix estimate)
= 7 views of A per step.  A (80 GB) is far larger than L2 (126 MB): every view streams it from HBM,
no flush is needed (stated in `config`).

value = A bytes of all views of the step / step time (GB/s); the three calls run concurrently on
three contexts / streams (RSVD_ASYNC) at N = 1, sequentially on one communicator at N > 1.
N > 1 (torchrun, one process per GPU): the SAME matrix row-sharded over the N GPUs
(shard_rows, 128-row aligned; strong scaling), NCCL all-reduce of the A^T Y partials and Grams.

Secondary records: C5 (fp32 100000^2, 40 GB; tcgen05 3xTF32 views) SVD times and view fractions
(3xTF32 and strict 1x-flop), and the C2 per-call latencies.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C4|C5|C2|C3]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth as S  # noqa: E402

METRIC = "A-view HBM GB/s (fraction of roofline) and rank-k SVD time per view budget"
SQUARED = 1
# (algorithm, views, input (0 = A, 1 = A^T), flags) per config
PLANS = {
    "C4": [("krylov", 3, 0, 0), ("single_pass", 1, 0, 0), ("subspace", 3, 1, SQUARED)],
    "C5": [("subspace", 2, 0, 0), ("krylov", 4, 0, 0)],
    "C3": [("subspace", 3, 0, 0), ("krylov", 4, 0, 0), ("single_pass", 1, 0, 0)],
    "C2": [("subspace", 3, 0, 0), ("krylov", 4, 0, 0), ("single_pass", 1, 0, 0)],
}
DMMA_NOMINAL_TF, BF16_NOMINAL_TF, TF32_NOMINAL_TF = 40.0, 2250.0, 1100.0


def plan_views(plan):
    return sum(v for _, v, _, _ in plan)


def plan_name(plan):
    return " + ".join(f"{a} v={v}" + (" input=A^T" if i else "") + (" S^2" if f & SQUARED else "") for a, v, i, f in plan)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--sequential", action="store_true", help="N = 1: run the step's calls one after another")
    return ap.parse_args()


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(path)) if os.path.exists(path) else {}


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU oracle (cpu_baseline / reference arm)
def oracle_step(A, cfg, plan, Om, Omm, Phi):
    import oracle as O

    for alg, v, inp, _ in plan:
        O.svd_of(A, alg, cfg.k, cfg.p, v=v, Omega=Omm if inp else Om, l2=cfg.l2, Phi=Phi, transpose=bool(inp))


def oracle_sample_inputs(cfg, rows):
    """The config's recipe at a bounded row sample (rows x n), NumPy generator (host only)."""
    A = S.make_matrix(cfg, rows, cfg.n).astype(np.float64)
    Om = S.gaussian_test_matrix(cfg.n, cfg.l, cfg, S.ROLE_OMEGA).astype(np.float64)
    Omm = S.gaussian_test_matrix(rows, cfg.l, cfg, S.ROLE_OMEGA_M).astype(np.float64)
    Phi = S.gaussian_test_matrix(rows, cfg.l2, cfg, S.ROLE_PHI).astype(np.float64)
    return A, Om, Omm, Phi


SAMPLE_ROWS = {"C4": 12000, "C5": 8000, "C3": 20000, "C2": 4000}


def time_oracle(A, cfg, plan, Om, Omm, Phi, steps, warmup, budget_s):
    for _ in range(max(0, warmup)):
        oracle_step(A, cfg, plan, Om, Omm, Phi)
    ts = []
    t_all = time.perf_counter()
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        oracle_step(A, cfg, plan, Om, Omm, Phi)
        ts.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > budget_s:
            break
    step_s = statistics.median(ts)
    gbs = plan_views(plan) * A.shape[0] * A.shape[1] * cfg.itemsize / step_s / 1e9
    cores = len(os.sched_getaffinity(0))
    sample = (f"{len(ts)} oracle step(s) ({plan_name(plan)}) on a {A.shape[0]} x {A.shape[1]} row sample of "
              f"{cfg.name}'s recipe (the full matrix is {cfg.m} x {cfg.n}); NumPy/OpenBLAS fp64 on {cores} cores, "
              f"median step {step_s:.3f} s; value = A-view bytes of the sample / step time")
    return {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample, "step_s": step_s,
            "steps_done": len(ts)}


def reference_main(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cfg = S.CONFIGS[args.config]
    plan = PLANS[args.config]
    rows = SAMPLE_ROWS.get(cfg.name, cfg.m)
    A, Om, Omm, Phi = oracle_sample_inputs(cfg, rows)
    steps = max(1, min(args.steps, 3))
    warm = max(1, min(args.warmup, 3))
    base = time_oracle(A, cfg, plan, Om, Omm, Phi, steps, warm, budget_s=120.0)
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": "GB/s", "n_gpus": args.gpus,
            "steps": base["steps_done"], "warmup": warm, "ms_per_step": base["step_s"] * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name} ({cfg.m}x{cfg.n} {cfg.dtype}, k={cfg.k}, p={cfg.p}, l2={cfg.l2}); "
                                   f"step = {plan_name(plan)}; bounded row sample {rows} x {cfg.n}"},
            "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": base["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def call(ctx, alg, v, inp, fl, A, Om, Omm, Phi, cfg, m, row0, host_out=False):
    if alg == "subspace":
        return ctx.subspace(A, cfg.k, cfg.p, v, Omm if inp else Om, input=inp, flags=fl, m=m, row0=row0,
                            host_out=host_out)
    if alg == "krylov":
        return ctx.block_krylov(A, cfg.k, cfg.p, v, Omm if inp else Om, input=inp, flags=fl, m=m, row0=row0,
                                host_out=host_out)
    return ctx.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Phi, flags=fl, m=m, row0=row0, host_out=host_out)


def view_roofline(infos_per_call, peak_tf, alt_peak_tf, dtype):
    """Dominant kernels = the view kernels: algorithmic flops per launch / average launch duration
    (CUDA events on the ctx stream around every view launch, RSVD_PROFILE)."""
    vms = sum(i.view_ms for i in infos_per_call)
    vfl = sum(i.view_flops for i in infos_per_call)
    vby = sum(i.view_bytes for i in infos_per_call)
    n = sum(i.view_launches for i in infos_per_call)
    tot = sum(i.total_ms for i in infos_per_call)
    mult = 3.0 if dtype == "f32" else 1.0       # 3xTF32 executes three tensor products per flop
    ach = mult * vfl / (vms * 1e-3) / 1e12 if vms > 0 else None
    out = {"bound": "tensor", "achieved": ach, "peak": peak_tf, "unit": "TFLOP/s",
           "frac": ach / peak_tf if ach and peak_tf else None,
           "view_launches": n, "avg_view_ms": vms / max(n, 1),
           "flops_per_launch": vfl / max(n, 1), "bytes_per_launch": vby / max(n, 1),
           "hbm_gbs_during_views": vby / (vms * 1e-3) / 1e9 if vms > 0 else None,
           "view_share_of_calls": vms / tot if tot > 0 else None}
    if alt_peak_tf:
        out["peak_alt"] = alt_peak_tf
        out["frac_alt"] = ach / alt_peak_tf if ach else None
    if dtype == "f32" and ach:
        out["achieved_1x_flops"] = ach / 3.0
        out["frac_strict_1x"] = ach / 3.0 / peak_tf if peak_tf else None
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return reference_main(args)

    import torch
    import torch.distributed as dist

    from paper_1804_07531_b200 import rsvd
    from paper_1804_07531_b200.sharding import broadcast_uid, max_over_ranks as _mor, shard_rows

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=dev)
    cfg = S.CONFIGS[args.config]
    plan = PLANS[args.config]
    esz = cfg.itemsize
    peaks_file = measured_peaks()

    # ---- inputs: the whole matrix, row-sharded over the ranks (strong scaling, 128-row aligned)
    m, n = cfg.m, cfg.n
    sh = shard_rows(m, world, rank, align=128)
    A = S.make_matrix_torch(cfg, dev, row0=sh.row0, rows=sh.m_local)
    Om = S.gaussian_test_matrix_torch(n, cfg.l, cfg, S.ROLE_OMEGA, dev)                       # replicated
    Omm_full = S.gaussian_test_matrix_torch(m, cfg.l, cfg, S.ROLE_OMEGA_M, dev)
    Omm = Omm_full[sh.row0:sh.row0 + sh.m_local]                                            # A^T input: shard
    Phi_full = S.gaussian_test_matrix_torch(m, cfg.l2, cfg, S.ROLE_PHI, dev)
    Phi = Phi_full[sh.row0:sh.row0 + sh.m_local]
    torch.cuda.synchronize(dev)

    concurrent = world == 1 and not args.sequential
    if concurrent:
        streams = [torch.cuda.current_stream(dev)] + [torch.cuda.Stream(dev) for _ in plan[1:]]
    else:
        streams = [torch.cuda.current_stream(dev)]
    ctxs = [rsvd.Context(local, stream=s_) for s_ in streams]
    ctx = ctxs[0]
    if world > 1:
        uid = broadcast_uid(rsvd.get_unique_id() if rank == 0 else None, rank)
        ctx.comm_init(world, rank, uid)             # ONE communicator per rank; calls in a fixed order

    def step(flags=0):
        cur = torch.cuda.current_stream(dev)
        infos = []
        conc = concurrent and not (flags & rsvd.RSVD_PROFILE)
        for i, (alg, v, inp, fl) in enumerate(plan):
            c = ctxs[i] if conc else ctx
            s_ = streams[i] if conc else cur
            if conc and s_ != cur:
                s_.wait_stream(cur)
            r = call(c, alg, v, inp, fl | flags | (rsvd.RSVD_ASYNC if conc else 0), A, Om, Omm, Phi, cfg, m, sh.row0)
            infos.append(r[3])
        if conc:
            for c, s_, inf in zip(ctxs, streams, infos):
                c.wait(inf)
                if s_ != cur:
                    cur.wait_stream(s_)
        return infos

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        return _mor(x, device=dev)

    stream = torch.cuda.current_stream(dev)
    for _ in range(max(3, args.warmup)):
        step()
    barrier()

    # ---- timed region: CUDA events on the launching stream, A >> L2 (no flush needed)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        t_busy = time.perf_counter()
        while time.perf_counter() - t_busy < 0.5:        # samples start under load
            step()
            torch.cuda.synchronize(dev)
        barrier()
        for i in range(args.steps):
            evs[i][0].record(stream)
            infos = step()
            evs[i][1].record(stream)
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = max_over_ranks(sum(step_ms))
    ms_per_step = total_ms / args.steps
    a_bytes = m * n * esz                                   # the whole matrix (all ranks)
    bytes_step = plan_views(plan) * a_bytes
    value = bytes_step * args.steps / (total_ms * 1e-3) / 1e9
    launches_per_step = sum(inf.kernel_launches for inf in infos)

    # ---- per-call SVD time (sequential, graph replay, device events)
    svd_ms = {}
    for alg, v, inp, fl in plan:
        ts = []
        for _ in range(3):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            call(ctx, alg, v, inp, fl, A, Om, Omm, Phi, cfg, m, sh.row0)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ts.append(e0.elapsed_time(e1))
        key = f"{alg}_v{v}" + ("_AT" if inp else "") + ("_sq" if fl & SQUARED else "")
        svd_ms[key] = max_over_ranks(statistics.median(ts))
    # ---- view-kernel durations (RSVD_PROFILE: events around every view kernel on the ctx stream)
    prof = []
    for _ in range(args.profile_steps):
        barrier()
        prof += step(flags=rsvd.RSVD_PROFILE)
    try:
        t_dmma, g_read = ctx.probe_peaks()
        probed = {"dmma_fp64_tflops": t_dmma, "hbm_read_gbs": g_read}
    except Exception as e:  # pragma: no cover
        probed = {"error": str(e)}
    bf16 = peaks_file.get("bf16_tflops")
    if cfg.dtype == "f64":
        peak = probed.get("dmma_fp64_tflops")
        alt = bf16 * DMMA_NOMINAL_TF / BF16_NOMINAL_TF if bf16 else None
        roof = view_roofline(prof, peak, alt, "f64")
        roof["kernel"] = "view kernels k_view_ax / k_view_aty / k_view_fused (FP64 DMMA m8n8k4, TMA-fed)"
        roof["peak_source"] = ("FP64 DMMA throughput measured on this GPU by rsvd_probe_peaks (mma.sync m8n8k4, "
                               "all SMs); peak_alt = MEASURED_PEAKS bf16 burst x nominal fp64/bf16 40/2250")
    else:
        peak = bf16 * TF32_NOMINAL_TF / BF16_NOMINAL_TF if bf16 else None
        roof = view_roofline(prof, peak, None, "f32")
        roof["kernel"] = "k_view_tf32 (tcgen05 kind::tf32, 3xTF32, TMEM accumulators)"
        roof["peak_source"] = "MEASURED_PEAKS bf16 burst x nominal tf32/bf16 1100/2250"
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")
    roof["traffic"] = None
    if os.path.exists(tpath):
        try:
            roof["traffic"] = json.load(open(tpath)).get(cfg.name)
            roof["traffic_source"] = "profiles/ncu_traffic_r02.json (ncu dram__bytes_read.sum + write.sum per launch)"
        except Exception:
            pass
    view_roof_ms = {}
    for alg, v, inp, fl in plan:
        vb = v * a_bytes
        key = f"{alg}_v{v}" + ("_AT" if inp else "") + ("_sq" if fl & SQUARED else "")
        w = cfg.l + (cfg.l2 if alg == "single_pass" else 0)
        nvec = (v * cfg.l if alg == "subspace" else (v + v // 2 - 1) * cfg.l if alg == "krylov" else w)
        flops = 2.0 * m * n * nvec * (3.0 if cfg.dtype == "f32" else 1.0)
        t_roof = max(vb / (peaks_file.get("hbm_gbs", 6456.8) * 1e9), flops / ((peak or 1) * 1e12)) * 1e3
        view_roof_ms[key] = {"roofline_ms": t_roof, "frac_of_view_roofline": t_roof / svd_ms[key]}

    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype,
            "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.dtype} {m}x{n} ({a_bytes / 1e9:.0f} GB) "
                                   f"{'X diag(i^-1.5) Y^T rank 500 + 1e-8 G' if cfg.name == 'C4' else cfg.kind}, "
                                   f"k={cfg.k}, p={cfg.p}, l2={cfg.l2}; step = {plan_name(plan)} "
                                   f"({plan_views(plan)} views of A)",
                       "l2_flush": "none needed: A is larger than L2 and every view streams it from HBM",
                       "calls": "concurrent on %d streams (RSVD_ASYNC)" % len(plan) if concurrent else "sequential",
                       "parallelism": (f"A row-sharded over {world} GPUs (128-row aligned), NCCL all-reduce; the "
                                       f"same matrix at every N (strong scaling)") if world > 1 else "1 GPU"},
            "views_per_s": plan_views(plan) * args.steps / (total_ms * 1e-3),
            "svd_ms": svd_ms, "view_roofline_per_call": view_roof_ms, "roofline": roof, "peaks_probed": probed,
            "gpu_launches": launches_per_step * args.steps}

    # ---- CPU oracle on a bounded row sample of the same bytes (rank 0, N = 1)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rows = SAMPLE_ROWS.get(cfg.name, m)
        As = A[:rows].double().cpu().numpy()
        base = time_oracle(As, cfg, plan, Om.double().cpu().numpy(), Omm_full[:rows].double().cpu().numpy(),
                           Phi_full[:rows].double().cpu().numpy(), steps=1, warmup=0, budget_s=30.0)
        line["cpu_baseline"] = {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")}
        del As

    # ---- e2e: the same step through the C ABI with HOST buffers (pinned), copies inside the timed
    # region: every call stages A (and Omega / Phi) host -> device itself and returns U, S, V to host
    for c_ in ctxs[1:]:
        c_.close()
    if not args.no_e2e:
        Ah = torch.empty(A.shape, dtype=A.dtype, pin_memory=True)
        Ah.copy_(A)
        Omh = Om.t().contiguous().cpu().pin_memory().t()
        Ommh = Omm.t().contiguous().cpu().pin_memory().t()
        Phih = Phi.t().contiguous().cpu().pin_memory().t()
        del A, Omm_full, Phi_full
        ctx.close()
        torch.cuda.empty_cache()
        ctx = rsvd.Context(local)
        if world > 1:
            uid = broadcast_uid(rsvd.get_unique_id() if rank == 0 else None, rank)
            ctx.comm_init(world, rank, uid)

        def e2e_step():
            outs = []
            for alg, v, inp, fl in plan:
                outs.append(call(ctx, alg, v, inp, fl, Ah, Omh, Ommh, Phih, cfg, m, sh.row0, host_out=True))
            return outs

        e2e_step()                                       # warm-up (graph capture, workspace)
        barrier()
        K = max(2, args.e2e_steps)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(K):
            outs = e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / K)
        h2d = sum(Ah.numel() * esz + (Ommh if inp else Omh).numel() * esz + (Phih.numel() * esz if alg == "single_pass" else 0)
                  for alg, v, inp, fl in plan)
        d2h = sum(t.numel() * t.element_size() for o in outs for t in o[:3] if t is not None)
        line["e2e"] = {"value": bytes_step / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "steps": K,
                       "how": "the step's calls through the C ABI with pinned HOST A / Omega / Phi and host U, S, V: "
                              "each call stages A (80 GB for C4) host -> device in its own workspace and returns "
                              "U, S, V to host; synchronous calls, CUDA events around K steps; bound by the host "
                              "link (one A transfer per call)"}
        del Ah
    ctx.close()
    torch.cuda.empty_cache()

    if rank == 0 and world == 1 and not args.no_secondary and cfg.name == "C4":
        line["secondary_c5"] = secondary(rsvd, torch, dev, "C5", peaks_file)
        line["secondary_c2"] = secondary(rsvd, torch, dev, "C2", peaks_file, reps=10)
    line["clocks"] = clk.summary()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def secondary(rsvd, torch, dev, name, peaks_file, reps=3):
    """Per-call SVD times of another config (sequential, graph replay, device events) and its view
    kernels' roofline fraction (RSVD_PROFILE)."""
    cfg = S.CONFIGS[name]
    A = S.make_matrix_torch(cfg, dev)
    Om = S.gaussian_test_matrix_torch(cfg.n, cfg.l, cfg, S.ROLE_OMEGA, dev)
    Phi = S.gaussian_test_matrix_torch(cfg.m, cfg.l2, cfg, S.ROLE_PHI, dev)
    torch.cuda.synchronize(dev)
    ctx = rsvd.Context(dev.index)
    runs = {"C5": [("subspace", 2), ("subspace", 3), ("krylov", 3), ("krylov", 4)],
            "C2": [("subspace", 3), ("krylov", 4), ("single_pass", 1)]}[name]
    out = {"workload": f"{name}: {cfg.dtype} {cfg.m}x{cfg.n}, k={cfg.k}, p={cfg.p}", "svd_ms": {}}
    stream = torch.cuda.current_stream(dev)
    prof = []
    bf16 = peaks_file.get("bf16_tflops")
    for alg, v in runs:
        call(ctx, alg, v, 0, 0, A, Om, None, Phi, cfg, cfg.m, 0)
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            call(ctx, alg, v, 0, 0, A, Om, None, Phi, cfg, cfg.m, 0)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ts.append(e0.elapsed_time(e1))
        out["svd_ms"][f"{alg}_v{v}"] = statistics.median(ts)
        prof.append(call(ctx, alg, v, 0, rsvd.RSVD_PROFILE, A, Om, None, Phi, cfg, cfg.m, 0)[3])
    if cfg.dtype == "f32":
        peak = bf16 * TF32_NOMINAL_TF / BF16_NOMINAL_TF if bf16 else None
        out["roofline"] = view_roofline(prof, peak, None, "f32")
        out["roofline"]["peak_source"] = "MEASURED_PEAKS bf16 burst x nominal tf32/bf16 1100/2250"
    else:
        t, _ = ctx.probe_peaks()
        out["roofline"] = view_roofline(prof, t, None, "f64")
    ctx.close()
    del A
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
