"""Projected strong scaling of the row-sharded path from measured 1-GPU phase times.

For each call: T_1 = measured call time (graph replay, CUDA events); its kernels are timed with
CUPTI (torch.profiler) and classified:
  V     : the A-view kernels (the library's own RSVD_PROFILE view time), / N;
  repl  : the w x w work every rank repeats (core Jacobi, Cholesky / triangular inverse, MinVar,
          small products) plus the launch gaps (T_1 minus the summed kernel time);
  tall  : everything else, including the view kernels that run the Grams / applies of wide
          tall-skinny blocks (profiled k_view_* time minus V), slot sums, copies; split by the side-M
          share of the rows.  Alg. 2 / 9 shard BOTH sides (side M by A's row shards, side N by
          32-aligned row chunks, Exec::plan_shard_n): all of it / N.  The single pass keeps side N
          replicated: side-M share / N, side-N share replicated.
    T_N = V / N + tall / N + repl + comm(N)                     (Alg. 2 / 9)
    T_N = V / N + tall_M / N + tall_N + repl + comm(N)          (single pass)
comm(N)  : Alg. 2 / 9: per co-range view a reduce-scatter of the n x w partial, per range view after
           the first an all-gather of the n x w basis, the final all-gather of V (n x k), plus the
           chunk / unchunk copies of those blocks at HBM speed; single pass: the all-reduce of
           Y_r (n x l2).  Every w x w Gram is all-reduced (latency only).  Bytes moved:
           (N-1)/N per reduce-scatter / all-gather, 2 (N-1)/N per all-reduce, at 725 GB/s (measured
           8-rank NVLink bus bandwidth, B200_PROFILING.md) + 25 us latency each.
Usage: python tools/scaling_projection.py > profiles/scaling_projection_r02.md"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth as S  # noqa: E402
from paper_1804_07531_b200 import build, rsvd  # noqa: E402

BUS = 725e9
HBM = 6.0e12
LAT = 25e-6
build.build()
dev = torch.device("cuda", 0)
ctx = rsvd.Context(0)
rows_out = []


def measure(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


REPL = ("k_jacobi", "k_chol", "k_minvar", "k_small_gemm", "k_diag", "k_tri_inv", "k_pinv_svd", "k_nys",
        "k_symmetrize", "k_mask_cols", "k_square")


def kernel_split(fn, reps=2):
    """(view_s, repl_s, tall_s) kernel time per call"""
    from torch.profiler import ProfilerActivity, profile
    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    v = r = t = 0.0
    for ev in prof.events():
        if ev.device_type != torch.autograd.DeviceType.CUDA:
            continue
        us = ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        nm = ev.name.replace("(anonymous namespace)::", "").replace("rsvd::", "").replace("void ", "")
        if "k_view" in nm:
            v += us
        elif any(k in nm for k in REPL):
            r += us
        else:
            t += us
    return v * 1e-6 / reps, r * 1e-6 / reps, t * 1e-6 / reps


for name, runs in (("C4", [("krylov", 3, 0), ("single_pass", 1, 0), ("subspace", 3, 1)]),
                   ("C5", [("subspace", 2, 0), ("subspace", 3, 0), ("krylov", 4, 0)])):
    cfg = S.CONFIGS[name]
    A = S.make_matrix_torch(cfg, dev)
    Om = S.gaussian_test_matrix_torch(cfg.n, cfg.l, cfg, S.ROLE_OMEGA, dev)
    Omm = S.gaussian_test_matrix_torch(cfg.m, cfg.l, cfg, S.ROLE_OMEGA_M, dev)
    Phi = S.gaussian_test_matrix_torch(cfg.m, cfg.l2, cfg, S.ROLE_PHI, dev)
    esz = cfg.itemsize
    for alg, v, inp in runs:
        def call(flags=0):
            if alg == "subspace":
                return ctx.subspace(A, cfg.k, cfg.p, v, Omm if inp else Om, input=inp, flags=flags)
            if alg == "krylov":
                return ctx.block_krylov(A, cfg.k, cfg.p, v, Om, flags=flags)
            return ctx.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Phi, flags=flags)
        t1 = measure(call) * 1e-3
        Vall, repl, tall = kernel_split(call)
        V = call(rsvd.RSVD_PROFILE)[3].view_ms * 1e-3      # the A views alone
        tall += max(Vall - V, 0.0)                           # view kernels on tall-skinny blocks
        gaps = max(t1 - (V + repl + tall), 0.0)              # launch gaps: replicated
        rest = max(t1 - V, 0.0)
        l = cfg.l
        W = l * ((v // 2) if (alg == "krylov" and v % 2 == 0) else ((v - 1) // 2 if alg == "krylov" else 1))
        # co-range views (partials all-reduced): input A -> even views; sizes n x width
        n_co = v // 2 if not inp else (v + 1) // 2
        co_bytes = n_co * cfg.n * max(l, W) * 8 if alg != "single_pass" else cfg.n * cfg.l2 * 8
        n_gram = 3 * v + 4
        # side-M share of the tall-skinny work (Grams, applies of the m-side blocks)
        m_side = (cfg.m if not inp else cfg.n)
        n_side = (cfg.n if not inp else cfg.m)
        frac_m = m_side / (m_side + n_side) if alg == "single_pass" else 1.0
        width = max(l, W)
        n_ax = (v + 1) // 2 if not inp else v // 2          # range views (X all-gathered after the first)
        row = {"cfg": name, "call": f"{alg} v={v}" + (" input=A^T" if inp else ""), "T1_ms": t1 * 1e3,
               "views_ms": V * 1e3, "rest_ms": rest * 1e3, "repl_ms": (repl + gaps) * 1e3, "tall_ms": tall * 1e3}
        for N in (1, 2, 4, 8):
            if N == 1:
                comm = 0.0
            elif alg == "single_pass":
                comm = 2 * (N - 1) / N * co_bytes / BUS + (1 + n_gram) * LAT
            else:
                nb = cfg.n * width * 8                          # one side-N block
                moved = n_co * nb + max(n_ax - (0 if inp else 1), 0) * nb + cfg.n * cfg.k * 8
                n_coll = n_co + max(n_ax - (0 if inp else 1), 0) + 1
                comm = (N - 1) / N * moved / BUS + (n_coll + n_gram) * LAT + 2 * 2 * moved / HBM
            tN = (V / N + tall * frac_m / N + tall * (1 - frac_m) + repl + gaps + comm) if N > 1 else t1
            row[f"T{N}_ms"] = tN * 1e3
            row[f"x{N}"] = t1 / tN
        rows_out.append(row)
        print(row, file=sys.stderr, flush=True)
    del A
    torch.cuda.empty_cache()

print("| config | call | 1-GPU ms | views ms | replicated ms | tall-skinny ms | 2 GPUs | 4 GPUs | 8 GPUs |")
print("|---|---|---|---|---|---|---|---|---|")
for r in rows_out:
    print(f"| {r['cfg']} | {r['call']} | {r['T1_ms']:.1f} | {r['views_ms']:.1f} | {r['repl_ms']:.1f} | {r['tall_ms']:.1f} | "
          f"{r['T2_ms']:.1f} ({r['x2']:.2f}x) | {r['T4_ms']:.1f} ({r['x4']:.2f}x) | {r['T8_ms']:.1f} ({r['x8']:.2f}x) |")
