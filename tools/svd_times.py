"""Rank-k SVD time per view budget (the second half of BASELINE.json's metric) for every config
C1..C5 at full size and every algorithm / v listed in synth.CONFIGS[..].runs: device time of one
call (CUDA events, graph replay, median of reps; L2 flushed before each rep), views/s, and the
fraction of the pure view roofline (v views at max(A bytes / HBM, view flops / tensor peak)).
usage: python tools/svd_times.py [C1 C2 ...]  -> JSON lines"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import synth as S
from paper_1804_07531_b200 import rsvd

peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
HBM = peaks["hbm_gbs"] * 1e9
TF32 = peaks["bf16_tflops"] * 1.1 / 2.25 * 1e12
DMMA = 37.1e12
names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
ctx = rsvd.Context(0)
dev = torch.device("cuda", 0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for name in names:
    cfg = S.CONFIGS[name]
    A = S.make_matrix_torch(cfg, dev, panel_rows=2048)
    m, n, l = cfg.m, cfg.n, cfg.l
    es = 4 if cfg.dtype == "f32" else 8
    Om = S.gaussian_test_matrix_torch(n, l, cfg, S.ROLE_OMEGA, dev)
    Phi = S.gaussian_test_matrix_torch(m, cfg.l2, cfg, S.ROLE_PHI, dev)
    reps = 3 if m * n * es > 4e9 else 10
    peak = TF32 / 3 if cfg.dtype == "f32" else DMMA   # 3xTF32: a third of the tf32 rate for useful flops

    def view_floor(width):
        return max(m * n * es / HBM, 2.0 * m * n * width / peak)

    runs = []
    for v in cfg.runs.get("subspace", []):
        runs.append(("subspace", v, lambda v=v: ctx.subspace(A, cfg.k, cfg.p, v, Om), v * view_floor(l)))
    for v in cfg.runs.get("krylov", []):
        nb = v // 2 if v % 2 == 0 else (v - 1) // 2
        floor = (v - 1) * view_floor(l) + view_floor(nb * l)
        runs.append(("krylov", v, lambda v=v: ctx.block_krylov(A, cfg.k, cfg.p, v, Om), floor))
    for v in cfg.runs.get("normal", []):
        # A^T A ~ V diag(S) V^T by Alg. 4 (Nystrom): Omega on the m side for odd v, n side for even v
        Omn = Om if v % 2 == 0 else S.gaussian_test_matrix_torch(m, l, cfg, S.ROLE_OMEGA_M, dev)
        runs.append(("nystrom", v, lambda v=v, Omn=Omn: ctx.nystrom(A, cfg.k, cfg.p, v, Omn), v * view_floor(l)))
    if cfg.runs.get("single_pass"):
        runs.append(("single_pass", 1, lambda: ctx.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Phi),
                     max(m * n * es / HBM, 2.0 * m * n * (l + cfg.l2) / peak)))
    for alg, v, fn, floor in runs:
        ms = timed(fn, reps)
        print(json.dumps({"config": name, "dtype": cfg.dtype, "m": m, "n": n, "k": cfg.k, "p": cfg.p, "alg": alg,
                          "v": v, "svd_ms": ms, "views_per_s": v / (ms * 1e-3),
                          "view_roofline_ms": floor * 1e3, "frac_of_view_roofline": floor * 1e3 / ms}), flush=True)
    del A, Om, Phi
    torch.cuda.empty_cache()
