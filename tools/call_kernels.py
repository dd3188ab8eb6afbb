"""Warm per-kernel device time of one call per algorithm (graph replay, CUPTI via torch.profiler): the
kernels on a call's critical path, without ncu's cold-cache serialisation.
usage: python tools/call_kernels.py [C2|C3|C4|C5] [alg_v ...]   (e.g. C5 subspace_v2 krylov_v4)"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import synth as S
from paper_1804_07531_b200 import rsvd

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = S.CONFIGS[name]
ctx = rsvd.Context(0)
A = torch.from_numpy(S.make_matrix(cfg)).cuda() if name in ("C1", "C2", "C3") else S.make_matrix_torch(cfg, torch.device("cuda", 0))
m, n = A.shape
Om = S.gaussian_test_matrix_torch(n, cfg.l, cfg, S.ROLE_OMEGA, torch.device("cuda", 0))
Ph = S.gaussian_test_matrix_torch(m, cfg.l2, cfg, S.ROLE_PHI, torch.device("cuda", 0))
wanted = sys.argv[2:] or ["subspace_v3", "krylov_v4", "single_pass_v1"]
calls = {}
for nm in wanted:
    alg, v = nm.rsplit("_v", 1)
    v = int(v)
    if alg == "subspace":
        calls[nm] = (lambda v=v: ctx.subspace(A, cfg.k, cfg.p, v, Om))
    elif alg == "krylov":
        calls[nm] = (lambda v=v: ctx.block_krylov(A, cfg.k, cfg.p, v, Om))
    elif alg == "krylov_rows":
        calls[nm] = (lambda v=v: ctx.block_krylov_rows(A, cfg.k, cfg.p, v, Om))
    else:
        calls[nm] = (lambda: ctx.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Ph))
REPS = 5 if name in ("C1", "C2", "C3") else 2
for cname, fn in calls.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(REPS):
            fn()
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    first = last = None
    for ev in prof.events():
        if ev.device_type != torch.autograd.DeviceType.CUDA:
            continue
        k = ev.name.replace("(anonymous namespace)::", "").replace("rsvd::", "").replace("void ", "").split("(")[0]
        agg[k][0] += 1
        agg[k][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        t0, t1 = ev.time_range.start, ev.time_range.end
        first = t0 if first is None else min(first, t0)
        last = t1 if last is None else max(last, t1)
    tot = sum(v[1] for v in agg.values())
    print(f"== {name} {cname}: kernel time {tot / REPS:.1f} us per call, span {(last - first) / REPS:.1f} us per call")
    for k, (cnt, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"   {k[:60]:60s} {cnt // REPS:3d}x  {us / REPS:8.1f} us  {100 * us / tot:5.1f}%")
