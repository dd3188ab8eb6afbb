"""Sweeps and time of the core Jacobi inside the C2 calls (info.jacobi_sweeps of the last core SVD),
plus the standalone core_svd timing at w = 30 / 60 on synthetic graded cores."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_1804_07531_b200 import rsvd
import synth as S

ctx = rsvd.Context(0)
cfg = S.CONFIGS["C2"]
A = torch.from_numpy(S.make_matrix(cfg)).cuda()
Om = torch.from_numpy(np.ascontiguousarray(S.gaussian_test_matrix(A.shape[1], cfg.l, cfg, S.ROLE_OMEGA).T)).cuda().t()
for name, fn in (("subspace3", lambda: ctx.subspace(A, cfg.k, cfg.p, 3, Om)),
                 ("krylov4", lambda: ctx.block_krylov(A, cfg.k, cfg.p, 4, Om))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); U, s, V, info = fn(); e1.record(); torch.cuda.synchronize()
    print(json.dumps(dict(call=name, ms=e0.elapsed_time(e1), core_sweeps=info.jacobi_sweeps)), flush=True)
