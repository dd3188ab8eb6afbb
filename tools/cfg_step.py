"""One call of an algorithm on a full-size config (after one warm-up), for ncu launch lists.
usage: python tools/cfg_step.py C4 krylov 3"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import synth as S
from paper_1804_07531_b200 import rsvd

name, alg, v = sys.argv[1], sys.argv[2], int(sys.argv[3])
cfg = S.CONFIGS[name]
dev = torch.device("cuda", 0)
A = S.make_matrix_torch(cfg, dev, panel_rows=2048)
Om = S.gaussian_test_matrix_torch(cfg.n, cfg.l, cfg, S.ROLE_OMEGA, dev)
Phi = S.gaussian_test_matrix_torch(cfg.m, cfg.l2, cfg, S.ROLE_PHI, dev)
ctx = rsvd.Context(0)
for _ in range(2):
    if alg == "subspace":
        r = ctx.subspace(A, cfg.k, cfg.p, v, Om)
    elif alg == "krylov":
        r = ctx.block_krylov(A, cfg.k, cfg.p, v, Om)
    else:
        r = ctx.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Phi)
    torch.cuda.synchronize()
print("ok", r[3].kernel_launches)
