"""One C2 block Krylov v = 4 and one C2 single pass through the library (two calls each: capture +
replay), no profiler attached: the target of the round-2 ncu captures of the latency kernels.
usage: python tools/c2_calls.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import synth as S
from paper_1804_07531_b200 import rsvd

cfg = S.CONFIGS["C2"]
dev = torch.device("cuda", 0)
ctx = rsvd.Context(0)
A = S.make_matrix_torch(cfg, dev)
m, n = A.shape
Om = S.gaussian_test_matrix_torch(n, cfg.l, cfg, S.ROLE_OMEGA, dev)
Ph = S.gaussian_test_matrix_torch(m, cfg.l2, cfg, S.ROLE_PHI, dev)
for _ in range(2):
    ctx.block_krylov(A, cfg.k, cfg.p, 4, Om)
    ctx.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Ph)
torch.cuda.synchronize()
print("ok")
