"""Run W warm-up steps and ONE step of the benchmark hot path (C2) — for ncu launch lists."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth as S
from paper_1804_07531_b200 import rsvd

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
A = S.make_matrix_torch(cfg, dev)
Om = S.gaussian_test_matrix_torch(cfg.n, cfg.l, cfg, S.ROLE_OMEGA, dev)
Phi = S.gaussian_test_matrix_torch(cfg.m, cfg.l2, cfg, S.ROLE_PHI, dev)
ctx = rsvd.Context(0)
torch.cuda.synchronize()
for i in range(warm + 1):
    if i == warm:
        torch.cuda.nvtx.range_push("step")
    ctx.subspace(A, cfg.k, cfg.p, 3, Om)
    ctx.block_krylov(A, cfg.k, cfg.p, 4, Om)
    ctx.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Phi)
    torch.cuda.synchronize()
print("ok")
