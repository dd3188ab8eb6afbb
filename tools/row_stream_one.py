"""One call (after one warm-up) of rsvd_row_stream or rsvd_subspace(v=2) at a config, for ncu."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth as S
from paper_1804_07531_b200 import rsvd
name, alg = sys.argv[1], sys.argv[2]
cfg = S.CONFIGS[name]
dev = torch.device("cuda", 0)
A = S.make_matrix_torch(cfg, dev)
Om = S.gaussian_test_matrix_torch(cfg.n, cfg.l, cfg, S.ROLE_OMEGA, dev)
ctx = rsvd.Context(0)
for _ in range(2):
    (ctx.row_stream(A, cfg.k, cfg.p, Om) if alg == "row" else ctx.subspace(A, cfg.k, cfg.p, 2, Om))
    torch.cuda.synchronize()
