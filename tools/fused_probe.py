"""Time the one-read single pass (k_view_fused_cl) against the two-view path on C4-shaped A:
python tools/fused_probe.py [m n]  (RSVD_PROFILE view time and the whole call)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth as S  # noqa: E402
from paper_1804_07531_b200 import build, rsvd  # noqa: E402

build.build()
cfg = S.CONFIGS["C4"]
m = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.m
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
dev = torch.device("cuda", 0)
A = S.make_matrix_torch(cfg, dev, m, n) if (m, n) != (cfg.m, cfg.n) else S.make_matrix_torch(cfg, dev)
Om = S.gaussian_test_matrix_torch(n, cfg.l, cfg, S.ROLE_OMEGA, dev)
Phi = S.gaussian_test_matrix_torch(m, cfg.l2, cfg, S.ROLE_PHI, dev)
ctx = rsvd.Context(0)
for rep, fl in ((0, rsvd.RSVD_ONE_READ), (1, rsvd.RSVD_ONE_READ), (2, 0), (3, 0)):
    U, s, V, info = ctx.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Phi, flags=rsvd.RSVD_PROFILE | fl)
    tf = 2.0 * m * n * (cfg.l + cfg.l2) / (info.view_ms * 1e-3) / 1e12
    print(f"{m}x{n} single pass: view launches {info.view_launches}, view {info.view_ms:.2f} ms ({tf:.1f} TF/s), "
          f"call {info.total_ms:.2f} ms", flush=True)
