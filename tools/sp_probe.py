"""Single-pass sketch timing by path on a config (RSVD_PROFILE): default vs RSVD_ONE_READ.
python tools/sp_probe.py C3|C4 [one_read_only]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth as S  # noqa: E402
from paper_1804_07531_b200 import build, rsvd  # noqa: E402

build.build()
cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
only = len(sys.argv) > 2
dev = torch.device("cuda", 0)
A = S.make_matrix_torch(cfg, dev)
Om = S.gaussian_test_matrix_torch(cfg.n, cfg.l, cfg, S.ROLE_OMEGA, dev)
Phi = S.gaussian_test_matrix_torch(cfg.m, cfg.l2, cfg, S.ROLE_PHI, dev)
ctx = rsvd.Context(0)
for fl, nm in ((rsvd.RSVD_ONE_READ, "one-read"),) + (() if only else ((0, "default"),)):
    for rep in range(3):
        U, s, V, info = ctx.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Phi, flags=rsvd.RSVD_PROFILE | fl)
    print(f"{cfg.name} single pass {nm}: view launches {info.view_launches}, views {info.view_ms:.3f} ms, "
          f"call {info.total_ms:.3f} ms", flush=True)
