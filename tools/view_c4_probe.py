"""The C4 views alone (80 GB fp64 A, w = 120): A X and A^T Y once each (RSVD_PROFILE), for ncu
launch lists / DRAM counters.  python tools/view_c4_probe.py [rows]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth as S  # noqa: E402
from paper_1804_07531_b200 import build, rsvd  # noqa: E402

build.build()
cfg = S.CONFIGS["C4"]
m = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.m
dev = torch.device("cuda", 0)
A = S.make_matrix_torch(cfg, dev, row0=0, rows=m) if m != cfg.m else S.make_matrix_torch(cfg, dev)
X = S.gaussian_test_matrix_torch(cfg.n, cfg.l, cfg, S.ROLE_OMEGA, dev)
Y = S.gaussian_test_matrix_torch(m, cfg.l, cfg, S.ROLE_OMEGA_M, dev)
ctx = rsvd.Context(0)
for trans, Z in ((0, X), (1, Y)):
    _, info = ctx.view(A, Z, trans=bool(trans), flags=rsvd.RSVD_PROFILE)
    tf = 2.0 * m * cfg.n * cfg.l / (info.view_ms * 1e-3) / 1e12
    print(f"{'A^T Y' if trans else 'A X'} {m}x{cfg.n} w={cfg.l}: {info.view_ms:.3f} ms, {tf:.2f} TF/s, "
          f"algorithmic bytes {m * cfg.n * 8 / 1e9:.2f} GB", flush=True)
