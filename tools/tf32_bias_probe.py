"""Accumulation bias of the tcgen05 3xTF32 views vs an fp64 reference (the chunk length is
view_tf32.cu's kTf32Chunk; round-2 measurements of 1e6 / 1024 / 256 / 64 are in DESIGN §6.2).
    python tools/tf32_bias_probe.py
Reports ||Y||/||Y_ref|| - 1 (the systematic shrink) and the max relative column error, and the
view time (RSVD_PROFILE), for A x X and A^T x Y on a C5-shaped fp32 A (20000 x 100000, w = 250)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07531_b200 import build, rsvd  # noqa: E402

build.build()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(7)
m, n, w = int(os.environ.get("M", 20000)), 100000, 250
A = torch.randn(m, n, generator=g, device=dev, dtype=torch.float32)
ctx = rsvd.Context(0)
for trans in (0, 1):
    X = torch.randn(w, m if trans else n, generator=g, device=dev, dtype=torch.float32).t()
    Y, info = ctx.view(A, X, trans=bool(trans), flags=rsvd.RSVD_PROFILE)
    Yr = (A.double().t() @ X.double()) if trans else (A.double() @ X.double())
    Yg = Y.double()
    shrink = (Yg.norm() / Yr.norm() - 1).item()
    colerr = ((Yg - Yr).norm(dim=0) / Yr.norm(dim=0)).max().item()
    bias = ((Yg - Yr) * Yr.sign()).mean().item() / Yr.abs().mean().item()
    print(f"{'ATY' if trans else 'AX'} shrink={shrink:.3e} "
          f"bias={bias:.3e} max_col_rel_err={colerr:.3e} view_ms={info.view_ms:.3f}", flush=True)
    del Yr, Yg
