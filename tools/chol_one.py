"""One CholeskyQR2 of a tall block of width w (k_chol_big for 160 < w <= 512), for ncu:
python tools/chol_one.py [rows] [w]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07531_b200 import build, rsvd  # noqa: E402

build.build()
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
w = int(sys.argv[2]) if len(sys.argv) > 2 else 250
g = torch.Generator(device="cuda")
g.manual_seed(1)
Y = (torch.randn(w, rows, generator=g, device="cuda", dtype=torch.float64) *
     torch.logspace(0, -3, w, device="cuda", dtype=torch.float64)[:, None]).t()
ctx = rsvd.Context(0)
for _ in range(3):
    Q, R, info = ctx.orth(Y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
Q, R, info = ctx.orth(Y)
e1.record()
torch.cuda.synchronize()
print(f"orth {rows}x{w}: {e0.elapsed_time(e1):.3f} ms", flush=True)
