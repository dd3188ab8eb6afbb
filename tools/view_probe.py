"""Time the view kernels alone (rsvd_view primitive, RSVD_PROFILE events) at several shapes/widths."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1804_07531_b200 import rsvd
ctx = rsvd.Context(0)
peak = 37.1
out = []
shapes = [(4000, 4000), (20000, 8000), (50000, 40000)]
for (m, n) in shapes:
    A = torch.randn(m, n, dtype=torch.float64, device="cuda")
    for w in (20, 30, 64, 70, 120, 128):
        for trans in (0, 1):
            X = torch.randn(w, n if trans == 0 else m, dtype=torch.float64, device="cuda").t()
            for _ in range(2):
                Y, info = ctx.view(A, X, trans=bool(trans), flags=rsvd.RSVD_PROFILE)
            ms = []
            for _ in range(5):
                Y, info = ctx.view(A, X, trans=bool(trans), flags=rsvd.RSVD_PROFILE)
                ms.append(info.view_ms)
            t = min(ms)
            tf = 2.0 * m * n * w / (t * 1e-3) / 1e12
            out.append(dict(m=m, n=n, w=w, trans=trans, ms=t, tflops=tf, frac=tf / peak, gbs=m * n * 8 / (t * 1e-3) / 1e9))
            print(json.dumps(out[-1]), flush=True)
    del A
    torch.cuda.empty_cache()
