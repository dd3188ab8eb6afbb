"""Median view-kernel time (rsvd_view primitive, RSVD_PROFILE events) over a width sweep at C2's 4000^2 and
C3's 20000 x 8000, A*X and A^T*Y; one JSON line (us).  Used for A/B builds of the view kernels."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1804_07531_b200 import rsvd
ctx = rsvd.Context(0)
res = {}
for (m, n, ws) in ((4000, 4000, (30, 60, 90, 120)), (20000, 8000, (70, 140))):
    A = torch.randn(m, n, dtype=torch.float64, device="cuda")
    for w in ws:
        for trans in (0, 1):
            X = torch.randn(w, n if trans == 0 else m, dtype=torch.float64, device="cuda").t()
            ms = []
            for _ in range(10):
                Y, info = ctx.view(A, X, trans=bool(trans), flags=rsvd.RSVD_PROFILE)
                ms.append(info.view_ms)
            res[f"{m}:{'aty' if trans else 'ax'}{w}"] = round(sorted(ms[2:])[len(ms[2:]) // 2] * 1000, 1)
    del A
print(json.dumps(res))
