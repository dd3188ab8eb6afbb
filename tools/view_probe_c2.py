"""C2-shaped view kernel timing (rsvd_view primitive, RSVD_PROFILE events): ax/aty at w = 30 / 60 and
the fused sketch at l = 30, l2 = 60.  Used for A/B builds."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1804_07531_b200 import rsvd
ctx = rsvd.Context(0)
m = n = 4000
A = torch.randn(m, n, dtype=torch.float64, device="cuda")
res = {}
for w in (30, 60):
    for trans in (0, 1):
        X = torch.randn(w, n if trans == 0 else m, dtype=torch.float64, device="cuda").t()
        ms = []
        for _ in range(12):
            Y, info = ctx.view(A, X, trans=bool(trans), flags=rsvd.RSVD_PROFILE)
            ms.append(info.view_ms)
        res[f"{'aty' if trans else 'ax'}{w}"] = round(sorted(ms[2:])[len(ms[2:]) // 2] * 1000, 1)
Om = torch.randn(30, n, dtype=torch.float64, device="cuda").t()
Ph = torch.randn(60, m, dtype=torch.float64, device="cuda").t()
ms = []
for _ in range(12):
    r = ctx.view_fused(A, Om, Ph, flags=rsvd.RSVD_PROFILE)
    ms.append(r[-1].view_ms)
res["fused30_60"] = round(sorted(ms[2:])[len(ms[2:]) // 2] * 1000, 1)
print(json.dumps(res))
