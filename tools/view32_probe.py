"""Time the fp32 (tcgen05 3xTF32) view kernels alone via rsvd_view + RSVD_PROFILE, and one C5-shaped
subspace SVD; prints JSON lines.  usage: python tools/view32_probe.py [m] [n]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_1804_07531_b200 import rsvd

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
TF32_PEAK = 1673.8 * 1.1 / 2.25   # measured bf16 burst x nominal tf32/bf16 ratio (B200_PROFILING.md)
HBM = 6456.8
ctx = rsvd.Context(0)
A = torch.empty(m, n, dtype=torch.float32, device="cuda")
for r0 in range(0, m, 8192):
    A[r0:r0 + 8192].normal_()
for w in (64, 128, 250, 500):
    for trans in (0, 1):
        X = torch.randn(w, m if trans else n, dtype=torch.float32, device="cuda").t()
        for _ in range(2):
            ctx.view(A, X, trans=bool(trans), flags=rsvd.RSVD_PROFILE)
        ms = []
        for _ in range(5):
            _, info = ctx.view(A, X, trans=bool(trans), flags=rsvd.RSVD_PROFILE)
            ms.append(info.view_ms)
        t = min(ms)
        fl = 2.0 * m * n * w
        rec = dict(m=m, n=n, w=w, trans=trans, ms=t, tf_1x=fl / t / 1e9, tf_3x=3 * fl / t / 1e9,
                   frac_tensor_3x=3 * fl / t / 1e9 / TF32_PEAK, gbs=m * n * 4 / t / 1e6,
                   frac_hbm=m * n * 4 / t / 1e6 / HBM)
        print(json.dumps(rec), flush=True)
        del X
Om = torch.randn(250, n, dtype=torch.float32, device="cuda").t()
for v in (2, 3):
    ctx.subspace(A, 200, 50, v, Om, flags=rsvd.RSVD_PROFILE)
    U, s, V, info = ctx.subspace(A, 200, 50, v, Om, flags=rsvd.RSVD_PROFILE)
    print(json.dumps(dict(alg="subspace", v=v, total_ms=info.total_ms, view_ms=info.view_ms,
                          views=info.view_launches)), flush=True)
