"""Time the core-SVD Jacobi kernels (rsvd_core_svd, CUDA events around the call) on QR-preconditioned
cores shaped like the algorithms' (R^T of a CholeskyQR of a sketch with decaying spectrum)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_1804_07531_b200 import rsvd
ctx = rsvd.Context(0)
rng = np.random.default_rng(0)
for w in [int(x) for x in (sys.argv[1:] or ["30", "60", "70", "120", "140", "160", "200", "250", "500"])]:
    for kind in ("exp", "flat"):
        s = np.exp(-np.arange(w) / 100.0) if kind == "exp" else 1.0 + 0.01 * rng.standard_normal(w)
        X = np.linalg.qr(rng.standard_normal((w, w)))[0]
        Yh = np.linalg.qr(rng.standard_normal((4 * w, w)))[0]
        R = np.linalg.qr((Yh * s) @ X.T)[1]          # R of a sketch with spectrum s
        Md = torch.from_numpy(np.ascontiguousarray(R.T)).cuda().t()
        for flags in (rsvd.RSVD_CORE_NO_J,):
            ctx.core_svd(Md, flags=flags)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            U, S, V, info = ctx.core_svd(Md, flags=flags)
            e1.record()
            torch.cuda.synchronize()
            err = float(np.max(np.abs(S.cpu().numpy() - np.linalg.svd(R, compute_uv=False)) / s.max()))
            print(json.dumps(dict(w=w, kind=kind, ms=e0.elapsed_time(e1), sweeps=info.jacobi_sweeps, err=err)), flush=True)
