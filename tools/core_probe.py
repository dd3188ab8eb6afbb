"""Core SVD (Jacobi) time and sweeps by width on R factors shaped like the algorithms' cores:
R = qr(A Omega).R for a graded A (sigma_i = exp(-i/100) + noise, C5-like), Jacobi on R^T
(what alg_subspace does).  python tools/core_probe.py [widths...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07531_b200 import build, rsvd  # noqa: E402

build.build()
ctx = rsvd.Context(0)
widths = [int(x) for x in sys.argv[1:]] or [30, 60, 70, 120, 140, 250, 500]
rng = np.random.default_rng(3)
for w in widths:
    m = 4 * w + 200
    U, _ = np.linalg.qr(rng.standard_normal((m, m)))
    V, _ = np.linalg.qr(rng.standard_normal((m, m)))
    s = np.exp(-np.arange(m) / (w / 2.5)) + 1e-6
    A = (U * s) @ V.T
    R = np.linalg.qr(A @ rng.standard_normal((m, w)))[1]
    M = torch.from_numpy(np.ascontiguousarray(R)).cuda().t()   # M = R^T, column-major
    for flags, nm in ((rsvd.RSVD_CORE_NO_J, "noJ"), (0, "J")):
        ctx.core_svd(M, flags=flags)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            Uc, S, Vc, info = ctx.core_svd(M, flags=flags)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        sref = np.linalg.svd(R, compute_uv=False)
        err = np.max(np.abs(S.cpu().numpy() - sref) / sref)
        print(f"w={w:4d} {nm:3s} ms={np.median(ts):8.3f} sweeps={info.jacobi_sweeps:3d} max_rel_sigma_err={err:.2e}",
              flush=True)
