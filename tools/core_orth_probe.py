"""Core SVD orthogonality vs grading: max |U^T U - I|, |V^T V - I| and sigma error of the Jacobi
core on R = qr(A Omega).R for A with sigma_i = 10^(-d i / w).  python tools/core_orth_probe.py d w..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07531_b200 import build, rsvd  # noqa: E402

build.build()
ctx = rsvd.Context(0)
d = float(sys.argv[1])
widths = [int(x) for x in sys.argv[2:]] or [120, 250]
rng = np.random.default_rng(5)
for w in widths:
    m = 2 * w + 100
    U, _ = np.linalg.qr(rng.standard_normal((m, m)))
    V, _ = np.linalg.qr(rng.standard_normal((m, m)))
    s = 10.0 ** (-d * np.arange(m) / w)
    A = (U * s) @ V.T
    R = np.linalg.qr(A @ rng.standard_normal((m, w)))[1]
    M = torch.from_numpy(np.ascontiguousarray(R)).cuda().t()
    sref = np.linalg.svd(R, compute_uv=False)
    for flags, nm in ((rsvd.RSVD_CORE_NO_J, "noJ"), (0, "J")):
        Uc, S, Vc, info = ctx.core_svd(M, flags=flags)
        torch.cuda.synchronize()
        Uh, Sh, Vh = Uc.cpu().numpy(), S.cpu().numpy(), Vc.cpu().numpy()
        eu = np.max(np.abs(Uh.T @ Uh - np.eye(w)))
        ev = np.max(np.abs(Vh.T @ Vh - np.eye(w)))
        es = np.max(np.abs(Sh - sref) / sref)
        print(f"d={d} w={w:4d} {nm:3s} sweeps={info.jacobi_sweeps:3d} |UtU-I|={eu:.2e} |VtV-I|={ev:.2e} "
              f"rel_sigma={es:.2e}", flush=True)
