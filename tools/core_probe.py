"""Time the core SVD (rsvd_core_svd) on cores taken from real C2 runs; print sweeps."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import synth as S
from paper_1804_07531_b200 import rsvd
cfg = S.CONFIGS["C2"]
A = S.make_matrix(cfg); Om = S.gaussian_test_matrix(cfg.n, cfg.l, cfg, S.ROLE_OMEGA)
Qc, Rc = np.linalg.qr(A @ Om); Qr, Rr = np.linalg.qr(A.T @ Qc)
K = np.hstack([Qc, np.linalg.qr(A @ (A.T @ Qc))[0]]); Qk = np.linalg.qr(K)[0]; _, Rk = np.linalg.qr(A.T @ Qk)
ctx = rsvd.Context(0)
out = {}
for name, R in [("Rr30", Rr), ("Rr30T", Rr.T.copy()), ("Rk60", Rk), ("Rk60T", Rk.T.copy())]:
    Md = torch.from_numpy(np.ascontiguousarray(R.T)).cuda().t()
    for it in range(3):
        U, s, V, info = ctx.core_svd(Md, flags=rsvd.RSVD_PROFILE)
    out[name] = {"sweeps": info.jacobi_sweeps, "ms": info.total_ms}
print(json.dumps(out))
