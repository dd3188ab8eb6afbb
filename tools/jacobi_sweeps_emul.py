"""Host emulation (NumPy, exact angles) of the core Jacobi's sweep count on the real C2 cores, with
and without a QR preconditioning of the core: does a preconditioned start save sweeps?  The
round-robin ordering, the threshold (sqrt(w) u) and the 'no rotation above 1e-10' early exit are
those of k_jacobi_small.  usage: python tools/jacobi_sweeps_emul.py  (CPU only, ~1 min)"""
import os
import sys

import numpy as np
import scipy.linalg as sl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth as S


def sweeps(W, tol):
    W = W.copy()
    c = W.shape[1]
    if c & 1:
        W = np.hstack([W, np.zeros((W.shape[0], 1))])
    ce = W.shape[1]
    m1, npairs = ce - 1, ce // 2
    for sw in range(60):
        rot = big = False
        for rnd in range(m1):
            ps = [rnd] + [min((rnd + g) % m1, (rnd - g) % m1) for g in range(1, npairs)]
            qs = [m1] + [max((rnd + g) % m1, (rnd - g) % m1) for g in range(1, npairs)]
            X, Y = W[:, ps], W[:, qs]
            a, b, cc = (X * X).sum(0), (Y * Y).sum(0), (X * Y).sum(0)
            do = (cc * cc > tol * tol * a * b) & (cc != 0)
            if not do.any():
                continue
            rot = True
            big |= bool((cc * cc > 1e-20 * a * b)[do].any())
            d = b - a
            with np.errstate(over="ignore", divide="ignore", invalid="ignore"):
                rho = np.clip(2 * cc / np.maximum(np.abs(d), 1e-300), -1e100, 1e100)
                t = np.where(d < 0, -1, 1) * rho / (1 + np.sqrt(1 + rho * rho))
            cs = np.where(do, 1 / np.sqrt(1 + t * t), 1.0)
            sn = np.where(do, cs * t, 0.0)
            W[:, ps], W[:, qs] = cs * X - sn * Y, sn * X + cs * Y
        if not rot or not big:
            return sw + 1
    return 60


cfg = S.CONFIGS["C2"]
A = S.make_matrix(cfg)
Om = S.gaussian_test_matrix(A.shape[1], cfg.l, cfg, S.ROLE_OMEGA)
Y1 = A @ Om
cores = {}
Q, _ = np.linalg.qr(np.hstack([Y1, A @ (A.T @ Y1)]))          # Alg. 9 v = 4: K = [A Om, A A^T A Om]
cores["krylov_v4 (w=60)"] = np.linalg.qr(A.T @ Q)[1]
Q, _ = np.linalg.qr(Y1)                                          # Alg. 2 v = 3: last qr(A Q_r)
Qr, _ = np.linalg.qr(A.T @ Q)
cores["subspace_v3 (w=30)"] = np.linalg.qr(A @ Qr)[1]
for name, R in cores.items():
    tol = 2.220446049250313e-16 * np.sqrt(R.shape[0])
    row = {"R^T (as built)": sweeps(R.T, tol), "R": sweeps(R, tol)}
    row["qr(R^T).R^T"] = sweeps(np.linalg.qr(R.T)[1].T, tol)
    row["qrp(R^T).R^T"] = sweeps(sl.qr(R.T, pivoting=True)[1].T, tol)
    row["norm-sorted R^T"] = sweeps(R.T[:, np.argsort(-np.linalg.norm(R.T, axis=0))], tol)
    print(name, row, flush=True)
