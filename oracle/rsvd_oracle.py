"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct fp64 CPU implementation of the pass-efficient randomized
SVD algorithms of arXiv 1804.07531 (Bjarkason, "Pass-efficient randomized algorithms for
low-rank matrix approximation using any number of views").  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may
import it.  It shares no code with the CUDA path (``paper_1804_07531_b200``).

Notation follows the paper (PAPER.md lines noted as P:<line>):
    A is n_r x n_c; p = target rank; l = oversampling (sketch width p + l);
    Omega_r is the range test matrix (n_c x (p+l)); Omega_c the co-range one (n_r x (p+l2)).
The C ABI (BASELINE.json) calls the same two integers (k, p) — positionally identical:
    oracle (p, l)  ==  ABI (k, p).

Every routine is in float64 regardless of the input dtype (fp32 inputs are upcast once, so the
oracle gives the exact-arithmetic answer for the given fp32 bytes).

Conventions the paper leaves open:
  * qr: Householder (numpy/LAPACK), thin, signs normalised so diag(R) >= 0 (reading R1).
  * tsvd: LAPACK SVD, singular values descending (reading R2).
  * Random test matrices are INPUTS (reading R3): the caller passes Omega_r / Omega_c, which
    replace the paper's randn calls.

Pins: see tests/test_oracle_pins.py.  Parity unpinned: the actual values of the randomized
outputs on noisy / slowly decaying inputs have no closed form; they are pinned only indirectly
(exact-rank recovery, diagonal closed forms, Alg.2==Alg.1 / Alg.9==Alg.2 identities, brute
force at full sampling, Thm A.1, the Thm 3.1/4.1 bounds).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "qr", "orth", "tsvd", "chol_lower", "jacobi_svd",
    "std_subspace_iteration", "gen_subspace_iteration", "qrqc", "one_view_tropp", "one_view_woolfe",
    "plan_flat", "plan_decay", "plan_rapid", "plan_balanced", "minvar_spectra", "minvar_select",
    "one_view_minvar", "one_view_extended", "plan_extended", "pinv",
    "row_stream_qb",
    "gen_block_krylov", "row_block_krylov", "normal_matrix_tevd", "nystrom_tevd", "pinched_tevd", "recommend_input", "svd_of",
    "views_and_vectors", "PanelOp", "rel_frobenius_error", "rel_spectral_error", "projector_distance",
    "residual_fro", "half_power_lhs_rhs", "thm_bound",
    "GOAL_SVD", "GOAL_LEFT", "GOAL_RIGHT", "GOAL_NORMAL",
]


# ============================================================ dense primitives

def _f64(M) -> np.ndarray:
    return np.asarray(M, dtype=np.float64)


def qr(M):
    """[Q, R] = qr(M): thin QR, Q n_r x n_c orthonormal, R n_c x n_c upper triangular.

    Householder via LAPACK; column signs normalised so diag(R) >= 0 (reading R1: the paper
    defines qr without a sign)."""
    M = _f64(M)
    Q, R = np.linalg.qr(M, mode="reduced")
    s = np.where(np.diag(R) < 0, -1.0, 1.0)
    return Q * s, R * s[:, None]


def orth(M):
    """Q = orth(M): orthonormal basis of range(M).  Used only where the paper writes orth;
    for full-column-rank M this is qr(M).Q."""
    return qr(M)[0]


def tsvd(M, p):
    """[U_p, Lambda_p, V_p] = tsvd(M, p): exact rank-p truncated SVD, M = U Lambda V^* (P:67)."""
    M = _f64(M)
    U, s, Vt = np.linalg.svd(M, full_matrices=False)
    return U[:, :p], s[:p], Vt[:p, :].T


def chol_lower(S):
    """C_L = chol(S, LOWER) with S = C_L C_L^* (P:69); plain column Cholesky–Banachiewicz."""
    S = _f64(S)
    n = S.shape[0]
    L = np.zeros_like(S)
    for j in range(n):
        d = S[j, j] - np.dot(L[j, :j], L[j, :j])
        if d <= 0.0:
            raise np.linalg.LinAlgError("chol: non-positive pivot")
        L[j, j] = np.sqrt(d)
        for i in range(j + 1, n):
            L[i, j] = (S[i, j] - np.dot(L[i, :j], L[j, :j])) / L[j, j]
    return L


def jacobi_svd(M, tol=None, max_sweeps=60):
    """Full SVD by cyclic one-sided (Hestenes) Jacobi: orthogonalise the columns of W = M J by
    plane rotations until every pair is orthogonal to ``tol``; then sigma_i = ||W_i||,
    U_i = W_i / sigma_i, V = J.  Independent of LAPACK; used to brute-force small cases."""
    W = _f64(M).copy()
    n_r, n_c = W.shape
    transposed = False
    if n_r < n_c:
        W = W.T.copy()
        n_r, n_c = n_c, n_r
        transposed = True
    J = np.eye(n_c)
    tol = (n_c * np.finfo(np.float64).eps) if tol is None else tol
    for _ in range(max_sweeps):
        rotated = False
        for i in range(n_c - 1):
            for j in range(i + 1, n_c):
                a = np.dot(W[:, i], W[:, i])
                b = np.dot(W[:, j], W[:, j])
                c = np.dot(W[:, i], W[:, j])
                if abs(c) <= tol * np.sqrt(a * b) or c == 0.0:
                    continue
                rotated = True
                zeta = (b - a) / (2.0 * c)
                t = np.sign(zeta) / (abs(zeta) + np.sqrt(1.0 + zeta * zeta)) if zeta != 0 else 1.0
                cs = 1.0 / np.sqrt(1.0 + t * t)
                sn = cs * t
                wi, wj = W[:, i].copy(), W[:, j].copy()
                W[:, i] = cs * wi - sn * wj
                W[:, j] = sn * wi + cs * wj
                ji, jj = J[:, i].copy(), J[:, j].copy()
                J[:, i] = cs * ji - sn * jj
                J[:, j] = sn * ji + cs * jj
        if not rotated:
            break
    else:
        raise RuntimeError("jacobi_svd: not converged")
    s = np.sqrt(np.sum(W * W, axis=0))
    order = np.argsort(-s, kind="stable")
    s = s[order]
    W = W[:, order]
    J = J[:, order]
    U = np.zeros_like(W)
    nz = s > 0
    U[:, nz] = W[:, nz] / s[nz]
    if transposed:
        return J, s, U
    return U, s, J


# ============================================================ matrix access ("views")

class _Op:
    """A or its transpose as the algorithm's input matrix (P:198 'with either J or J^* as input').

    ``apply(X)`` = (input) X ; ``adjoint(Y)`` = (input)^* Y.  Each call is one matrix view."""

    def __init__(self, A, transpose=False):
        self.A = _f64(A)
        self.T = bool(transpose)
        self.views = 0
        self.vectors = 0

    @property
    def shape(self):
        r, c = self.A.shape
        return (c, r) if self.T else (r, c)

    def apply(self, X):
        self.views += 1
        self.vectors += X.shape[1]
        return (self.A.T @ X) if self.T else (self.A @ X)

    def adjoint(self, Y):
        self.views += 1
        self.vectors += Y.shape[1]
        return (self.A @ Y) if self.T else (self.A.T @ Y)


class PanelOp(_Op):
    """The same operator as _Op, with every view evaluated one row panel of A at a time
    ("views as BLAS A[panel] @ X / A[panel].T @ Y over row panels", so that an
    80 GB A never has to be held in fp64 at once).  ``A`` is any row-sliceable array (ndarray or
    memmap) of any float dtype; each panel is upcast to fp64 on its own.

        (A X)[panel]  = A[panel] X                      (rows are independent: same numbers as _Op)
        A^* Y         = sum over panels, in row order, of A[panel]^* Y[panel]

    Only the summation order of A^* Y differs from the dense product (the definition of the view,
    P:100); the algorithms above are unchanged."""

    def __init__(self, A, transpose=False, panel_rows=4096):
        self.A = A
        self.T = bool(transpose)
        self.views = 0
        self.vectors = 0
        self.panel_rows = int(panel_rows)

    def _rows(self, X):                           # A X
        X = _f64(X)
        m = self.A.shape[0]
        Y = np.empty((m, X.shape[1]))
        for r0 in range(0, m, self.panel_rows):
            r1 = min(m, r0 + self.panel_rows)
            Y[r0:r1] = _f64(self.A[r0:r1]) @ X
        return Y

    def _cols(self, Y):                           # A^* Y
        Y = _f64(Y)
        m, n = self.A.shape
        Z = np.zeros((n, Y.shape[1]))
        for r0 in range(0, m, self.panel_rows):
            r1 = min(m, r0 + self.panel_rows)
            Z += _f64(self.A[r0:r1]).T @ Y[r0:r1]
        return Z

    def apply(self, X):
        self.views += 1
        self.vectors += X.shape[1]
        return self._cols(X) if self.T else self._rows(X)

    def adjoint(self, Y):
        self.views += 1
        self.vectors += Y.shape[1]
        return self._rows(Y) if self.T else self._cols(Y)


# ============================================================ Algorithm 1

def std_subspace_iteration(A, p, l, q, Omega_r, transpose=False, _op=None):
    """Alg. 1 — randomized SVD using standard subspace iteration, 2(q+1) views.

    Returns (U_p, Lambda_p, V_p) of the input matrix (A, or A^* if transpose)."""
    op = _op or _Op(A, transpose)
    Omega_r = _f64(Omega_r)
    Qc, _ = qr(op.apply(Omega_r))                 # line 2
    for _j in range(q):                           # lines 3-6
        Qr, _ = qr(op.adjoint(Qc))
        Qc, _ = qr(op.apply(Qr))
    Qr, Rr = qr(op.adjoint(Qc))                   # line 7
    Vh, lam, Uh = tsvd(Rr, p)                     # line 8: R_r = Vh Lam Uh^*
    return Qc @ Uh, lam, Qr @ Vh                  # line 9


# ============================================================ Algorithm 2

def gen_subspace_iteration(A, p, l, v, Omega_r, transpose=False, _op=None):
    """Alg. 2 — randomized SVD using generalized subspace iteration, any v >= 2.

    Omega_r (n_c x (p+l)) replaces line 1's randn.  Returns (U_p, Lambda_p, V_p) of the input
    matrix; odd j: [Q_c,R_c] = qr(A Q_r); even j: [Q_r,R_r] = qr(A^* Q_c)."""
    if v < 2:
        raise ValueError("Alg. 2 needs v >= 2 (P:142)")
    op = _op or _Op(A, transpose)
    Qr = _f64(Omega_r)                            # line 1
    Qc = Rc = Rr = None
    for j in range(1, v + 1):                     # lines 2-8
        if j % 2 == 1:
            Qc, Rc = qr(op.apply(Qr))
        else:
            Qr, Rr = qr(op.adjoint(Qc))
    if v % 2 == 0:                                # lines 9-13
        Vh, lam, Uh = tsvd(Rr, p)                 # R_r = Vh Lam Uh^*
    else:
        Uh, lam, Vh = tsvd(Rc, p)                 # R_c = Uh Lam Vh^*
    return Qc @ Uh, lam, Qr @ Vh                  # line 14


def qrqc(A, p, l, v, Omega_r, transpose=False, _op=None):
    """Alg. 3 — QrQc: approximate range (v odd, returns Q_c) or co-range (v even, returns Q_r)
    basis after v views."""
    op = _op or _Op(A, transpose)
    Qr = _f64(Omega_r)
    Qc = None
    for j in range(1, v + 1):
        if j % 2 == 1:
            Qc, _ = qr(op.apply(Qr))
        else:
            Qr, _ = qr(op.adjoint(Qc))
    return Qr if v % 2 == 0 else Qc


# ============================================================ Algorithm 7

def one_view_tropp(A, p, l1, l2, lc, Omega_r, Omega_c, transpose=False, _op=None):
    """Alg. 7 — randomized 1-view TSVD, Tropp variant with truncation parameter l_c.

    Omega_r: n_c x (p+l1); Omega_c: n_r x (p+l2); 0 <= lc <= l1 <= l2.  lc = l1 gives the
    baseline [Tropp Alg. 7].  The optional orth of the test matrices (line 2) is off
    ('not used for the experiments').  Line 3's a) and b) are one logical pass; the
    oracle counts it as one view."""
    if not (0 <= lc <= l1 <= l2):
        raise ValueError("Alg. 7 needs 0 <= l_c <= l_1 <= l_2 (P:663)")
    op = _op or _Op(A, transpose)
    Omega_r = _f64(Omega_r)
    Omega_c = _f64(Omega_c)
    Yc = op.apply(Omega_r)                        # line 3 a)
    Yr = op.adjoint(Omega_c)                      # line 3 b)
    op.views -= 1                                 # a) and b) together are ONE view
    if lc < l1:                                   # lines 4-7
        Qc, Rc = qr(Yc)
        Qhc, _, _ = tsvd(Rc, p + lc)
        Qc = Qc @ Qhc
    else:                                         # line 9
        Qc, _ = qr(Yc)
    Qh, Rh = qr(Omega_c.T @ Qc)                   # line 11
    X = np.linalg.solve(Rh, Qh.T @ Yr.T)          # line 12: X = Rh^{-1} Qh^* Y_r^*
    Uh, lam, Vp = tsvd(X, p)                      # line 13
    return Qc @ Uh, lam, Vp                       # line 14


# ============================================================ Algorithm 8

def one_view_woolfe(A, p, l1, l2, lc, Omega_r, Omega_c, transpose=False, _op=None):
    """Alg. 8 — randomized 1-view TSVD, Woolfe variant.

    Both bases are truncated to their p + l_c leading singular directions (lines 4-6) and the
    small least-squares problem (Omega_c^* Q_c) Xh = Y_r^* Q_r (line 7) is solved by QR, as
    Alg. 7 line 11-12 does."""
    if not (0 <= lc <= l1 <= l2):
        raise ValueError("Alg. 8 needs 0 <= l_c <= l_1 <= l_2 (P:701)")
    op = _op or _Op(A, transpose)
    Omega_r = _f64(Omega_r)
    Omega_c = _f64(Omega_c)
    Yc = op.apply(Omega_r)                        # line 3 a)
    Yr = op.adjoint(Omega_c)                      # line 3 b)
    op.views -= 1                                 # one logical pass
    Qc, Rc = qr(Yc)                               # line 4 a)
    Qr, Rr = qr(Yr)                               # line 4 b)
    Qhc, _, _ = tsvd(Rc, p + lc)                  # line 5 a)
    Qhr, _, _ = tsvd(Rr, p + lc)                  # line 5 b)
    Qc = Qc @ Qhc                                 # line 6 a)
    Qr = Qr @ Qhr                                 # line 6 b)
    Qh, Rh = qr(Omega_c.T @ Qc)                   # line 7: least squares via QR
    Xh = np.linalg.solve(Rh, Qh.T @ (Yr.T @ Qr))
    Uh, lam, Vh = tsvd(Xh, p)                     # line 8
    return Qc @ Uh, lam, Qr @ Vh                  # line 9 c), d)


# ============================================================ oversampling

def plan_flat(p, T):
    """Eq. (overflat): l_1 for a flat spectrum, l_2 = T - 2p - l_1 (needs T >= 2p + 6,
    P:604)."""
    if T < 2 * p + 6:
        raise ValueError("T >= 2p + 6 required (P:604)")
    num = np.sqrt(p * (T - p - 2) * (1.0 - 2.0 / (T - 1))) - (p - 1)
    l1 = max(2, int(np.floor((T - 1) * num / (T - 2 * p - 1))) - p)
    return l1, T - 2 * p - l1


def plan_decay(p, T):
    """Eq. (overmed): l_1 = max{2, floor((T-1)/3) - p}."""
    if T < 2 * p + 6:
        raise ValueError("T >= 2p + 6 required (P:604)")
    l1 = max(2, (T - 1) // 3 - p)
    return l1, T - 2 * p - l1


def plan_rapid(p, T):
    """Eq. (overrapid): l_1 = floor((T-2)/2) - p."""
    if T < 2 * p + 6:
        raise ValueError("T >= 2p + 6 required (P:604)")
    l1 = (T - 2) // 2 - p
    return l1, T - 2 * p - l1


def plan_balanced(p, T, alpha):
    """l_1 ~= l_2 with l_1 = floor(T/2) - p and l_c = floor(alpha l_1), 0 <= alpha <= 1
    (Eq. lcutfixedratio).  Returns (l1, l2, lc)."""
    if not (0.0 <= alpha <= 1.0):
        raise ValueError("0 <= alpha <= 1 (P:720)")
    l1 = T // 2 - p
    l2 = T - 2 * p - l1
    return l1, l2, int(np.floor(alpha * l1))


# ============================================================ minimum-variance l_c

def minvar_spectra(Yc, Yr, Omega_c, p, l1):
    """lambda_{1..p}(l_c) for l_c = 0..l_1: the top-p singular values of X(l_c) of Alg. 7 with
    Q_c = the p + l_c leading left singular vectors of Y_c (one SVD of Y_c, one
    Omega_c^* Q_c product, the first p + l_c columns per trial).  Each trial solves its own
    least-squares problem by QR as Alg. 7 lines 11-12.  Returns a (l_1 + 1) x p array."""
    Yc, Yr, Omega_c = _f64(Yc), _f64(Yr), _f64(Omega_c)
    Qc, Rc = qr(Yc)
    Uc, _, _ = tsvd(Rc, Rc.shape[1])              # left singular vectors of Y_c = Q_c U_c
    M = Omega_c.T @ (Qc @ Uc)
    lam = np.zeros((l1 + 1, p))
    for lc in range(l1 + 1):
        Qh, Rh = qr(M[:, :p + lc])
        X = np.linalg.solve(Rh, Qh.T @ Yr.T)
        lam[lc] = np.linalg.svd(X, compute_uv=False)[:p]
    return lam


def _ratio(a, b):
    """lambda_i(j) / lambda_i(l_c) with 0/0 = 1 and a/0 = inf (reading R20)."""
    if b > 0:
        return a / b
    return 1.0 if a == 0 else np.inf


def minvar_select(lam):
    """Eq. (MinVar): s(l_c) stacks lambda_i(l_c - 1)/lambda_i(l_c) (l_c > 0),
    lambda_i(l_c)/lambda_i(l_c) and lambda_i(l_c + 1)/lambda_i(l_c); l_c^MinVar = argmin Var[s(l_c)]
    over 0 <= l_c < l_1.  Var is the unbiased sample variance and ties go to the smallest l_c
    (readings R19, R20).  lam: (l_1 + 1) x p.  Returns (lc, variances)."""
    l1 = lam.shape[0] - 1
    if l1 <= 0:
        return 0, np.zeros(0)
    var = np.zeros(l1)
    for lc in range(l1):
        s = []
        for j in ([lc - 1] if lc > 0 else []) + [lc, lc + 1]:
            s += [_ratio(lam[j, i], lam[lc, i]) for i in range(lam.shape[1])]
        s = np.array(s)
        if not np.all(np.isfinite(s)):
            var[lc] = np.inf
            continue
        mu = sum(s) / len(s)
        var[lc] = sum((x - mu) ** 2 for x in s) / (len(s) - 1)
    best = 0
    for lc in range(1, l1):
        if var[lc] < var[best]:
            best = lc
    return best, var


def one_view_minvar(A, p, l1, l2, Omega_r, Omega_c, transpose=False, _op=None):
    """Alg. 7 with l_c chosen by the minimum-variance post-processing.  The trials
    reuse the one view's sketches ('does not require re-evaluating the sketches').
    Returns (U, lam, V, lc)."""
    op = _op or _Op(A, transpose)
    Yc = op.apply(_f64(Omega_r))
    Yr = op.adjoint(_f64(Omega_c))
    op.views -= 1
    lc, _ = minvar_select(minvar_spectra(Yc, Yr, Omega_c, p, l1))
    U, lam, V = one_view_tropp(None, p, l1, l2, lc, Omega_r, Omega_c, _op=_Sketched(op, Yc, Yr))
    return U, lam, V, lc


class _Sketched:
    """Replays an already-taken pair of sketches (Y_c, Y_r) to Alg. 7 without touching A again."""

    def __init__(self, op, Yc, Yr):
        self.op, self.Yc, self.Yr = op, Yc, Yr
        self.views = op.views + 1

    def apply(self, X):
        return self.Yc

    def adjoint(self, X):
        return self.Yr


# ============================================================ extended sketch

def pinv(M, rcond=1e-12):
    """Moore-Penrose pseudo-inverse with singular values below rcond * sigma_max dropped (the
    paper writes the dagger without a cutoff; reading R24)."""
    return np.linalg.pinv(_f64(M), rcond=rcond)


def one_view_extended(A, p, l1, l2, Omega_r, Omega_c, Phi_r, Phi_c, variant="bwz2", transpose=False, _op=None):
    """Extended 1-view sketch: Y_c = A Omega_r, Y_r = A^* Omega_c, Z = Phi_r^* A Phi_c
    (Phi_r n_r x s, Phi_c n_c x s, SRFT inputs, s >= p + l1); Q_c R_c := Y_c, Q_r R_r := Y_r,
    U_c T_c := Phi_r^* Q_c, U_r T_r := Phi_c^* Q_r, and
      bwz  (Eq. bwz):         A ~ Q_c T_c^+ [[U_c^* Z U_r]]_p (T_r^*)^+ Q_r^*
      bwz2 (Eq. bwzimproved): A ~ Q_c [[T_c^+ U_c^* Z U_r (T_r^*)^+]]_p Q_r^*
    Returns the rank-p SVD (U, lambda, V) of the approximation.  A Omega_r and A Phi_c are one
    product with the test matrices side by side, and Y_r comes from the same access: one view."""
    if variant not in ("bwz", "bwz2"):
        raise ValueError(variant)
    op = _op or _Op(A, transpose)
    Omega_r, Omega_c = _f64(Omega_r), _f64(Omega_c)
    Phi_r, Phi_c = _f64(Phi_r), _f64(Phi_c)
    if Phi_r.shape[1] < p + l1 or Phi_c.shape[1] < p + l1:
        raise ValueError("s >= p + l_1 (P:805)")
    Yc = op.apply(Omega_r)
    Yr = op.adjoint(Omega_c)
    W = op.apply(Phi_c)
    op.views -= 2
    Z = Phi_r.T @ W                               # Z = Phi_r^* A Phi_c
    Qc, _ = qr(Yc)
    Qr, _ = qr(Yr)
    Uc, Tc = qr(Phi_r.T @ Qc)
    Ur, Tr = qr(Phi_c.T @ Qr)
    Tcp, Trp = pinv(Tc), pinv(Tr)
    if variant == "bwz2":
        core = Tcp @ (Uc.T @ Z @ Ur) @ Trp.T
    else:
        Ux, sx, Vx = tsvd(Uc.T @ Z @ Ur, p)
        core = (Tcp @ Ux) @ np.diag(sx) @ (Trp @ Vx).T
    Uk, lam, Vk = tsvd(core, p)
    return Qc @ Uk, lam, Qr @ Vk


def plan_extended(p, T, n_r, n_c):
    """Eq. (bwzafac8): l_1 = l_2 = floor(0.8 floor(T/2 - p)) and s the largest value with
    (2p + l_1 + l_2 + 1)(n_r + n_c) + s(s + 2) <= T (n_r + n_c) (reading R25: 'approximately
    equals' taken as <=, floored at p + l_1).  Returns (l1, l2, s)."""
    if T < 2 * p + 6:
        raise ValueError("T >= 2p + 6 required (P:604)")
    l1 = int(np.floor(0.8 * np.floor(T / 2 - p)))
    budget = T * (n_r + n_c) - (2 * p + 2 * l1 + 1) * (n_r + n_c)
    s = 0
    while (s + 1) * (s + 3) <= budget:
        s += 1
    if s < p + l1:
        raise ValueError("budget leaves s < p + l_1")
    return l1, l1, s


# ============================================================ single pass over the rows

def row_stream_qb(A, p, l, Omega_r, panel_rows=1, order=None):
    """Single pass over the rows of A: Y_c[i, :] = A[i, :] Omega_r and
    Yhat_r = sum_i A[i, :]^* Y_c[i, :] accumulated row by row (rows visited once, in `order`);
    [Q_c, R_c] = qr(Y_c); B^* R_c = Yhat_r solved with the TSVD pseudo-inverse of R_c (P:855:
    'estimating a solution using a pseudoinverse'); then the rank-p SVD of Q_c B.  With R_c
    invertible, B^* = A^* Q_c and this is Alg. 2 with v = 2.  Returns (U, lambda, V)."""
    A = _f64(A)
    Omega_r = _f64(Omega_r)
    n_r, n_c = A.shape
    w = Omega_r.shape[1]
    Yc = np.zeros((n_r, w))
    Yr_hat = np.zeros((n_c, w))
    rows = np.arange(n_r) if order is None else np.asarray(order)
    for i0 in range(0, n_r, panel_rows):
        idx = rows[i0:i0 + panel_rows]
        Yc[idx] = A[idx] @ Omega_r                # Y_c[i, :] = A[i, :] Omega_r
        Yr_hat += A[idx].T @ Yc[idx]              # Yhat_r += A[i, :]^* Y_c[i, :]
    Qc, Rc = qr(Yc)
    Bt = Yr_hat @ pinv(Rc)                        # B^* = Yhat_r R_c^+   (n_c x w)
    Qb, Rb = qr(Bt)                               # Q_c B = Q_c R_b^* Q_b^*
    Uh, lam, Vh = tsvd(Rb.T, p)
    return Qc @ Uh, lam, Qb @ Vh


# ============================================================ Algorithm 9

def gen_block_krylov(A, p, l, v, Omega_r, transpose=False, _op=None, return_basis=False):
    """Alg. 9 — randomized SVD using the generalized block Krylov method, any v >= 2.

    Blocks Q^j for j < v-1 are orthonormalised, the last block Q^{v-1} is left raw (lines 3-4);
    K_c = [Q_c^1 Q_c^3 ... Q_c^{v-1}] (v even) or K_r = [Q_r^2 ... Q_r^{v-1}] (v odd) is
    orthonormalised with qr (lines 9/14), then one more view and a tsvd."""
    if v < 2:
        raise ValueError("Alg. 9 needs v >= 2 (P:903)")
    op = _op or _Op(A, transpose)
    Q = {0: _f64(Omega_r)}                        # line 1: Q_r^0
    for j in range(1, v):                         # lines 2-7
        if j % 2 == 1:
            B = op.apply(Q[j - 1])
        else:
            B = op.adjoint(Q[j - 1])
        Q[j] = qr(B)[0] if j < v - 1 else B
    if v % 2 == 0:                                # lines 8-12
        Kc = np.hstack([Q[j] for j in range(1, v, 2)])
        Qc, _ = qr(Kc)
        Qr, Rr = qr(op.adjoint(Qc))
        Vh, lam, Uh = tsvd(Rr, p)
    else:                                         # lines 13-17
        Kr = np.hstack([Q[j] for j in range(2, v, 2)])
        Qr, _ = qr(Kr)
        Qc, Rc = qr(op.apply(Qr))
        Uh, lam, Vh = tsvd(Rc, p)
    out = (Qc @ Uh, lam, Qr @ Vh)                 # line 18
    if return_basis:
        return out, (Qc, Qr)
    return out


# ============================================================ block Krylov, matrix read row wise

def row_block_krylov(A, p, l, v, Omega_r, panel_rows=1):
    """Block Krylov method for a matrix accessed row by row: A^* A times a block is
    evaluated in ONE pass over the rows, Y[i, :] = A[i, :] X and Z = sum_i A[i, :]^* Y[i, :] (the
    single-pass product of P:849-851), so the Krylov blocks of Alg. 9 need about half
    the views.  Returns ((U_p, Lambda_p, V_p), passes over A).

    v odd  (co-range Krylov subspace): Q^0 = Omega_r; pass i = 1..(v-1)/2 gives
           Z_i = A^* A Q^{i-1}, Q^i = qr(Z_i).Q (the last Z_i stays raw, as Alg. 9 lines 3-6);
           K_r = [Z_1 .. Z_{(v-1)/2}] (orthonormalised blocks, last raw) spans Alg. 9's K_r
           (A^*A Omega, (A^*A)^2 Omega, ...); then Alg. 9 lines 14-17: Q_r = qr(K_r),
           [Q_c, R_c] = qr(A Q_r), tsvd(R_c).  (v-1)/2 + 1 passes instead of v views.
    v even (range Krylov subspace): the same passes also give the range blocks A Q^{i-1}:
           K_c = [A Q^0 .. A Q^{v/2-1}] spans Alg. 9's K_c (A Omega, A A^*A Omega, ...);
           the last block needs only a range pass; then lines 9-12: Q_c = qr(K_c),
           [Q_r, R_r] = qr(A^* Q_c), tsvd(R_r).  v/2 + 1 passes.
    With every intermediate R invertible the subspaces equal Alg. 9's, so the outputs equal
    gen_block_krylov's up to rounding."""
    if v < 2:
        raise ValueError("v >= 2 (P:903)")
    A = _f64(A)
    Omega_r = _f64(Omega_r)
    n_r = A.shape[0]
    passes = 0

    def row_pass(X, want_z=True):
        """One pass over the rows: (A X, A^* A X) accumulated row panel by row panel."""
        nonlocal passes
        passes += 1
        Y = np.zeros((n_r, X.shape[1]))
        Z = np.zeros((A.shape[1], X.shape[1]))
        for i0 in range(0, n_r, panel_rows):
            rows = slice(i0, min(n_r, i0 + panel_rows))
            Y[rows] = A[rows] @ X                  # Y[i, :] = A[i, :] X
            if want_z:
                Z += A[rows].T @ Y[rows]           # Z += A[i, :]^* Y[i, :]
        return Y, Z

    Q = Omega_r
    if v % 2 == 1:
        nb = (v - 1) // 2
        blocks = []
        for i in range(nb):
            _, Z = row_pass(Q)
            if i < nb - 1:
                Q = qr(Z)[0]
                blocks.append(Q)
            else:
                blocks.append(Z)                  # last block raw (Alg. 9 line 4/6, j = v-1)
        Qr, _ = qr(np.hstack(blocks))             # line 15
        Yc, _ = row_pass(Qr, want_z=False)        # line 16: one more (range) pass
        Qc, Rc = qr(Yc)
        Uh, lam, Vh = tsvd(Rc, p)                 # line 17
    else:
        nb = v // 2
        blocks = []
        for i in range(nb):
            Y, Z = row_pass(Q, want_z=(i < nb - 1))
            blocks.append(Y)                      # A Q^{i}: range block (raw)
            if i < nb - 1:
                Q = qr(Z)[0]
        Qc, _ = qr(np.hstack(blocks))             # line 10
        Zr = np.zeros((A.shape[1], Qc.shape[1]))  # line 11: A^* Q_c, one more pass over the rows
        passes += 1
        for i0 in range(0, n_r, panel_rows):
            rows = slice(i0, min(n_r, i0 + panel_rows))
            Zr += A[rows].T @ Qc[rows]
        Qr, Rr = qr(Zr)
        Vh, lam, Uh = tsvd(Rr, p)                 # line 12: R_r = Vh Lam Uh^*
    return (Qc @ Uh, lam, Qr @ Vh), passes


# ============================================================ orientation / outputs

GOAL_SVD, GOAL_LEFT, GOAL_RIGHT, GOAL_NORMAL = 0, 1, 2, 3


def recommend_input(goal, v):
    """Which matrix to feed Alg. 2/9 (0 = A, 1 = A^*):
    even v: V (right) more accurate -> RIGHT/NORMAL use A; odd v: U more accurate -> use A^*.
    LEFT goal uses the reverse rule.  SVD: A."""
    if goal in (GOAL_RIGHT, GOAL_NORMAL):
        return 0 if v % 2 == 0 else 1
    if goal == GOAL_LEFT:
        return 1 if v % 2 == 0 else 0
    return 0


def svd_of(A, algorithm, k, p, v=None, Omega=None, l2=None, lc=None, Phi=None, transpose=False, panel_rows=None):
    """Run an algorithm on A (transpose=False) or on A^* (transpose=True) and return the TSVD
    of A itself: (U, sigma, V) with A ~ U diag(sigma) V^T.  When the algorithm ran on A^*, its
    (U, V) are A's (V, U) (reading R6).  panel_rows: evaluate every view over
    row panels of that many rows (PanelOp; for matrices too large to upcast at once)."""
    op = _Op(A, transpose) if panel_rows is None else PanelOp(A, transpose, panel_rows)
    if algorithm == "subspace":
        U, s, V = gen_subspace_iteration(None, k, p, v, Omega, _op=op)
    elif algorithm == "krylov":
        U, s, V = gen_block_krylov(None, k, p, v, Omega, _op=op)
    elif algorithm == "single_pass" and lc == "minvar":
        U, s, V, _ = one_view_minvar(None, k, p, l2 - k, Omega, Phi, _op=op)
    elif algorithm == "single_pass":
        lc = p if lc is None else lc
        U, s, V = one_view_tropp(None, k, p, l2 - k, lc, Omega, Phi, _op=op)
    elif algorithm == "woolfe":
        lc = p if lc is None else lc
        U, s, V = one_view_woolfe(None, k, p, l2 - k, lc, Omega, Phi, _op=op)
    else:
        raise ValueError(algorithm)
    if transpose:
        U, V = V, U
    return U, s, V, op


def normal_matrix_tevd(A, k, p, v, Omega, algorithm="subspace", transpose=None):
    """Normal-matrix estimate A^T A ~ V diag(sigma^2) V^T from Alg. 2/9 in the recommended
    orientation: input = A for even v, A^* for odd v.
    Returns (V, sigma^2)."""
    if transpose is None:
        transpose = bool(recommend_input(GOAL_NORMAL, v))
    _, s, V, _ = svd_of(A, algorithm, k, p, v=v, Omega=Omega, transpose=transpose)
    return V, s * s


# ============================================================ Algorithms 4 and 5

def nystrom_tevd(A, p, l, v, Omega):
    """Alg. 4 — modified prolonged (Nystrom) TEVD of the normal matrix J^* J, v >= 2 views
    (P:274-297).  J = A.  Omega replaces line 2's / Alg. 3's randn: n_c x (p+l) for even v
    (Q_r built from J), n_r x (p+l) for odd v (Q_r built from J^*, line 6).
    Returns (V_p, Lambda_p^2) with J^* J ~ V_p diag(Lambda_p^2) V_p^*.

    Readings: ||Y_r|| in line 9 is the spectral norm; tsvd(F, p) of the wide
    F (line 13) is the exact rank-p truncated SVD."""
    if v < 2:
        raise ValueError("Alg. 4 needs v >= 2 (P:277)")
    J = _f64(A)
    if v == 2:                                    # lines 1-2
        Qr = orth(_f64(Omega))
    elif v % 2 == 0:                              # lines 3-4: QrQc(J, p, l, v-2) -> Q_r
        Qr = qrqc(J, p, l, v - 2, Omega)
    else:                                         # lines 5-6: QrQc(J^*, p, l, v-2) -> its Q_c
        Qr = qrqc(J, p, l, v - 2, Omega, transpose=True)
    Yr = J.T @ (J @ Qr)                           # line 8 (two views)
    nu = 2.2e-16 * np.linalg.norm(Yr, 2)          # line 9
    Yr = Yr + nu * Qr                             # line 10
    B = Qr.T @ Yr                                 # line 11
    CL = chol_lower((B + B.T) / 2.0)              # line 12
    F = np.linalg.solve(CL, Yr.T)                 # line 13: F = C_L^-1 Y_r^*
    _, lam_hat, Vp = tsvd(F, p)                   # line 14
    lam2 = lam_hat ** 2 - nu                      # line 15
    lam2[lam2 < 0] = 0.0
    return Vp, lam2


def pinched_tevd(A, p, l, v, Omega):
    """Alg. 5 — modified pinched TEVD of J^* J, v >= 2 views.  J = A.
    Omega: n_r x (p+l) for even v (Q_r = QrQc(J^*, v-1), line 2), n_c x (p+l) for odd v
    (Q_r = QrQc(J, v-1), line 4).  Returns (V_p, Lambda_p^2)."""
    if v < 2:
        raise ValueError("Alg. 5 needs v >= 2")
    J = _f64(A)
    if v % 2 == 0:
        Qr = qrqc(J, p, l, v - 1, Omega, transpose=True)   # odd v-1 on J^*: its Q_c
    else:
        Qr = qrqc(J, p, l, v - 1, Omega)                   # even v-1 on J: Q_r
    Bc = J @ Qr                                            # line 6 (one view)
    evals, evecs = np.linalg.eigh(Bc.T @ Bc)               # line 7: tevd, descending
    order = np.argsort(evals)[::-1][:p]
    lam2 = np.maximum(evals[order], 0.0)
    return Qr @ evecs[:, order], lam2                      # line 8


def views_and_vectors(algorithm, v, width):
    """(views, matrix-vector products) of each algorithm: Alg. 2 uses v views and
    v (p+l) vectors; Alg. 9 uses v views and (v + floor(v/2) - 1)(p+l) vectors; Alg. 7 one view
    (its two sketches are counted as vectors l + l2 by the caller)."""
    if algorithm == "subspace":
        return v, v * width
    if algorithm == "krylov":
        return v, (v + v // 2 - 1) * width
    raise ValueError(algorithm)


# ============================================================ error metrics

def rel_frobenius_error(A, Ahat, p):
    """||A - Ahat||_F / ||A - [[A]]_p||_F - 1."""
    A = _f64(A)
    s = np.linalg.svd(A, compute_uv=False)
    return np.linalg.norm(A - Ahat) / np.sqrt(np.sum(s[p:] ** 2)) - 1.0


def rel_spectral_error(A, Ahat, p):
    """||A - Ahat|| / ||A - [[A]]_p|| - 1."""
    A = _f64(A)
    s = np.linalg.svd(A, compute_uv=False)
    return np.linalg.norm(A - Ahat, 2) / s[p] - 1.0


def projector_distance(U, Uo):
    """||U U^T - Uo Uo^T||_F computed stably as sqrt(2) ||U - Uo (Uo^T U)||_F for U, Uo with
    orthonormal columns of equal count (SURVEY c-14): sign- and rotation-invariant."""
    U = _f64(U)
    Uo = _f64(Uo)
    return float(np.sqrt(2.0) * np.linalg.norm(U - Uo @ (Uo.T @ U)))


def residual_fro(A, U, s, V, panel=4096):
    """||A - U diag(s) V^T||_F by an explicit pass over A (row panels)."""
    A = np.asarray(A)
    U = _f64(U)
    V = _f64(V)
    tot = 0.0
    for r0 in range(0, A.shape[0], panel):
        r1 = min(A.shape[0], r0 + panel)
        D = _f64(A[r0:r1]) - (U[r0:r1] * s) @ V.T
        tot += float(np.sum(D * D))
    return float(np.sqrt(tot))


# ============================================================ theory checks

def half_power_lhs_rhs(A, Qr, q):
    """Thm A.1: ||A (I - Q_r Q_r^*)||^{2q} <= ||(A^*A)^q (I - Q_r Q_r^*)||.
    Returns (lhs, rhs)."""
    A = _f64(A)
    P = np.eye(A.shape[1]) - Qr @ Qr.T
    lhs = np.linalg.norm(A @ P, 2) ** (2 * q)
    AtA = A.T @ A
    rhs = np.linalg.norm(np.linalg.matrix_power(AtA, q) @ P, 2)
    return lhs, rhs


def thm_bound(sig, p, l, e):
    """Right-hand side of Thm 3.1 / 4.1 and the even/odd bounds (P:110-118, P:182-190,
    P:210-243) with exponent e (= 2q+1, 2q, v-1 or v):
    [ (1 + sqrt(p/(l-1))) sig_{p+1}^e + e_const sqrt(p+l)/l (sum_{j>p} sig_j^{2e})^{1/2} ]^{1/e}."""
    sig = _f64(sig)
    t1 = (1.0 + np.sqrt(p / (l - 1.0))) * sig[p] ** e
    t2 = np.e * np.sqrt(p + l) / l * np.sqrt(np.sum(sig[p:] ** (2 * e)))
    return (t1 + t2) ** (1.0 / e)
