"""Pins for the CPU oracle (-m "not gpu").

Each test ties the oracle to something other than itself: worked values (tests/golden), closed
forms, exact identities stated by the paper, brute force at full sampling, the paper's
inequalities, or an independent route to the same quantity.  Citations are PAPER.md lines (P:).
"""
import json
import os

import numpy as np
import pytest
from scipy.sparse.linalg import LinearOperator, eigsh

import oracle as O
import synth as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "micro_cases.json")))


def proj(U, Uo):
    return O.projector_distance(U, Uo)


def spec_norm_resid(A, Q, side):
    """|| A - Q Q^T A || (side='c') or || A - A Q Q^T || (side='r') by Lanczos on the Gram op."""
    if side == "c":
        R = A - Q @ (Q.T @ A)
    else:
        R = A - (A @ Q) @ Q.T
    n = R.shape[1]
    op = LinearOperator((n, n), matvec=lambda x: R.T @ (R @ x), dtype=np.float64)
    w = eigsh(op, k=1, which="LA", tol=1e-10, return_eigenvectors=False)
    return float(np.sqrt(max(w[0], 0.0)))


# ------------------------------------------------------------------ golden micro cases

def test_golden_qr():
    g = GOLD["qr_3_4"]
    Q, R = O.qr(np.array(g["M"]))
    np.testing.assert_allclose(Q, g["Q"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(R, g["R"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("case", ["svd_perm_diag", "svd_diag_3_1"])
def test_golden_svd(case):
    g = GOLD[case]
    M = np.array(g["M"])
    for U, s, V in (O.tsvd(M, 2), O.jacobi_svd(M)):
        np.testing.assert_allclose(s, g["sigma"], rtol=0, atol=1e-15)
        np.testing.assert_allclose((U * s) @ V.T, M, atol=1e-15)
        if "U_abs" in g:
            np.testing.assert_allclose(np.abs(U), g["U_abs"], atol=1e-15)
            np.testing.assert_allclose(np.abs(V), g["V_abs"], atol=1e-15)


def test_golden_chol():
    g = GOLD["chol_4_2_5"]
    np.testing.assert_allclose(O.chol_lower(np.array(g["S"])), g["L"], atol=1e-15)


def test_golden_diag_full_sampling():
    g = GOLD["diag_54321_rank2"]
    A = np.diag(g["d"])
    Om = S.gaussian((5, g["p"] + g["l"]), 9, S.ROLE_OMEGA)
    for v in (2, 3, 4):
        _, s, _ = O.gen_subspace_iteration(A, g["p"], g["l"], v, Om)
        np.testing.assert_allclose(s, g["sigma"], rtol=1e-13)
    _, s, _ = O.std_subspace_iteration(A, g["p"], g["l"], 1, Om)
    np.testing.assert_allclose(s, g["sigma"], rtol=1e-13)


# ------------------------------------------------------------------ P3 orthonormality / QR contract

@pytest.mark.parametrize("shape", [(50, 10), (300, 40), (17, 17)])
def test_qr_contract(shape):
    M = S.random_gaussian_matrix(*shape, seed=shape[0])
    Q, R = O.qr(M)
    assert Q.shape == shape and R.shape == (shape[1], shape[1])
    np.testing.assert_allclose(Q.T @ Q, np.eye(shape[1]), atol=1e-14)
    assert np.all(np.tril(R, -1) == 0.0)
    assert np.all(np.diag(R) >= 0.0)
    assert np.linalg.norm(Q @ R - M) <= 1e-14 * np.linalg.norm(M)


def test_chol_reconstruct():
    G = S.random_gaussian_matrix(6, 6, seed=3)
    Sm = G.T @ G + np.eye(6)
    L = O.chol_lower(Sm)
    assert np.allclose(np.triu(L, 1), 0)
    assert np.linalg.norm(L @ L.T - Sm) <= 1e-13 * np.linalg.norm(Sm)


def test_jacobi_svd_closed_form():
    """Jacobi SVD of U diag(d) V^T returns d (known spectrum) and the same subspaces."""
    d = np.array([7.0, 3.0, 2.5, 1.0, 0.5, 1e-3])
    A = S.exact_rank_matrix(9, 6, d, seed=1)
    U, s, V = O.jacobi_svd(A)
    np.testing.assert_allclose(s, d, rtol=1e-13, atol=1e-14 * d[0])  # A itself carries eps*||A|| rounding
    X, Y = S.exact_rank_factors(9, 6, 6, seed=1)
    # the sigma=1e-3 direction moves by ~eps*||A||/sigma_6 ~ 1e-12 under A's own rounding
    assert proj(U, X) < 1e-11 and proj(V, Y) < 1e-11


def test_jacobi_matches_eigensolve():
    """sigma(M)^2 = eig(M^T M): brute-force symmetric eigensolve (S:75 oracle)."""
    M = S.random_gaussian_matrix(8, 6, seed=5)
    _, s, _ = O.jacobi_svd(M)
    ev = np.sort(np.linalg.eigvalsh(M.T @ M))[::-1]
    np.testing.assert_allclose(s ** 2, ev, rtol=1e-12)
    _, s2, _ = O.jacobi_svd(M.T)
    np.testing.assert_allclose(s, s2, rtol=1e-13)


# ------------------------------------------------------------------ P5 brute force on tiny inputs

ALGS = [("subspace", 2), ("subspace", 3), ("subspace", 4), ("subspace", 5),
        ("krylov", 2), ("krylov", 3), ("krylov", 4), ("krylov", 5)]


@pytest.mark.parametrize("shape", [(12, 9), (9, 12), (10, 10)])
@pytest.mark.parametrize("alg,v", ALGS)
def test_full_sampling_equals_full_svd(shape, alg, v):
    """l = min(m,n): the sketch spans the whole (co-)range, so the randomized TSVD equals the
    exact TSVD, computed here by the oracle's own Jacobi (independent of LAPACK).  Krylov with
    widths > min(m,n) is skipped (qr needs rows >= cols)."""
    m, n = shape
    N = min(m, n)
    k = 3
    A = S.random_gaussian_matrix(m, n, seed=m * 100 + n)
    Om = S.gaussian((n, N), 11, S.ROLE_OMEGA)
    if alg == "krylov":
        kw = (v // 2) * N if v % 2 == 0 else ((v - 1) // 2) * N
        if kw > N:
            pytest.skip("Krylov basis wider than the space")
    U, s, V, _ = O.svd_of(A, alg, k, N - k, v=v, Omega=Om)
    Uj, sj, Vj = O.jacobi_svd(A)
    np.testing.assert_allclose(s, sj[:k], rtol=1e-12)
    assert proj(U, Uj[:, :k]) < 1e-11
    assert proj(V, Vj[:, :k]) < 1e-11


def test_single_pass_full_sampling():
    m, n, k = 12, 10, 3
    A = S.random_gaussian_matrix(m, n, seed=77)
    Om = S.gaussian((n, n), 12, S.ROLE_OMEGA)
    Phi = S.gaussian((m, m), 12, S.ROLE_PHI)
    U, s, V, _ = O.svd_of(A, "single_pass", k, n - k, Omega=Om, l2=m, Phi=Phi)
    Uj, sj, Vj = O.jacobi_svd(A)
    np.testing.assert_allclose(s, sj[:k], rtol=1e-11)
    assert proj(U, Uj[:, :k]) < 1e-10 and proj(V, Vj[:, :k]) < 1e-10


# ------------------------------------------------------------------ P1 exact rank-r recovery

@pytest.mark.parametrize("alg,v", ALGS + [("single_pass", 1)])
@pytest.mark.parametrize("r_is", ["k", "l"])
def test_exact_rank_recovery(alg, v, r_is):
    m, n, k, p = 120, 90, 5, 5
    l = k + p
    r = k if r_is == "k" else l
    sig = np.linspace(3.0, 1.0, r) * np.array([1.0 + 0.1 * i for i in range(r)])[::-1] / 2.0
    sig = np.sort(sig)[::-1]
    A = S.exact_rank_matrix(m, n, sig, seed=r)
    X, Y = S.exact_rank_factors(m, n, r, seed=r)
    Om = S.gaussian((n, l), 20 + r, S.ROLE_OMEGA)
    Phi = S.gaussian((m, 2 * l), 20 + r, S.ROLE_PHI)
    U, s, V, _ = O.svd_of(A, alg, k, p, v=v, Omega=Om, l2=2 * l, Phi=Phi)
    np.testing.assert_allclose(s, sig[:k], rtol=1e-12)
    assert proj(U, X[:, :k]) < 1e-11 and proj(V, Y[:, :k]) < 1e-11
    res = O.residual_fro(A, U, s, V)
    floor = np.sqrt(np.sum(sig[k:] ** 2))
    assert abs(res - floor) <= 1e-12 * np.linalg.norm(sig)


# ------------------------------------------------------------------ P2 diagonal closed forms

def test_diagonal_structured_omega_exact():
    """A = diag(d), Omega = I[:, :l]: every sketch is diag(d)[:, :l], every Q = I[:, :l], every
    R = diag(d_1..d_l): sigma = d[:k] and U = V = I[:, :k] (up to sign) in every algorithm."""
    n, k, p = 40, 4, 3
    l = k + p
    d = S.paper_poly(n, R=1, rho=1.5)[::-1].copy()[::-1]  # strictly decreasing
    d = np.sort(d)[::-1] * np.linspace(1.0, 0.5, n)
    A = np.diag(d)
    Om = np.eye(n)[:, :l]
    Phi = np.eye(n)[:, :2 * l]
    E = np.eye(n)[:, :k]
    for alg, v in ALGS + [("single_pass", 1)]:
        U, s, V, _ = O.svd_of(A, alg, k, p, v=v, Omega=Om, l2=2 * l, Phi=Phi)
        np.testing.assert_allclose(s, d[:k], rtol=2e-16, atol=0)
        np.testing.assert_allclose(np.abs(U), E, atol=1e-15)
        np.testing.assert_allclose(np.abs(V), E, atol=1e-15)


@pytest.mark.parametrize("spec", ["polyfast", "polyslow", "expslow", "expfast"])
@pytest.mark.parametrize("v", [2, 3, 4])
def test_eckart_young_floor(spec, v):
    """||A - U S V^T||_F >= sqrt(sum_{i>p} d_i^2) (optimality of [[A]]_p), on the paper's
    diagonal test matrices, n = 300, R = 10, p = l = 10 (P:1014 setting)."""
    n = 300
    d = {"polyfast": S.paper_poly(n, 10, 2.0), "polyslow": S.paper_poly(n, 10, 1.0),
         "expslow": S.paper_exp(n, 10, 0.25), "expfast": S.paper_exp(n, 10, 1.0)}[spec]
    A = np.diag(d)
    Om = S.gaussian((n, 20), 30, S.ROLE_OMEGA, v)
    U, s, V, _ = O.svd_of(A, "subspace", 10, 10, v=v, Omega=Om)
    floor = np.sqrt(np.sum(d[10:] ** 2))
    assert O.residual_fro(A, U, s, V) >= floor - 1e-12
    assert np.all(s <= d[:10] + 1e-14)   # Ritz values never exceed the true singular values


# ------------------------------------------------------------------ P4 identities and counts

@pytest.mark.parametrize("q", [0, 1, 2])
def test_alg2_even_equals_alg1(q):
    """Alg. 2 with v = 2(q+1) IS Alg. 1 with q iterations: bitwise."""
    cfg = S.CONFIGS["C1"]
    A = S.make_matrix(cfg)
    Om = S.gaussian_test_matrix(cfg.n, cfg.l, cfg, S.ROLE_OMEGA)
    U1, s1, V1 = O.std_subspace_iteration(A, cfg.k, cfg.p, q, Om)
    U2, s2, V2 = O.gen_subspace_iteration(A, cfg.k, cfg.p, 2 * (q + 1), Om)
    assert np.array_equal(s1, s2) and np.array_equal(U1, U2) and np.array_equal(V1, V2)


@pytest.mark.parametrize("v", [2, 3])
def test_alg9_equals_alg2_below_4(v):
    """Alg. 9 'is the same as Alg. 2 for v < 4': bitwise."""
    cfg = S.CONFIGS["C1"]
    A = S.make_matrix(cfg)
    Om = S.gaussian_test_matrix(cfg.n, cfg.l, cfg, S.ROLE_OMEGA)
    a = O.gen_subspace_iteration(A, cfg.k, cfg.p, v, Om)
    b = O.gen_block_krylov(A, cfg.k, cfg.p, v, Om)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("v", [2, 3, 4, 5, 6])
def test_view_and_vector_counts(v):
    """Alg. 2: v views, v(p+l) vectors; Alg. 9: v views, (v + floor(v/2) - 1)(p+l) vectors."""
    A = S.random_gaussian_matrix(80, 60, seed=v)
    w = 6
    Om = S.gaussian((60, w), 40, S.ROLE_OMEGA)
    _, _, _, op = O.svd_of(A, "subspace", 3, 3, v=v, Omega=Om)
    assert (op.views, op.vectors) == O.views_and_vectors("subspace", v, w) == (v, v * w)
    _, _, _, op = O.svd_of(A, "krylov", 3, 3, v=v, Omega=Om)
    assert (op.views, op.vectors) == O.views_and_vectors("krylov", v, w) == (v, (v + v // 2 - 1) * w)
    Phi = S.gaussian((80, 2 * w), 40, S.ROLE_PHI)
    _, _, _, op = O.svd_of(A, "single_pass", 3, 3, Omega=Om, l2=2 * w, Phi=Phi)
    assert op.views == 1 and op.vectors == 3 * w


@pytest.mark.parametrize("trial", range(20))
def test_half_power_inequality(trial):
    """Thm A.1 holds deterministically for ANY orthonormal Q_r and q >= 1."""
    m, n = 30, 20
    A = S.random_gaussian_matrix(m, n, seed=500 + trial) * np.linspace(2.0, 0.1, n)
    Qr = np.linalg.qr(S.random_gaussian_matrix(n, 5, seed=600 + trial))[0]
    for q in (1, 2, 3):
        lhs, rhs = O.half_power_lhs_rhs(A, Qr, q)
        assert lhs <= rhs * (1 + 1e-10)


def test_half_power_on_alg_basis():
    """Thm A.1 with the Q_r Alg. 3 actually produces (v = 2q views)."""
    A = np.diag(S.paper_poly(200, 10, 1.0))
    for q in (1, 2):
        Om = S.gaussian((200, 12), 41, S.ROLE_OMEGA, q)
        Qr = O.qrqc(A, 6, 6, 2 * q, Om)
        lhs, rhs = O.half_power_lhs_rhs(A, Qr, q)
        assert lhs <= rhs * (1 + 1e-10)


# ------------------------------------------------------------------ statistical (Thm 3.1/4.1, Fig. 2/5 trends)

def _mean_errors(A, v, trials, p=10, l=10, alg="subspace"):
    ec, er = [], []
    n = A.shape[1]
    for t in range(trials):
        Om = S.gaussian((n, p + l), 50, S.ROLE_OMEGA, v, t)
        if alg == "subspace":
            (_, _, _), (Qc, Qr) = _bases_subspace(A, p, l, v, Om)
        else:
            _, (Qc, Qr) = O.gen_block_krylov(A, p, l, v, Om, return_basis=True)
        ec.append(spec_norm_resid(A, Qc, "c"))
        er.append(spec_norm_resid(A, Qr, "r"))
    return float(np.mean(ec)), float(np.mean(er))


def _bases_subspace(A, p, l, v, Om):
    Qr = Om
    Qc = None
    for j in range(1, v + 1):
        if j % 2:
            Qc = O.qr(A @ Qr)[0]
        else:
            Qr = O.qr(A.T @ Qc)[0]
    return (None, None, None), (Qc, Qr)


@pytest.mark.parametrize("name", ["polyslow", "lowrankmed"])
def test_expected_error_bounds_and_monotone(name):
    """Means over 20 calls of ||A - Q_c Q_c^* A|| and ||A - A Q_r Q_r^*|| lie below the
    even/odd-view bounds (Thm 3.1/4.1) and decrease with v (Fig. 2).
    Paper setting: n = 1000, R = 10, target rank p = 10, oversampling l = 10."""
    n, p, l = 1000, 10, 10
    if name == "polyslow":
        d = S.paper_poly(n, 10, 1.0)
        A = np.diag(d)
    else:
        A = S.paper_lowrank_noise(n, 10, 1e-2)
        d = np.linalg.svd(A, compute_uv=False)
    prev = None
    for v in (2, 3, 4, 5):
        mc, mr = _mean_errors(A, v, trials=20)
        ec, er = (v - 1, v) if v % 2 == 0 else (v, v - 1)
        assert mc <= O.thm_bound(d, p, l, ec)
        assert mr <= O.thm_bound(d, p, l, er)
        cur = max(mc, mr)
        if prev is not None:
            assert cur <= prev * 1.0001
        prev = cur
        # a (p+l)-dimensional basis never beats [[A]]_{p+l}: error >= sigma_{p+l+1}
        assert mc >= d[p + l] * (1 - 1e-9) and mr >= d[p + l] * (1 - 1e-9)


def test_krylov_beats_subspace_at_fixed_views():
    """'for fixed oversampling and views the block Krylov method is more accurate'."""
    n = 1000
    A = np.diag(S.paper_poly(n, 10, 1.0))
    for v in (4, 5):
        s_sub = _mean_errors(A, v, 10)
        s_kry = _mean_errors(A, v, 10, alg="krylov")
        assert max(s_kry) <= max(s_sub)


# ------------------------------------------------------------------ P6 single pass specifics

def test_single_pass_baseline_is_least_squares():
    """With l_c = l_1, Alg. 7 lines 11-12 compute X = (Omega_c^* Q_c)^dagger Y_r^* (P:595):
    check against the pseudo-inverse route (independent of the qr-based solve)."""
    cfg = S.CONFIGS["C1"]
    A = S.make_matrix(cfg)
    Om = S.gaussian_test_matrix(cfg.n, cfg.l, cfg, S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(cfg.m, cfg.l2, cfg, S.ROLE_PHI)
    U, s, V, _ = O.svd_of(A, "single_pass", cfg.k, cfg.p, Omega=Om, l2=cfg.l2, Phi=Phi)
    Yc, Yr = A @ Om, A.T @ Phi
    Qc = np.linalg.svd(Yc, full_matrices=False)[0]       # any orthonormal basis of range(Y_c)
    X = np.linalg.pinv(Phi.T @ Qc) @ Yr.T
    Ux, sx, Vtx = np.linalg.svd(X, full_matrices=False)
    np.testing.assert_allclose(s, sx[:cfg.k], rtol=1e-11)
    assert proj(U, Qc @ Ux[:, :cfg.k]) < 1e-10
    assert proj(V, Vtx[:cfg.k].T) < 1e-10


def test_single_pass_lc_truncation_is_tsvd_of_Yc():
    """l_c < l_1: Q_c = Q_c Qhat_c equals the p+l_c leading left singular vectors of Y_c."""
    m, n, p, l1, lc = 150, 120, 6, 6, 2
    A = S.random_gaussian_matrix(m, n, seed=8) * np.linspace(3, 0.01, n)
    Om = S.gaussian((n, p + l1), 60, S.ROLE_OMEGA)
    Yc = A @ Om
    Qc, Rc = O.qr(Yc)
    Qh, _, _ = O.tsvd(Rc, p + lc)
    Uy = np.linalg.svd(Yc, full_matrices=False)[0][:, :p + lc]
    assert proj(Qc @ Qh, Uy) < 1e-12


# ------------------------------------------------------------------ P7 normal mode / orientation

@pytest.mark.parametrize("v", [2, 3, 4])
def test_normal_mode_full_sampling(v):
    """Full sampling: V diag(sigma^2) V^T = eig(A^T A) top-k (P:247, P:278 'EVD of J^*J')."""
    m, n, k = 14, 10, 4
    A = S.random_gaussian_matrix(m, n, seed=90 + v)
    Om = S.gaussian((n if v % 2 == 0 else m, n), 70, S.ROLE_OMEGA, v)
    V, s2 = O.normal_matrix_tevd(A, k, n - k, v, Om)
    ev, EV = np.linalg.eigh(A.T @ A)
    ev, EV = ev[::-1], EV[:, ::-1]
    np.testing.assert_allclose(s2, ev[:k], rtol=1e-12)
    assert proj(V, EV[:, :k]) < 1e-11


def test_recommend_input_table():
    """P:245-247 and P:897."""
    g = O
    assert [g.recommend_input(g.GOAL_NORMAL, v) for v in (2, 3, 4, 5)] == [0, 1, 0, 1]
    assert [g.recommend_input(g.GOAL_RIGHT, v) for v in (2, 3)] == [0, 1]
    assert [g.recommend_input(g.GOAL_LEFT, v) for v in (2, 3)] == [1, 0]
    assert g.recommend_input(g.GOAL_SVD, 3) == 0


@pytest.mark.parametrize("alg,v", [("subspace", 2), ("subspace", 3), ("krylov", 4), ("single_pass", 1)])
def test_transposed_input_returns_A_factors(alg, v):
    m, n, k, p = 70, 50, 4, 4
    sig = np.array([5.0, 4.0, 3.0, 2.0])
    A = S.exact_rank_matrix(m, n, sig, seed=33)
    X, Y = S.exact_rank_factors(m, n, 4, seed=33)
    Om = S.gaussian((m, k + p), 80, S.ROLE_OMEGA_M)
    Phi = S.gaussian((n, 2 * (k + p)), 80, S.ROLE_PHI)
    U, s, V, _ = O.svd_of(A, alg, k, p, v=v, Omega=Om, l2=2 * (k + p), Phi=Phi, transpose=True)
    np.testing.assert_allclose(s, sig, rtol=1e-12)
    assert U.shape == (m, k) and V.shape == (n, k)
    assert proj(U, X) < 1e-11 and proj(V, Y) < 1e-11


def test_argument_errors():
    A = np.eye(5)
    with pytest.raises(ValueError):
        O.gen_subspace_iteration(A, 2, 1, 1, np.eye(5)[:, :3])
    with pytest.raises(ValueError):
        O.gen_block_krylov(A, 2, 1, 1, np.eye(5)[:, :3])
    with pytest.raises(ValueError):
        O.one_view_tropp(A, 2, 2, 1, 0, np.eye(5)[:, :4], np.eye(5)[:, :3])


def test_projector_distance_stable_form():
    """sqrt(2)||U - Uo Uo^T U||_F equals the explicit ||UU^T - UoUo^T||_F."""
    U = np.linalg.qr(S.random_gaussian_matrix(30, 4, seed=1))[0]
    Uo = np.linalg.qr(U + 1e-3 * S.random_gaussian_matrix(30, 4, seed=2))[0]
    explicit = np.linalg.norm(U @ U.T - Uo @ Uo.T)
    assert abs(O.projector_distance(U, Uo) - explicit) < 1e-12


# ------------------------------------------------------------------ Alg. 4 (Nystrom) and Alg. 5 (pinched)

def _nys_inputs(v, pinched=False, seed=1):
    cfg = S.CONFIGS["C1"]
    A = S.make_matrix(cfg)
    # Alg. 4 builds Q_r from J for even v and from J^* for odd v; Alg. 5 the other way round
    from_At = (v % 2 == 0) if pinched else (v % 2 == 1)
    rows = A.shape[0] if from_At else A.shape[1]
    return cfg, A, S.gaussian_test_matrix(rows, cfg.l, cfg, S.ROLE_OMEGA, seed)


@pytest.mark.parametrize("v", [2, 3, 4, 5, 6])
def test_nystrom_equals_alg2_recommended(v):
    """P:365 (with P:343, eq. gennystrom2): Alg. 4 with v views is algebraically the recommended
    use of Alg. 2 for J^* J (input J for even v, J^* for odd v) — same Omega, same TEVD."""
    cfg, A, Om = _nys_inputs(v)
    V, lam2 = O.nystrom_tevd(A, cfg.k, cfg.p, v, Om)
    Vs, s2 = O.normal_matrix_tevd(A, cfg.k, cfg.p, v, Om)   # Alg. 2, recommended orientation
    assert np.max(np.abs(lam2 - s2) / s2) <= 1e-12
    assert proj(V, Vs) <= 1e-12


@pytest.mark.parametrize("v", [2, 3, 4, 5])
def test_pinched_equals_alg2_other_orientation(v):
    """Alg. 5 with v views equates to Alg. 2 for J^* J in the NON-recommended
    orientation (input J^* for even v, J for odd v)."""
    cfg, A, Om = _nys_inputs(v, pinched=True)
    V, lam2 = O.pinched_tevd(A, cfg.k, cfg.p, v, Om)
    Vs, s2 = O.normal_matrix_tevd(A, cfg.k, cfg.p, v, Om, transpose=(v % 2 == 0))
    assert np.max(np.abs(lam2 - s2) / s2) <= 1e-12
    assert proj(V, Vs) <= 1e-12


@pytest.mark.parametrize("v", [2, 3, 4])
def test_nystrom_exact_rank_and_full_sampling(v):
    """Exactly rank-r J (r <= p + l): the Nystrom TEVD recovers eig(J^* J) (the nu shift of
    P:289-296 is removed again in line 15).  Full sampling l = n: same, for any J."""
    sig = np.array([5.0, 3.0, 2.0, 1.5, 1.0, 0.5])
    A = S.exact_rank_matrix(60, 40, sig, seed=3)
    k, p = 4, 4
    Om = S.random_gaussian_matrix(60 if v % 2 else 40, k + p, seed=v)
    V, lam2 = O.nystrom_tevd(A, k, p, v, Om)
    np.testing.assert_allclose(lam2, sig[:k] ** 2, rtol=1e-12)
    X, Y = S.exact_rank_factors(60, 40, len(sig), seed=3)
    assert proj(V, Y[:, :k]) <= 1e-11
    B = S.random_gaussian_matrix(12, 9, seed=11)
    Om = S.random_gaussian_matrix(12 if v % 2 else 9, 9, seed=12)
    V, lam2 = O.nystrom_tevd(B, 9, 0, v, Om)
    ev = np.sort(np.linalg.eigvalsh(B.T @ B))[::-1]
    np.testing.assert_allclose(lam2, ev, rtol=1e-10, atol=1e-13 * ev[0])


def test_nystrom_more_accurate_than_pinched():
    """P:369 / section 'results normal matrix': with the same view budget the modified prolonged
    (Nystrom) TEVD is more accurate than the pinched one (mean over seeds, PolySlow-like decay)."""
    n = 120
    d = 1.0 / np.arange(1, n + 1) ** 0.5
    A = np.diag(d)
    k, p = 10, 5
    err_n, err_p = [], []
    for seed in range(20):
        for v in (2, 3):
            On = S.random_gaussian_matrix(n, k + p, seed=1000 + seed)
            V, lam2 = O.nystrom_tevd(A, k, p, v, On)
            Vp, lp = O.pinched_tevd(A, k, p, v, On)
            N = A.T @ A
            err_n.append(np.linalg.norm(N - (V * lam2) @ V.T, 2))
            err_p.append(np.linalg.norm(N - (Vp * lp) @ Vp.T, 2))
    assert np.mean(err_n) < np.mean(err_p)


# ---------------------------------------------------------------- f3: adaptive single pass

@pytest.mark.parametrize("plan,p,T,expect", [
    # hand evaluation of Eq. (overflat) P:610-618 at p=5, T=24:
    # sqrt(5*17*(1-2/23)) = 8.8096; -(p-1) -> 4.8096; *23/13 = 8.509 -> 8 - 5 = 3; l2 = 24-10-3 = 11
    ("flat", 5, 24, (3, 11)),
    ("flat", 5, 16, (2, 4)),        # max{2, .} floor
    ("decay", 5, 24, (2, 12)),      # max{2, floor(23/3) - 5 = 2}
    ("decay", 5, 40, (8, 22)),      # floor(39/3) - 5 = 8
    ("rapid", 5, 24, (6, 8)),       # floor(22/2) - 5 = 6
    ("rapid", 5, 16, (2, 4)),       # floor(14/2) - 5 = 2
])
def test_oversampling_plans_worked_values(plan, p, T, expect):
    f = {"flat": O.plan_flat, "decay": O.plan_decay, "rapid": O.plan_rapid}[plan]
    assert f(p, T) == expect
    l1, l2 = f(p, T)
    assert 0 <= l1 <= l2 and 2 * p + l1 + l2 == T


def test_oversampling_plans_invariants_and_errors():
    for p in range(1, 12):
        for T in range(2 * p + 6, 2 * p + 80):
            for f in (O.plan_flat, O.plan_decay, O.plan_rapid):
                l1, l2 = f(p, T)
                assert 2 <= l1 <= l2 and 2 * p + l1 + l2 == T
    # l1 = floor(T/2) - p = 7, l2 = 7, lc = floor(0.5 * 7) = 3   (Eq. lcutfixedratio)
    assert O.plan_balanced(5, 24, 0.5) == (7, 7, 3)
    assert O.plan_balanced(5, 24, 1.0)[2] == 7 and O.plan_balanced(5, 24, 0.0)[2] == 0
    with pytest.raises(ValueError):
        O.plan_flat(5, 15)


def test_minvar_select_hand_table():
    """Eq. (MinVar) on hand-made spectra (p = 2, l_1 = 3).
    s(0) = [1, 1, .5, .5]          -> unbiased var = 4 * (1/4)^2 / 3 = 1/12
    s(1) = [2, 2, 1, 1, 1, 1]      -> mean 4/3, sum sq dev = 2*(2/3)^2 + 4*(1/3)^2 = 4/3 -> /5 = 4/15
    s(2) = [1, 1, 1, 1, 1, 1]      -> 0   => l_c = 2."""
    lam = np.array([[4.0, 2.0], [2.0, 1.0], [2.0, 1.0], [2.0, 1.0]])
    lc, var = O.minvar_select(lam)
    assert lc == 2
    np.testing.assert_allclose(var, [1 / 12, 4 / 15, 0.0], atol=1e-15)
    # ties: all variances zero -> the smallest l_c (reading R19)
    lc, var = O.minvar_select(np.array([[2.0, 1.0]] * 4))
    assert lc == 0 and np.all(var == 0)
    # l_1 = 1: the only candidate is 0; l_1 = 0: l_c = 0 (empty range, reading R20)
    assert O.minvar_select(np.array([[3.0, 1.0], [1.0, 1.0]]))[0] == 0
    assert O.minvar_select(np.array([[3.0, 1.0]]))[0] == 0
    # zero spectra: 0/0 = 1, a/0 = inf -> that candidate is skipped (reading R20)
    lam = np.array([[1.0, 0.0], [1.0, 1.0], [1.0, 1.0], [1.0, 1.0]])
    lc, var = O.minvar_select(lam)
    # s(1) = [1, 0, 1, 1, 1, 1] (var 1/6), s(2) = ones (var 0)
    assert np.isinf(var[0]) and lc == 2 and abs(var[1] - 1 / 6) <= 1e-15


def test_minvar_spectra_equal_alg7_per_trial():
    """The trial spectra reuse one SVD of Y_c and slice Omega_c^* Q_c; each must equal
    the lambda of a full Alg. 7 run at that l_c (Alg. 7 lines 4-13, its own QR-then-TSVD path)."""
    cfg = S.CONFIGS["C2"]
    A = S.make_matrix(cfg, 600, 500)
    k, l1, l2 = 8, 6, 14
    Om = S.random_gaussian_matrix(500, k + l1, seed=11)
    Phi = S.random_gaussian_matrix(600, k + l2, seed=12)
    lam = O.minvar_spectra(A @ Om, A.T @ Phi, Phi, k, l1)
    for lc in range(l1 + 1):
        _, ref, _ = O.one_view_tropp(A, k, l1, l2, lc, Om, Phi)
        np.testing.assert_allclose(lam[lc], ref, rtol=1e-10)


def test_minvar_exact_rank_picks_zero():
    """Exactly rank r <= p: every trial recovers sigma(A) exactly, s(l_c) = 1, all variances ~0;
    the chosen l_c's output is exact."""
    rng = np.random.default_rng(3)
    X = np.linalg.qr(rng.standard_normal((300, 4)))[0]
    Y = np.linalg.qr(rng.standard_normal((200, 4)))[0]
    sig = np.array([5.0, 3.0, 2.0, 1.0])
    A = X @ np.diag(sig) @ Y.T
    Om = rng.standard_normal((200, 9))
    Phi = rng.standard_normal((300, 14))
    U, s, V, lc = O.one_view_minvar(A, 5, 4, 9, Om, Phi)
    lam = O.minvar_spectra(A @ Om, A.T @ Phi, Phi, 5, 4)
    np.testing.assert_allclose(lam[:, :4], np.tile(sig, (5, 1)), rtol=1e-10)
    np.testing.assert_allclose(s[:4], sig, rtol=1e-10)
    assert np.linalg.norm(A - (U * s) @ V.T) <= 1e-10 * np.linalg.norm(A)


def test_woolfe_equals_tropp_when_square():
    """l_c = l_1 = l_2: Q_r spans A^* Omega_c exactly, so Y_r^* Q_r Q_r^* = Y_r^* and Alg. 8's
    X_hat Q_r^* equals Alg. 7's X: identical rank-p approximations (P:696-713 vs P:660-682)."""
    cfg = S.CONFIGS["C2"]
    A = S.make_matrix(cfg, 400, 300)
    k, l1 = 6, 6
    Om = S.random_gaussian_matrix(300, k + l1, seed=21)
    Phi = S.random_gaussian_matrix(400, k + l1, seed=22)
    Uw, sw, Vw = O.one_view_woolfe(A, k, l1, l1, l1, Om, Phi)
    Ut, st, Vt = O.one_view_tropp(A, k, l1, l1, l1, Om, Phi)
    np.testing.assert_allclose(sw, st, rtol=1e-9)
    assert proj(Uw, Ut) <= 1e-8 and proj(Vw, Vt) <= 1e-8


def test_woolfe_exact_rank_and_orthonormal():
    rng = np.random.default_rng(5)
    X = np.linalg.qr(rng.standard_normal((250, 3)))[0]
    Y = np.linalg.qr(rng.standard_normal((180, 3)))[0]
    A = X @ np.diag([4.0, 2.0, 1.0]) @ Y.T
    U, s, V = O.one_view_woolfe(A, 3, 3, 6, 1, rng.standard_normal((180, 6)), rng.standard_normal((250, 9)))
    np.testing.assert_allclose(s, [4.0, 2.0, 1.0], rtol=1e-10)
    assert np.linalg.norm(A - (U * s) @ V.T) <= 1e-10 * np.linalg.norm(A)
    np.testing.assert_allclose(V.T @ V, np.eye(3), atol=1e-12)


# ---------------------------------------------------------------- f4: extended sketch (bwz / bwz2)

def test_srft_generator_orthonormal():
    """Phi = D F P with F the orthonormal DCT-II: orthonormal columns, and each
    column is a signed DCT basis vector (entries of modulus sqrt(2/n) cos(.) or sqrt(1/n))."""
    P = S.srft_matrix(64, 20, seed=1)
    np.testing.assert_allclose(P.T @ P, np.eye(20), atol=1e-14)
    # row k = 0 of the DCT-II matrix is the constant 1/sqrt(n) and D scales rows by +-1: with all
    # columns sampled, the first row of D F P has entries of modulus 1/8 (n = 64)
    P0 = S.srft_matrix(64, 64, seed=2)
    np.testing.assert_allclose(np.abs(P0[0, :]), np.full(64, 1 / 8), rtol=1e-14)


def test_plan_extended_worked_value_and_budget():
    # hand evaluation: l1 = l2 = floor(0.8 * 7) = 5; s(s+2) <= (24 - 21) * 2000 = 6000
    # -> s = 76 (76 * 78 = 5928, 77 * 79 = 6083)
    assert O.plan_extended(5, 24, 1000, 1000) == (5, 5, 76)
    prev = 0
    for T in range(16, 60):
        l1, l2, s = O.plan_extended(5, T, 1000, 1000)
        assert (2 * 5 + l1 + l2 + 1) * 2000 + s * (s + 2) <= T * 2000 < (2 * 5 + l1 + l2 + 1) * 2000 + (s + 1) * (s + 3)
        if l1 == O.plan_extended(5, max(16, T - 1), 1000, 1000)[0]:
            assert s >= prev
        prev = s
    with pytest.raises(ValueError):
        O.plan_extended(5, 15, 1000, 1000)


@pytest.mark.parametrize("variant", ["bwz", "bwz2"])
def test_extended_exact_rank_recovery(variant):
    """Exactly rank r <= p with s >= p + l1: Z, Y_c, Y_r capture A exactly, both estimators
    reproduce A (the rank-p truncation is the identity on an exact rank-p core)."""
    rng = np.random.default_rng(7)
    m, n, r, p, l1 = 300, 240, 4, 5, 5
    X = np.linalg.qr(rng.standard_normal((m, r)))[0]
    Y = np.linalg.qr(rng.standard_normal((n, r)))[0]
    A = X @ np.diag([4.0, 3.0, 2.0, 1.0]) @ Y.T
    Om_r = rng.standard_normal((n, p + l1))
    Om_c = rng.standard_normal((m, p + l1))
    s = 24
    U, lam, V = O.one_view_extended(A, p, l1, l1, Om_r, Om_c, S.srft_matrix(m, s, 3), S.srft_matrix(n, s, 4),
                                    variant=variant)
    np.testing.assert_allclose(lam[:4], [4.0, 3.0, 2.0, 1.0], rtol=1e-10)
    assert np.linalg.norm(A - (U * lam) @ V.T) <= 1e-10 * np.linalg.norm(A)


def test_extended_bwz2_at_least_as_accurate_on_average():
    """P:830 ('a more accurate low-rank approximation can be found'): mean relative Frobenius error
    of bwz2 <= that of bwz over 12 draws on a low-rank + noise matrix (p = 5, l1 = l2 = 5, s = 40)."""
    rng = np.random.default_rng(11)
    m, n, p, l1 = 400, 300, 5, 5
    X = np.linalg.qr(rng.standard_normal((m, 10)))[0]
    Y = np.linalg.qr(rng.standard_normal((n, 10)))[0]
    A = X @ np.diag(np.linspace(1, 0.5, 10)) @ Y.T + 0.02 * rng.standard_normal((m, n)) / np.sqrt(n)
    errs = {"bwz": [], "bwz2": []}
    for t in range(12):
        Om_r = rng.standard_normal((n, p + l1))
        Om_c = rng.standard_normal((m, p + l1))
        Pr, Pc = S.srft_matrix(m, 40, 100 + t), S.srft_matrix(n, 40, 200 + t)
        for v in errs:
            U, lam, V = O.one_view_extended(A, p, l1, l1, Om_r, Om_c, Pr, Pc, variant=v)
            errs[v].append(np.linalg.norm(A - (U * lam) @ V.T) / np.linalg.norm(A))
    assert np.mean(errs["bwz2"]) <= np.mean(errs["bwz"]) * 1.0001


# ---------------------------------------------------------------- f1: single pass over the rows

def test_row_stream_equals_two_view_alg2():
    """with R_c invertible, B^* = Yhat_r R_c^-1 = A^* Q_c, so the row-wise single pass gives
    the basic 2-view approximation (Alg. 2, v = 2) — an independent route (Alg. 2's two views)."""
    cfg = S.CONFIGS["C2"]
    A = S.make_matrix(cfg, 700, 500)
    Om = S.random_gaussian_matrix(500, 30, seed=41)
    U, lam, V = O.row_stream_qb(A, 20, 10, Om, panel_rows=64)
    Uo, lo, Vo = O.gen_subspace_iteration(A, 20, 10, 2, Om)
    np.testing.assert_allclose(lam, lo, rtol=1e-10)
    assert proj(U, Uo) <= 1e-9 and proj(V, Vo) <= 1e-9


def test_row_stream_order_and_panels_invariant():
    """Rows visited once in any order / any panel size: the sums are order-independent."""
    cfg = S.CONFIGS["C1"]
    A = S.make_matrix(cfg)
    Om = S.random_gaussian_matrix(A.shape[1], 20, seed=42)
    U1, l1, V1 = O.row_stream_qb(A, 10, 10, Om, panel_rows=1)
    perm = np.random.default_rng(3).permutation(A.shape[0])
    U2, l2, V2 = O.row_stream_qb(A, 10, 10, Om, panel_rows=7, order=perm)
    np.testing.assert_allclose(l1, l2, rtol=1e-12)
    assert proj(U1, U2) <= 1e-11 and proj(V1, V2) <= 1e-11


def test_row_stream_exact_rank_and_single_row():
    rng = np.random.default_rng(9)
    X = np.linalg.qr(rng.standard_normal((120, 3)))[0]
    Y = np.linalg.qr(rng.standard_normal((90, 3)))[0]
    A = X @ np.diag([3.0, 2.0, 1.0]) @ Y.T
    U, lam, V = O.row_stream_qb(A, 3, 4, rng.standard_normal((90, 7)), panel_rows=16)
    np.testing.assert_allclose(lam, [3.0, 2.0, 1.0], rtol=1e-10)
    assert np.linalg.norm(A - (U * lam) @ V.T) <= 1e-10 * np.linalg.norm(A)
    a = rng.standard_normal((1, 40))                      # single-row matrix: rank-1 exact
    U, lam, V = O.row_stream_qb(a, 1, 0, rng.standard_normal((40, 1)))
    np.testing.assert_allclose(lam[0], np.linalg.norm(a), rtol=1e-13)


# ------------------------------------------------------------------ Krylov-specific closed form

@pytest.mark.parametrize("v", [4, 5])
def test_krylov_recovers_rank_between_l_and_2l_exactly(v):
    """Exact rank r with l < r <= 2l and distinct sigma.  Alg. 9 at v = 4 builds
    K_c = [A Omega, (A A^*) A Omega] (2l columns), which spans range(A) for r <= 2l, so
    the final view and tsvd return the top-k triplets EXACTLY; at v = 5 K_r = [A^*A Omega,
    (A^*A)^2 Omega] spans the row space.  Alg. 2 at the same v keeps only l columns
    (< r), so it does NOT recover them: the test fails if the Krylov blocks are assembled wrongly
    (a missing raw last block, a block repeated, K taken on the wrong side)."""
    m, n, k, p = 150, 110, 6, 4
    l = k + p
    r = 2 * l - 3                                     # l < r <= 2l
    sig = 1.0 / np.arange(1, r + 1) ** 0.7             # distinct, slowly decaying
    A = S.exact_rank_matrix(m, n, sig, seed=77)
    X, Y = S.exact_rank_factors(m, n, r, seed=77)
    Om = S.gaussian((n, l), 77, S.ROLE_OMEGA, v)
    U, s, V = O.gen_block_krylov(A, k, p, v, Om)
    np.testing.assert_allclose(s, sig[:k], rtol=1e-11)
    assert proj(U, X[:, :k]) < 1e-10 and proj(V, Y[:, :k]) < 1e-10
    Us, ss, Vs = O.gen_subspace_iteration(A, k, p, v, Om)
    assert np.max(np.abs(ss - sig[:k]) / sig[:k]) > 1e-6      # Alg. 2: not exact at width l < r


# ------------------------------------------------------------------ error metrics

def test_relative_error_metrics_closed_form():
    """P:993-1001 on A = diag(d) with a known tail: the best rank-p approximation gives 0 for both
    metrics, and dropping the p-th direction gives the closed forms
    Frobenius: sqrt(sum_{i>=p} d_i^2) / sqrt(sum_{i>p} d_i^2) - 1,  spectral: d_p / d_{p+1} - 1."""
    d = np.array([5.0, 4.0, 3.0, 2.0, 1.5, 1.0, 0.5, 0.25])
    A = np.diag(d)
    p = 3
    best = np.diag(np.where(np.arange(8) < p, d, 0.0))
    assert abs(O.rel_frobenius_error(A, best, p)) < 1e-15
    assert abs(O.rel_spectral_error(A, best, p)) < 1e-15
    worse = np.diag(np.where(np.arange(8) < p - 1, d, 0.0))   # rank p-1
    tail_p, tail_p1 = np.sqrt(np.sum(d[p - 1:] ** 2)), np.sqrt(np.sum(d[p:] ** 2))
    assert abs(O.rel_frobenius_error(A, worse, p) - (tail_p / tail_p1 - 1.0)) < 1e-14
    assert abs(O.rel_spectral_error(A, worse, p) - (d[p - 1] / d[p] - 1.0)) < 1e-14
    # a rotated A has the same singular values: the metrics are unitarily invariant
    Q1, Q2 = O.qr(S.gaussian((8, 8), 5, S.ROLE_MISC))[0], O.qr(S.gaussian((8, 8), 6, S.ROLE_MISC))[0]
    assert abs(O.rel_frobenius_error(Q1 @ A @ Q2.T, Q1 @ worse @ Q2.T, p) - (tail_p / tail_p1 - 1.0)) < 1e-13


def test_thm_bound_limits():
    """Thm 3.1 / 4.1 right-hand side: it is never below the unavoidable
    error sigma_{p+1} (Eckart-Young), it tends to sigma_{p+1} as the exponent grows (the
    (.)^{1/e} root of a sum dominated by sigma_{p+1}^e), it is 0 for an exactly rank-p spectrum,
    and it grows with the tail."""
    sig = 1.0 / np.arange(1, 201) ** 1.0
    p, l = 10, 10
    for e in (1, 2, 3, 5, 9):
        assert O.thm_bound(sig, p, l, e) >= sig[p]
    assert abs(O.thm_bound(sig, p, l, 100) / sig[p] - 1.0) < 0.02   # (2 + ...)^(1/100) ~ 1.012
    assert O.thm_bound(np.r_[sig[:p], np.zeros(50)], p, l, 3) == 0.0
    heavier = sig.copy()
    heavier[p + 5:] *= 2.0
    assert O.thm_bound(heavier, p, l, 3) > O.thm_bound(sig, p, l, 3)


# ------------------------------------------------------------------ row-panel views

@pytest.mark.parametrize("alg,v,tr", [("subspace", 3, False), ("krylov", 4, False), ("krylov", 5, True),
                                      ("single_pass", 1, False)])
@pytest.mark.parametrize("panel", [7, 64, 10_000])
def test_panel_views_equal_dense_views(alg, v, tr, panel):
    """PanelOp evaluates A X panel by panel (same rows, same numbers) and A^* Y as a sum over
    panels: the algorithms' outputs equal the dense-operator oracle to rounding, and bitwise when
    one panel covers A (the full-size C4 / C5 parity tests use panels of a copied-back A)."""
    cfg = S.CONFIGS["C2"]
    A = S.make_matrix(cfg, 300, 220)
    m, n = A.shape
    Om = S.gaussian_test_matrix(m if tr else n, cfg.l, cfg, S.ROLE_OMEGA_M if tr else S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(m, cfg.l2, cfg, S.ROLE_PHI)
    a = O.svd_of(A, alg, cfg.k, cfg.p, v=v, Omega=Om, l2=cfg.l2, Phi=Phi, transpose=tr)
    b = O.svd_of(A, alg, cfg.k, cfg.p, v=v, Omega=Om, l2=cfg.l2, Phi=Phi, transpose=tr, panel_rows=panel)
    if panel >= m:
        for x, y in zip(a[:3], b[:3]):
            assert np.array_equal(x, y)
    np.testing.assert_allclose(b[1], a[1], rtol=1e-13)
    assert proj(b[0], a[0]) < 1e-12 and proj(b[2], a[2]) < 1e-12
    assert b[3].views == a[3].views and b[3].vectors == a[3].vectors
    # fp32 input: panels are upcast one by one, the same as upcasting A once
    A32 = A.astype(np.float32)
    c = O.svd_of(A32, alg, cfg.k, cfg.p, v=v, Omega=Om, l2=cfg.l2, Phi=Phi, transpose=tr, panel_rows=panel)
    d = O.svd_of(A32.astype(np.float64), alg, cfg.k, cfg.p, v=v, Omega=Om, l2=cfg.l2, Phi=Phi, transpose=tr)
    np.testing.assert_allclose(c[1], d[1], rtol=1e-13)


# ------------------------------------------------------------------ block Krylov read row wise

@pytest.mark.parametrize("v", [2, 3, 4, 5, 6, 7])
def test_row_block_krylov_equals_alg9(v):
    """The row-wise block Krylov (A^*A X in one pass over the rows) spans the same Krylov blocks as
    Alg. 9 with explicit views (P:941-943 vs P:907-923): same outputs to rounding, with
    (v-1)/2 + 1 passes for odd v (the co-range subspace with half the views) and v/2 + 1
    for even v."""
    cfg = S.CONFIGS["C2"]
    A = S.make_matrix(cfg, 400, 300)
    Om = S.gaussian_test_matrix(300, cfg.l, cfg, S.ROLE_OMEGA)
    (U, s, V), passes = O.row_block_krylov(A, cfg.k, cfg.p, v, Om, panel_rows=37)
    Uo, so, Vo = O.gen_block_krylov(A, cfg.k, cfg.p, v, Om)
    np.testing.assert_allclose(s, so, rtol=1e-11)
    assert proj(U, Uo) < 1e-9 and proj(V, Vo) < 1e-9
    assert passes == ((v - 1) // 2 + 1 if v % 2 else v // 2 + 1)


@pytest.mark.parametrize("v", [4, 5])
def test_row_block_krylov_exact_rank_and_order_invariance(v):
    """Exact rank l < r <= 2l recovered exactly (the Krylov closed form of
    test_krylov_recovers_rank_between_l_and_2l_exactly), and the panel size does not matter."""
    m, n, k, p = 150, 110, 6, 4
    l = k + p
    r = 2 * l - 3
    sig = 1.0 / np.arange(1, r + 1) ** 0.7
    A = S.exact_rank_matrix(m, n, sig, seed=78)
    X, Y = S.exact_rank_factors(m, n, r, seed=78)
    Om = S.gaussian((n, l), 78, S.ROLE_OMEGA, v)
    (U, s, V), _ = O.row_block_krylov(A, k, p, v, Om, panel_rows=1)
    np.testing.assert_allclose(s, sig[:k], rtol=1e-11)
    assert proj(U, X[:, :k]) < 1e-10 and proj(V, Y[:, :k]) < 1e-10
    (U2, s2, V2), _ = O.row_block_krylov(A, k, p, v, Om, panel_rows=1000)
    np.testing.assert_allclose(s2, s, rtol=1e-13)
