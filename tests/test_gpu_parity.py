"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded bytes.

Tolerances (BASELINE.json north_star, fp64): singular values 1e-10 relative; projectors
||UU^T - UoUo^T||_F <= 1e-9; residual ||A - U S V^T||_F within 1e-8 relative of the oracle's.
Integer-valued inputs make every view exact in fp64, so views are compared bit for bit.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu

TOL_S, TOL_P, TOL_R = 1e-10, 1e-9, 1e-8


@pytest.fixture(scope="module")
def ctx():
    from paper_1804_07531_b200 import build, rsvd

    build.build()
    c = rsvd.Context(0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.asarray(a)).cuda()


def colmajor_dev(a):
    """numpy (rows, w) -> CUDA tensor in column-major layout."""
    t = torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda()
    return t.t()


def host(t):
    return t.detach().cpu().numpy()


def check_svd(U, s, V, Uo, so, Vo, A=None, k=None):
    U, s, V = host(U), host(s), host(V)
    rel = np.max(np.abs(s - so) / np.abs(so))
    assert rel <= TOL_S, f"sigma rel err {rel:.3e}"
    pu, pv = O.projector_distance(U, Uo), O.projector_distance(V, Vo)
    assert pu <= TOL_P, f"P_U err {pu:.3e}"
    assert pv <= TOL_P, f"P_V err {pv:.3e}"
    if A is not None:
        r, ro = O.residual_fro(A, U, s, V), O.residual_fro(A, Uo, so, Vo)
        assert abs(r - ro) <= TOL_R * ro + 1e-300, f"residual {r:.6e} vs {ro:.6e}"
    return rel, pu, pv


# ------------------------------------------------------------------ views: bit-exact on integers

VIEW_SHAPES = [(1037, 777), (200, 200), (64, 2000), (3000, 96), (129, 129)]
VIEW_WIDTHS = [1, 7, 20, 30, 64, 70, 100, 120, 128, 140, 200]


@pytest.mark.parametrize("shape", VIEW_SHAPES)
@pytest.mark.parametrize("w", VIEW_WIDTHS)
@pytest.mark.parametrize("trans", [0, 1])
def test_view_bit_exact(ctx, shape, w, trans):
    m, n = shape
    A = S.integer_matrix(m, n, -8, 8, seed=m + n)
    X = S.integer_matrix(m if trans else n, w, -8, 8, seed=w, order="F")
    Y, info = ctx.view(dev(A), colmajor_dev(X), trans=bool(trans))
    ref = (A.T @ X) if trans else (A @ X)
    assert np.array_equal(host(Y), ref)
    assert info.view_launches == (w + 127) // 128


@pytest.mark.parametrize("shape", [(1037, 777), (200, 200), (4000, 64), (96, 3000)])
@pytest.mark.parametrize("l,l2", [(20, 40), (30, 60), (70, 140), (8, 8), (5, 77)])
def test_fused_view_bit_exact(ctx, shape, l, l2):
    m, n = shape
    if l > n or l2 > m:
        pytest.skip("sketch wider than the matrix")
    A = S.integer_matrix(m, n, -8, 8, seed=3 * m + n)
    Om = S.integer_matrix(n, l, -8, 8, seed=l, order="F")
    Phi = S.integer_matrix(m, l2, -8, 8, seed=1000 + l2, order="F")
    Yc, Yr, info = ctx.view_fused(dev(A), colmajor_dev(Om), colmajor_dev(Phi))
    assert np.array_equal(host(Yc), A @ Om)
    assert np.array_equal(host(Yr), A.T @ Phi)
    assert info.view_launches == 1


# ------------------------------------------------------------------ orth and core SVD

@pytest.mark.parametrize("rows,w", [(4000, 30), (1037, 20), (200000, 8), (777, 128), (5000, 160), (40, 40),
                                    (3000, 200), (5000, 250), (2000, 500),
                                    # cluster path: ragged rows (16-row chunks padded), the largest
                                    # W = 64 block it holds (16 x 272 rows) and one row more (other path)
                                    (3001, 30), (4000, 60), (4352, 64), (4353, 64)])
def test_orth_cholqr2(ctx, rows, w):
    Y = S.random_gaussian_matrix(rows, w, seed=rows + w) * np.logspace(0, -3, w)
    Q, R, info = ctx.orth(colmajor_dev(Y))
    Q, R = host(Q), host(R)
    np.testing.assert_allclose(Q.T @ Q, np.eye(w), atol=5e-14 * np.sqrt(w))
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) >= 0)
    assert np.linalg.norm(Q @ R - Y) <= 1e-13 * np.linalg.norm(Y)
    Qo, Ro = O.qr(Y)
    assert np.linalg.norm(R - Ro) <= 1e-11 * np.linalg.norm(Ro)
    assert info.rank_deficient_cols == 0


@pytest.mark.parametrize("rows,w", [(4000, 30), (4000, 60), (3001, 20), (777, 128), (5000, 250)])
def test_orth_shifted_cholqr3(ctx, rows, w):
    """Shifted CholeskyQR3 (the Krylov blocks' orthonormalisation) on an ill-conditioned block
    (kappa ~ 1e10, beyond CholeskyQR2): Q orthonormal, Y = Q R, and R upper triangular with exact
    zeros below the diagonal (R = R_2 R_1 R_0 is formed by a tiled product in the cluster kernel)."""
    from paper_1804_07531_b200 import rsvd

    Y = S.random_gaussian_matrix(rows, w, seed=rows + 3 * w) * np.logspace(0, -10, w)
    Q, R, info = ctx.orth(colmajor_dev(Y), flags=rsvd.RSVD_ORTH_SHIFTED)
    Q, R = host(Q), host(R)
    np.testing.assert_allclose(Q.T @ Q, np.eye(w), atol=5e-14 * np.sqrt(w))
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) >= 0)
    assert np.linalg.norm(Q @ R - Y) <= 1e-13 * np.linalg.norm(Y)
    Qo, Ro = O.qr(Y)
    # the trailing columns of an ill-conditioned block carry R entries known only to u * kappa
    # relative to ||Y||: compare R column by column against the oracle's Householder R
    assert np.linalg.norm(R - Ro) <= 1e-12 * np.linalg.norm(Ro)


@pytest.mark.parametrize("w,r", [(24, 17), (30, 21), (60, 43), (250, 201)])
def test_orth_rank_deficient(ctx, w, r):
    """Exactly rank-r input: the guarded Cholesky zeroes l - r columns; the kept Q spans range(Y)."""
    rows = 3000
    X, _ = S.exact_rank_factors(rows, w, r, seed=4)
    Y = X @ S.random_gaussian_matrix(r, w, seed=5)
    Q, R, info = ctx.orth(colmajor_dev(Y))
    Q = host(Q)
    kept = np.linalg.norm(Q, axis=0) > 0.5
    # the guard drops at least most of the w - r dependent columns (a column whose Gram pivot sits
    # at the Gram's rounding level, ~rows*u, may survive as an orthonormal noise direction, as a
    # Householder QR would keep all w); the kept Q is orthonormal and contains range(Y) = range(X)
    assert r <= kept.sum() <= r + 2 and info.rank_deficient_cols >= w - r - 2
    Qk = Q[:, kept]
    np.testing.assert_allclose(Qk.T @ Qk, np.eye(kept.sum()), atol=1e-12)
    assert np.linalg.norm(X - Qk @ (Qk.T @ X)) < 1e-10


@pytest.mark.parametrize("w", [2, 3, 20, 30, 64, 70, 120, 140, 160, 200, 250, 301, 500])
def test_core_svd_jacobi(ctx, w):
    Mx = np.triu(S.random_gaussian_matrix(w, w, seed=w)) * np.logspace(0, -4, w)[None, :]
    U, s, V, info = ctx.core_svd(colmajor_dev(Mx))
    U, s, V = host(U), host(s), host(V)
    so = np.linalg.svd(Mx, compute_uv=False)
    np.testing.assert_allclose(s, so, rtol=1e-12, atol=1e-15 * so[0])
    assert np.linalg.norm((U * s) @ V.T - Mx) <= 1e-13 * np.linalg.norm(Mx)
    np.testing.assert_allclose(V.T @ V, np.eye(w), atol=1e-13)
    assert 1 <= info.jacobi_sweeps < (30 if w <= 256 else 50)  # random graded triu, no QR preconditioning


def test_core_svd_golden(ctx):
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "micro_cases.json")))["svd_perm_diag"]
    U, s, V, _ = ctx.core_svd(colmajor_dev(np.array(g["M"])))
    np.testing.assert_allclose(host(s), g["sigma"], rtol=1e-15)


# ------------------------------------------------------------------ algorithms vs oracle

def cfg_inputs(name, m=None, n=None, transpose=False):
    cfg = S.CONFIGS[name]
    A = S.make_matrix(cfg, m, n)
    mm, nn = A.shape
    Om = S.gaussian_test_matrix(mm if transpose else nn, cfg.l, cfg, S.ROLE_OMEGA_M if transpose else S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(mm, cfg.l2, cfg, S.ROLE_PHI)
    return cfg, A, Om, Phi


SUBSPACE_CASES = [("C1", None, None, v) for v in (2, 3, 4)] + [("C2", None, None, v) for v in (2, 3, 4, 5, 6)] + \
                 [("C3", 3000, 1200, v) for v in (2, 3, 4, 5)] + [("C1", 333, 151, 3), ("C2", 1500, 4100, 4)]


@pytest.mark.parametrize("name,m,n,v", SUBSPACE_CASES)
def test_subspace_parity(ctx, name, m, n, v):
    cfg, A, Om, _ = cfg_inputs(name, m, n)
    U, s, V, info = ctx.subspace(dev(A), cfg.k, cfg.p, v, colmajor_dev(Om))
    Uo, so, Vo, op = O.svd_of(A, "subspace", cfg.k, cfg.p, v=v, Omega=Om)
    check_svd(U, s, V, Uo, so, Vo, A)
    assert info.views == v == op.views and info.vectors == op.vectors


KRYLOV_CASES = [("C1", None, None, v) for v in (2, 3, 4)] + [("C2", None, None, v) for v in (3, 4, 5)] + \
               [("C3", 3000, 1200, v) for v in (2, 3, 4, 5)]


@pytest.mark.parametrize("name,m,n,v", KRYLOV_CASES)
def test_block_krylov_parity(ctx, name, m, n, v):
    cfg, A, Om, _ = cfg_inputs(name, m, n)
    U, s, V, info = ctx.block_krylov(dev(A), cfg.k, cfg.p, v, colmajor_dev(Om))
    Uo, so, Vo, op = O.svd_of(A, "krylov", cfg.k, cfg.p, v=v, Omega=Om)
    check_svd(U, s, V, Uo, so, Vo, A)
    assert info.views == v and info.vectors == op.vectors


@pytest.mark.parametrize("name,m,n", [("C1", None, None), ("C2", None, None), ("C3", 3000, 1200), ("C1", 517, 203)])
@pytest.mark.parametrize("lc", [None, 0, 5])
def test_single_pass_parity(ctx, name, m, n, lc):
    cfg, A, Om, Phi = cfg_inputs(name, m, n)
    lcv = cfg.p if lc is None else lc
    U, s, V, info = ctx.single_pass(dev(A), cfg.k, cfg.p, cfg.l2, colmajor_dev(Om), colmajor_dev(Phi),
                                    lc=-1 if lc is None else lc)
    Uo, so, Vo, _ = O.svd_of(A, "single_pass", cfg.k, cfg.p, Omega=Om, l2=cfg.l2, lc=lcv, Phi=Phi)
    check_svd(U, s, V, Uo, so, Vo, A)
    assert info.views == 1 and info.view_launches == 1 and info.lc_used == lcv


@pytest.mark.parametrize("alg,v", [("subspace", 2), ("subspace", 3), ("krylov", 4), ("krylov", 5), ("subspace", 5)])
def test_transposed_input_parity(ctx, alg, v):
    cfg, A, Om, _ = cfg_inputs("C2", 1500, 2600, transpose=True)
    fn = ctx.subspace if alg == "subspace" else ctx.block_krylov
    U, s, V, _ = fn(dev(A), cfg.k, cfg.p, v, colmajor_dev(Om), input=1)
    Uo, so, Vo, _ = O.svd_of(A, alg, cfg.k, cfg.p, v=v, Omega=Om, transpose=True)
    check_svd(U, s, V, Uo, so, Vo, A)


@pytest.mark.parametrize("v", [2, 3, 4, 5])
def test_normal_mode_parity(ctx, v):
    """A^T A ~ V S^2 V^T in the recommended orientation."""
    from paper_1804_07531_b200 import rsvd

    inp = rsvd.recommend_input(rsvd.RSVD_GOAL_NORMAL, v)
    cfg, A, Om, _ = cfg_inputs("C1", transpose=bool(inp))
    _, s2, V, _ = ctx.subspace(dev(A), cfg.k, cfg.p, v, colmajor_dev(Om), input=inp, flags=rsvd.RSVD_SQUARED)
    Vo, s2o = O.normal_matrix_tevd(A, cfg.k, cfg.p, v, Om)
    np.testing.assert_allclose(host(s2), s2o, rtol=2 * TOL_S)
    assert O.projector_distance(host(V), Vo) <= TOL_P


@pytest.mark.parametrize("alg,v", [("subspace", 2), ("subspace", 3), ("krylov", 4), ("single_pass", 1)])
def test_exact_rank_recovery_gpu(ctx, alg, v):
    """Rank-r input with r < l: the sketches are exactly rank deficient (guarded Cholesky path),
    and sigma, U, V of the rank-k truncation are recovered exactly (P1)."""
    m, n, k, p, r = 900, 700, 8, 8, 12
    sig = np.linspace(4.0, 1.0, r)
    A = S.exact_rank_matrix(m, n, sig, seed=7)
    X, Y = S.exact_rank_factors(m, n, r, seed=7)
    Om = S.gaussian((n, k + p), 90, S.ROLE_OMEGA)
    Phi = S.gaussian((m, 2 * (k + p)), 90, S.ROLE_PHI)
    if alg == "single_pass":
        U, s, V, info = ctx.single_pass(dev(A), k, p, 2 * (k + p), colmajor_dev(Om), colmajor_dev(Phi))
    else:
        fn = ctx.subspace if alg == "subspace" else ctx.block_krylov
        U, s, V, info = fn(dev(A), k, p, v, colmajor_dev(Om))
    np.testing.assert_allclose(host(s), sig[:k], rtol=1e-12)
    assert O.projector_distance(host(U), X[:, :k]) < 1e-10
    assert O.projector_distance(host(V), Y[:, :k]) < 1e-10
    assert info.rank_deficient_cols > 0


def test_diagonal_structured_omega_gpu(ctx):
    """A = diag(d), Omega = I[:, :l]: sigma = d[:k] and U = V = I[:, :k] (P2)."""
    n, k, p = 300, 6, 4
    d = np.linspace(3.0, 0.5, n) ** 2
    A = np.diag(d)
    Om = np.asfortranarray(np.eye(n)[:, :k + p])
    E = np.eye(n)[:, :k]
    for fn in (ctx.subspace, ctx.block_krylov):
        for v in (2, 3, 4):
            U, s, V, _ = fn(dev(A), k, p, v, colmajor_dev(Om))
            np.testing.assert_allclose(host(s), d[:k], rtol=4e-16)
            np.testing.assert_allclose(np.abs(host(U)), E, atol=1e-15)
            np.testing.assert_allclose(np.abs(host(V)), E, atol=1e-15)


def test_full_sampling_equals_exact_svd(ctx):
    m, n, k = 150, 40, 10
    A = S.random_gaussian_matrix(m, n, seed=1)
    Om = S.gaussian((n, n), 91, S.ROLE_OMEGA)
    U, s, V, _ = ctx.subspace(dev(A), k, n - k, 2, colmajor_dev(Om))
    Uj, sj, Vj = O.jacobi_svd(A)
    np.testing.assert_allclose(host(s), sj[:k], rtol=1e-12)
    assert O.projector_distance(host(U), Uj[:, :k]) < 1e-11


# ------------------------------------------------------------------ plumbing

def test_graph_replay_and_no_graph_bitwise(ctx):
    from paper_1804_07531_b200 import rsvd

    cfg, A, Om, Phi = cfg_inputs("C2", 2000, 1800)
    Ad, Omd = dev(A), colmajor_dev(Om)
    r1 = ctx.subspace(Ad, cfg.k, cfg.p, 4, Omd)
    r2 = ctx.subspace(Ad, cfg.k, cfg.p, 4, Omd)
    r3 = ctx.subspace(Ad, cfg.k, cfg.p, 4, Omd, flags=rsvd.RSVD_NO_GRAPH)
    assert r2[3].graph_replayed == 1
    for a, b, c in zip(r1[:3], r2[:3], r3[:3]):
        assert torch.equal(a, b) and torch.equal(a, c)


def test_host_pointers(ctx):
    """Host (CPU) arguments are staged by the library; results equal the device-pointer call."""
    cfg, A, Om, Phi = cfg_inputs("C1")
    Ud, sd, Vd, _ = ctx.subspace(dev(A), cfg.k, cfg.p, 3, colmajor_dev(Om))
    Ah = torch.from_numpy(A).pin_memory()
    Omh = torch.from_numpy(np.ascontiguousarray(Om.T)).t()
    Uh, sh, Vh, info = ctx.subspace(Ah, cfg.k, cfg.p, 3, Omh)
    assert info.host_staged == 1
    assert torch.equal(Uh, Ud.cpu()) and torch.equal(sh, sd.cpu()) and torch.equal(Vh, Vd.cpu())
    Uh2, sh2, Vh2, _ = ctx.subspace(Ah, cfg.k, cfg.p, 3, Omh)   # graph replay with host staging
    assert torch.equal(Uh2, Ud.cpu())


def test_argument_errors(ctx):
    from paper_1804_07531_b200 import rsvd

    A = dev(np.zeros((50, 40)))
    Om = colmajor_dev(np.zeros((40, 10)))
    with pytest.raises(rsvd.RsvdError) as e:
        ctx.subspace(A, 5, 5, 1, Om)            # v < 2
    assert e.value.code == -1
    with pytest.raises(rsvd.RsvdError):
        ctx.subspace(A, 30, 20, 2, colmajor_dev(np.zeros((40, 50))))  # l > min(m, n)
    with pytest.raises(rsvd.RsvdError):
        ctx.single_pass(A, 5, 5, 8, Om, colmajor_dev(np.zeros((50, 8))))  # l2 < l
    with pytest.raises(rsvd.RsvdError) as e:
        ctx.subspace(dev(np.zeros((50, 40), dtype=np.float16)), 5, 5, 2, colmajor_dev(np.zeros((40, 10), np.float16)))
    assert e.value.code == -2  # only fp64 and fp32 are defined


# ------------------------------------------------------------------ Alg. 4 / Alg. 5 (normal matrix)

NORMAL_CASES = [("C1", None, None, v) for v in (2, 3, 4, 5)] + [("C2", None, None, v) for v in (2, 3, 4)] + \
               [("C3", 3000, 1200, 3), ("C1", 333, 151, 4)]


@pytest.mark.parametrize("name,m,n,v", NORMAL_CASES)
@pytest.mark.parametrize("alg", ["nystrom", "pinched"])
def test_normal_matrix_parity(ctx, alg, name, m, n, v):
    cfg = S.CONFIGS[name]
    A = S.make_matrix(cfg, m, n)
    mm, nn = A.shape
    from_At = (v % 2 == 1) if alg == "nystrom" else (v % 2 == 0)
    Om = S.gaussian_test_matrix(mm if from_At else nn, cfg.l, cfg, S.ROLE_OMEGA)
    fn = ctx.nystrom if alg == "nystrom" else ctx.pinched
    s2, V, info = fn(dev(A), cfg.k, cfg.p, v, colmajor_dev(Om))
    ofn = O.nystrom_tevd if alg == "nystrom" else O.pinched_tevd
    Vo, s2o = ofn(A, cfg.k, cfg.p, v, Om)
    s2 = host(s2)
    assert info.views == v
    assert np.max(np.abs(s2 - s2o) / s2o) <= 2 * TOL_S  # eigenvalues = sigma^2: twice sigma's relative error
    assert O.projector_distance(host(V), Vo) <= TOL_P


@pytest.mark.parametrize("shape", [(0, 40), (50, 0), (0, 0)])
def test_empty_matrix_rejected(ctx, shape):
    """An empty A is an argument error (RSVD_E_ARG, -1) for every entry point, never a crash."""
    from paper_1804_07531_b200 import rsvd

    m, n = shape
    A = torch.zeros(m, n, dtype=torch.float64, device="cuda")
    Om = colmajor_dev(np.zeros((max(n, 1), 2)))
    Phi = colmajor_dev(np.zeros((max(m, 1), 4)))
    Xi = colmajor_dev(np.zeros((max(m, n, 1), 4)))
    calls = [lambda: ctx.subspace(A, 1, 1, 2, Om), lambda: ctx.block_krylov(A, 1, 1, 3, Om),
             lambda: ctx.single_pass(A, 1, 1, 4, Om, Phi), lambda: ctx.row_stream(A, 1, 1, Om),
             lambda: ctx.single_pass_extended(A, 1, 1, 2, 4, Om, Phi, Xi, Xi),
             lambda: ctx.nystrom(A, 1, 1, 2, Om)]
    for fn in calls:
        with pytest.raises(rsvd.RsvdError) as e:
            fn()
        assert e.value.code == -1


def test_invalid_rank_rejected(ctx):
    from paper_1804_07531_b200 import rsvd

    A = dev(np.ones((50, 40)))
    Om = colmajor_dev(np.zeros((40, 10)))
    for k, p in ((0, 5), (-1, 5), (5, -1)):
        with pytest.raises(rsvd.RsvdError) as e:
            ctx.subspace(A, k, p, 2, Om)
        assert e.value.code == -1


# ------------------------------------------------------------------ cluster Cholesky (k_chol_cl)
# 64 < w <= 512: one 32-column panel per CTA; ragged last panels (w = 65: a 1-column panel),
# the largest cluster (w = 512, 16 CTAs) and the near-identity second pass all go through it.
@pytest.mark.parametrize("rows,w", [(2000, 65), (3000, 96), (3000, 97), (4000, 129), (5000, 255), (5000, 256),
                                    (5000, 257), (6000, 511), (6000, 512)])
def test_orth_cluster_cholesky_widths(ctx, rows, w):
    Y = S.random_gaussian_matrix(rows, w, seed=7 * w + rows) * np.logspace(0, -4, w)
    Q, R, info = ctx.orth(colmajor_dev(Y))
    Q, R = host(Q), host(R)
    np.testing.assert_allclose(Q.T @ Q, np.eye(w), atol=5e-14 * np.sqrt(w))
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) > 0)
    assert np.linalg.norm(Q @ R - Y) <= 1e-13 * np.linalg.norm(Y)
    Qo, Ro = O.qr(Y)
    assert np.linalg.norm(R - Ro) <= 1e-11 * np.linalg.norm(Ro)
    assert info.rank_deficient_cols == 0


@pytest.mark.parametrize("w,r", [(97, 61), (300, 190), (512, 333)])
def test_orth_cluster_cholesky_rank_deficient(ctx, w, r):
    """The guard inside the cluster kernel's register-resident diagonal factorisation: deficient
    pivots in every panel position zero their row of R and their column of R^-1 (reading R10)."""
    rows = 3000
    X, _ = S.exact_rank_factors(rows, w, r, seed=11)
    Y = X @ S.random_gaussian_matrix(r, w, seed=12)
    Q, R, info = ctx.orth(colmajor_dev(Y))
    Q, R = host(Q), host(R)
    kept = np.linalg.norm(Q, axis=0) > 0.5
    assert r <= kept.sum() <= r + 2 and info.rank_deficient_cols >= w - r - 2
    assert np.all(np.abs(R[~kept]).max(axis=1) == 0)      # rows of dropped pivots are exactly zero
    Qk = Q[:, kept]
    np.testing.assert_allclose(Qk.T @ Qk, np.eye(kept.sum()), atol=1e-12)
    assert np.linalg.norm(X - Qk @ (Qk.T @ X)) < 1e-10


@pytest.mark.parametrize("rows,w", [(5000, 300), (6000, 500)])
def test_orth_cluster_cholesky_shifted(ctx, rows, w):
    """Shifted CholeskyQR3 through the cluster kernel (shift pass + two guarded passes), kappa ~ 1e10."""
    from paper_1804_07531_b200 import rsvd

    Y = S.random_gaussian_matrix(rows, w, seed=rows + 5 * w) * np.logspace(0, -10, w)
    Q, R, info = ctx.orth(colmajor_dev(Y), flags=rsvd.RSVD_ORTH_SHIFTED)
    Q, R = host(Q), host(R)
    np.testing.assert_allclose(Q.T @ Q, np.eye(w), atol=5e-14 * np.sqrt(w))
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) >= 0)
    assert np.linalg.norm(Q @ R - Y) <= 1e-13 * np.linalg.norm(Y)
    Qo, Ro = O.qr(Y)
    assert np.linalg.norm(R - Ro) <= 1e-12 * np.linalg.norm(Ro)
