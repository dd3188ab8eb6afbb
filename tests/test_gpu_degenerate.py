"""Degenerate and boundary inputs through the C ABI (GPU): the zero matrix, a rank-1 spike,
k = 1 / p = 0, a single row or column, the smallest admissible l2 and lc = 0.  Each is checked
against its closed form (and, where one exists, the oracle) and for finite outputs."""
import numpy as np
import pytest
import torch

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_1804_07531_b200 import build, rsvd

    build.build()
    c = rsvd.Context(0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def cm(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().t()


def host(t):
    return t.detach().cpu().numpy()


def run(ctx, alg, A, k, p, v, Om, Phi=None, l2=None, lc=-1):
    if alg == "subspace":
        return ctx.subspace(dev(A), k, p, v, cm(Om))
    if alg == "krylov":
        return ctx.block_krylov(dev(A), k, p, v, cm(Om))
    return ctx.single_pass(dev(A), k, p, l2, cm(Om), cm(Phi), lc=lc)


ALGS = [("subspace", 2), ("subspace", 3), ("krylov", 4), ("single_pass", 1)]


@pytest.mark.parametrize("alg,v", ALGS)
def test_zero_matrix(ctx, alg, v):
    """A = 0: every sketch is zero, every pivot is rank deficient, sigma = 0 exactly, no NaN."""
    m, n, k, p = 300, 200, 5, 5
    A = np.zeros((m, n))
    Om = S.random_gaussian_matrix(n, k + p, seed=1)
    Phi = S.random_gaussian_matrix(m, 2 * (k + p), seed=2)
    U, s, V, info = run(ctx, alg, A, k, p, v, Om, Phi, 2 * (k + p))
    U, s, V = host(U), host(s), host(V)
    assert np.all(s == 0.0)
    assert np.all(np.isfinite(U)) and np.all(np.isfinite(V))
    assert info.rank_deficient_cols > 0


@pytest.mark.parametrize("alg,v", ALGS)
def test_rank_one_spike(ctx, alg, v):
    """A = 3 e_i e_j^T: sigma = (3, 0, ...), U_1 = +-e_i, V_1 = +-e_j (rank 1 < l: guard path)."""
    m, n, k, p = 257, 131, 3, 2
    A = np.zeros((m, n))
    A[100, 40] = 3.0
    Om = S.random_gaussian_matrix(n, k + p, seed=3)
    Phi = S.random_gaussian_matrix(m, 2 * (k + p), seed=4)
    U, s, V, _ = run(ctx, alg, A, k, p, v, Om, Phi, 2 * (k + p))
    U, s, V = host(U), host(s), host(V)
    np.testing.assert_allclose(s[0], 3.0, rtol=1e-14)
    assert np.all(np.abs(s[1:]) <= 1e-13)
    assert abs(abs(U[100, 0]) - 1.0) <= 1e-13 and abs(abs(V[40, 0]) - 1.0) <= 1e-13


@pytest.mark.parametrize("alg,v", ALGS)
def test_k1_p0_matches_oracle(ctx, alg, v):
    cfg = S.CONFIGS["C1"]
    A = S.make_matrix(cfg)
    Om = S.gaussian_test_matrix(A.shape[1], 1, cfg, S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(A.shape[0], 1, cfg, S.ROLE_PHI)
    U, s, V, _ = run(ctx, alg, A, 1, 0, v, Om, Phi, 1)
    Uo, so, Vo, _ = O.svd_of(A, alg, 1, 0, v=v, Omega=Om, l2=1, Phi=Phi)
    assert abs(host(s)[0] - so[0]) <= 1e-10 * so[0]
    assert O.projector_distance(host(U), Uo) <= 1e-9 and O.projector_distance(host(V), Vo) <= 1e-9


@pytest.mark.parametrize("shape", [(1, 50), (50, 1), (1, 1)])
@pytest.mark.parametrize("alg,v", [("subspace", 2), ("subspace", 3), ("single_pass", 1)])
def test_single_row_or_column(ctx, shape, alg, v):
    """m = 1 or n = 1 (l = 1 = min(m, n)): sigma = ||A||, U = +-1 / V = +-A / ||A||."""
    A = S.random_gaussian_matrix(*shape, seed=7)
    Om = S.random_gaussian_matrix(shape[1], 1, seed=8)
    Phi = S.random_gaussian_matrix(shape[0], 1, seed=9)
    U, s, V, _ = run(ctx, alg, A, 1, 0, v, Om, Phi, 1)
    np.testing.assert_allclose(host(s)[0], np.linalg.norm(A), rtol=1e-13)
    Uh, Vh = np.abs(host(U)[:, 0]), np.abs(host(V)[:, 0])
    nrm = np.linalg.norm(A)
    Ue = np.abs(A[:, 0]) / nrm if shape[1] == 1 else np.ones(1)
    Ve = np.abs(A[0]) / nrm if shape[0] == 1 else np.ones(1)
    np.testing.assert_allclose(Uh, Ue, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(Vh, Ve, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("lc", [0, 5, 10])
def test_single_pass_min_l2_and_lc(ctx, lc):
    """l2 = l (the smallest admissible co-range sketch) and the lc range ends, vs oracle."""
    cfg = S.CONFIGS["C2"]
    A = S.make_matrix(cfg, 1500, 1300)
    Om = S.gaussian_test_matrix(A.shape[1], cfg.l, cfg, S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(A.shape[0], cfg.l, cfg, S.ROLE_PHI)
    U, s, V, info = run(ctx, "single_pass", A, cfg.k, cfg.p, 1, Om, Phi, cfg.l, lc=lc)
    Uo, so, Vo, _ = O.svd_of(A, "single_pass", cfg.k, cfg.p, Omega=Om, l2=cfg.l, lc=lc, Phi=Phi)
    assert info.lc_used == lc
    assert np.max(np.abs(host(s) - so) / so) <= 1e-10
    assert O.projector_distance(host(U), Uo) <= 1e-9 and O.projector_distance(host(V), Vo) <= 1e-9


@pytest.mark.parametrize("alg,v", ALGS)
def test_fp32_zero_and_rank_one(ctx, alg, v):
    """The fp32 path (tcgen05 3xTF32 views, fp64 in between): A = 0 gives sigma = 0 exactly and
    finite vectors; a rank-1 spike gives sigma_1 = 3 and U_1 = +-e_i, V_1 = +-e_j (fp32 tolerances)."""
    m, n, k, p = 300, 200, 5, 5
    Om = S.random_gaussian_matrix(n, k + p, seed=31).astype(np.float32)
    Phi = S.random_gaussian_matrix(m, 2 * (k + p), seed=32).astype(np.float32)
    A = np.zeros((m, n), dtype=np.float32)
    U, s, V, _ = run(ctx, alg, A, k, p, v, Om, Phi, 2 * (k + p))
    assert np.all(host(s) == 0.0) and np.all(np.isfinite(host(U))) and np.all(np.isfinite(host(V)))
    A[123, 45] = 3.0
    U, s, V, _ = run(ctx, alg, A, k, p, v, Om, Phi, 2 * (k + p))
    s, U, V = host(s).astype(np.float64), host(U).astype(np.float64), host(V).astype(np.float64)
    assert abs(s[0] - 3.0) <= 1e-5 * 3.0 and np.all(np.abs(s[1:]) <= 1e-5)
    assert abs(abs(U[123, 0]) - 1.0) <= 1e-5 and abs(abs(V[45, 0]) - 1.0) <= 1e-5


@pytest.mark.parametrize("variant", ["row", "bwz", "bwz2"])
def test_new_paths_zero_and_rank_one(ctx, variant):
    """The row-wise pass and the extended sketch on A = 0 (sigma = 0 exactly, finite vectors) and on
    a rank-1 spike (sigma = (3, 0, ...), U_1 = +-e_i, V_1 = +-e_j)."""
    m, n, k, p = 300, 200, 5, 5
    Om = S.random_gaussian_matrix(n, k + p, seed=51)
    Phi = S.random_gaussian_matrix(m, 2 * (k + p), seed=52)
    Xr, Xc = S.srft_matrix(m, 30, 53), S.srft_matrix(n, 30, 54)

    def call(A):
        if variant == "row":
            return ctx.row_stream(dev(A), k, p, cm(Om))
        return ctx.single_pass_extended(dev(A), k, p, 2 * (k + p), 30, cm(Om), cm(Phi), cm(Xr), cm(Xc),
                                        variant=variant)

    A = np.zeros((m, n))
    U, s, V, _ = call(A)
    assert np.all(host(s) == 0.0) and np.all(np.isfinite(host(U))) and np.all(np.isfinite(host(V)))
    A[77, 123] = 3.0
    U, s, V, _ = call(A)
    s, U, V = host(s), host(U), host(V)
    np.testing.assert_allclose(s[0], 3.0, rtol=1e-14)
    assert np.all(np.abs(s[1:]) <= 1e-13)
    assert abs(abs(U[77, 0]) - 1.0) <= 1e-13 and abs(abs(V[123, 0]) - 1.0) <= 1e-13
