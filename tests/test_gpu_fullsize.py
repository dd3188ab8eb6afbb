"""Parity at BASELINE.json's full sizes (GPU, -m gpu).

C3 (fp64 20000 x 8000): element-wise against the oracle on the same bytes, in the launch
configuration bench.py uses (CUDA graphs).

C4 (fp64 50000 x 200000, 80 GB, built on the GPU with torch's generator — the oracle cannot hold
it): properties that hold at any size, checked by the oracle on sampled rows copied to the host:
  * Alg. 9 with odd v (= Alg. 2) ends with [Q_c, R_c] = qr(A Q_r) and tsvd(R_c), so
    A V = U diag(S) exactly (up to rounding): checked row by row, A[r, :] V = S * U[r, :], for
    sampled rows r (the oracle's own fp64 dot products);
  * U^T U = I, V^T V = I;
  * sigma_i(A) interlacing: the randomized sigma never exceeds the construction's
    (sigma_i + noise bound), and the top singular values match the construction
    sigma_i = i^-1.5 to the noise level 1e-8 (||G|| <~ sqrt(m) + sqrt(n));
  * the normal-matrix mode returns S^2 of the same triplets;
  * the single pass (its core is a least-squares estimate, not a projection): orthonormal
    factors and leading values near the construction; its parity with the oracle is checked on
    the same recipe and widths at 5000 x 20000 (test_c4_recipe_scaled_vs_oracle).
"""
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


def host(t):
    return t.detach().cpu().numpy()


def colmajor_dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().t()


# ------------------------------------------------------------------ C3 at full size vs the oracle
@pytest.fixture(scope="module")
def c3():
    cfg = S.CONFIGS["C3"]
    A = S.make_matrix(cfg)
    Om = S.gaussian_test_matrix(cfg.n, cfg.l, cfg, S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(cfg.m, cfg.l2, cfg, S.ROLE_PHI)
    return cfg, A, torch.from_numpy(A).cuda(), Om, Phi


@pytest.mark.parametrize("alg,v", [("subspace", 2), ("subspace", 3), ("subspace", 5), ("krylov", 4),
                                   ("krylov", 5), ("single_pass", 1)])
def test_c3_full_size_parity(ctx, c3, alg, v):
    cfg, A, Ad, Om, Phi = c3
    if alg == "subspace":
        U, s, V, info = ctx.subspace(Ad, cfg.k, cfg.p, v, colmajor_dev(Om))
    elif alg == "krylov":
        U, s, V, info = ctx.block_krylov(Ad, cfg.k, cfg.p, v, colmajor_dev(Om))
    else:
        U, s, V, info = ctx.single_pass(Ad, cfg.k, cfg.p, cfg.l2, colmajor_dev(Om), colmajor_dev(Phi))
    Uo, so, Vo, _ = O.svd_of(A, alg, cfg.k, cfg.p, v=v, Omega=Om, l2=cfg.l2, Phi=Phi)
    U, s, V = host(U), host(s), host(V)
    assert np.max(np.abs(s - so) / so) <= 1e-10
    assert O.projector_distance(U, Uo) <= 1e-9
    assert O.projector_distance(V, Vo) <= 1e-9
    r, ro = O.residual_fro(A, U, s, V), O.residual_fro(A, Uo, so, Vo)
    assert abs(r - ro) <= 1e-8 * ro


# ------------------------------------------------------------------ C4 at full size (80 GB)
@pytest.fixture(scope="module")
def c4():
    free, _ = torch.cuda.mem_get_info()
    if free < 110e9:
        pytest.skip(f"C4 needs ~110 GB of free device memory, have {free / 1e9:.0f}")
    cfg = S.CONFIGS["C4"]
    A = S.make_matrix_torch(cfg, torch.device("cuda", 0), panel_rows=2048)
    Om = S.gaussian_test_matrix_torch(cfg.n, cfg.l, cfg, S.ROLE_OMEGA, torch.device("cuda", 0))
    Omm = S.gaussian_test_matrix_torch(cfg.m, cfg.l, cfg, S.ROLE_OMEGA_M, torch.device("cuda", 0))
    Phi = S.gaussian_test_matrix_torch(cfg.m, cfg.l2, cfg, S.ROLE_PHI, torch.device("cuda", 0))
    torch.cuda.synchronize()
    yield cfg, A, Om, Omm, Phi
    del A
    torch.cuda.empty_cache()


def _sampled_rows(A, rows):
    return np.stack([A[r].cpu().numpy() for r in rows])


def _check_c4_triplets(cfg, A, U, s, V, exact_av):
    U, s, V = host(U), host(s), host(V)
    k = cfg.k
    np.testing.assert_allclose(U.T @ U, np.eye(k), atol=1e-12)
    np.testing.assert_allclose(V.T @ V, np.eye(k), atol=1e-12)
    assert np.all(np.diff(s) <= 0)
    sig = S.sigma_c4(cfg.rank)[:k]
    noise = cfg.noise * (np.sqrt(cfg.m) + np.sqrt(cfg.n)) * 1.1
    if exact_av:
        # projection methods: Ritz values never exceed sigma_i(A), top ones at the noise level
        assert np.all(s <= sig + noise)
        np.testing.assert_allclose(s[:20], sig[:20], rtol=0, atol=noise + 1e-12 * sig[0])
    else:
        # the single pass's core is a least-squares estimate, not a projection of A:
        # no interlacing; its leading values are still accurate to the 1-view error level
        np.testing.assert_allclose(s[:10], sig[:10], rtol=1e-2)
    rows = [0, 1, 4999, 25000, cfg.m - 1]
    Ar = _sampled_rows(A, rows)                             # oracle-side fp64 dot products
    AV = Ar @ V
    if exact_av:                                            # A V = U diag(S), row by row
        err = np.abs(AV - U[rows] * s) / s[0]
        assert err.max() <= 1e-12
    return AV


def test_c4_krylov_v3_full_size(ctx, c4):
    cfg, A, Om, _, _ = c4
    U, s, V, info = ctx.block_krylov(A, cfg.k, cfg.p, 3, Om)
    assert info.views == 3
    _check_c4_triplets(cfg, A, U, s, V, exact_av=True)
    # Alg. 9 == Alg. 2 for v < 4: the subspace call gives the same result
    U2, s2, V2, _ = ctx.subspace(A, cfg.k, cfg.p, 3, Om)
    assert np.max(np.abs(host(s2) - host(s)) / host(s)) <= 1e-10
    assert O.projector_distance(host(U2), host(U)) <= 1e-9


def test_c4_single_pass_full_size(ctx, c4):
    cfg, A, Om, _, Phi = c4
    U, s, V, info = ctx.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Phi)
    assert info.views == 1
    _check_c4_triplets(cfg, A, U, s, V, exact_av=False)


@pytest.mark.parametrize("alg,v,inp", [("single_pass", 1, 0), ("krylov", 3, 0), ("subspace", 3, 1)])
def test_c4_recipe_scaled_vs_oracle(ctx, alg, v, inp):
    """C4's recipe and widths (k=100, p=20, l2=240: the single pass takes the two-view path for
    l > 72) at 5000 x 20000, element-wise against the oracle."""
    from paper_1804_07531_b200 import rsvd

    cfg = S.CONFIGS["C4"]
    A = S.make_matrix(cfg, 5000, 20000)
    Om = S.gaussian_test_matrix(A.shape[0] if inp else A.shape[1], cfg.l, cfg,
                                S.ROLE_OMEGA_M if inp else S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(A.shape[0], cfg.l2, cfg, S.ROLE_PHI)
    Ad = torch.from_numpy(A).cuda()
    if alg == "single_pass":
        U, s, V, info = ctx.single_pass(Ad, cfg.k, cfg.p, cfg.l2, colmajor_dev(Om), colmajor_dev(Phi))
        assert info.view_launches >= 2      # Y_c (w=120) + Y_r (w=240 in two 128-wide chunks)
    elif alg == "krylov":
        U, s, V, info = ctx.block_krylov(Ad, cfg.k, cfg.p, v, colmajor_dev(Om))
    else:
        U, s, V, info = ctx.subspace(Ad, cfg.k, cfg.p, v, colmajor_dev(Om), input=inp, flags=rsvd.RSVD_SQUARED)
        s = s.sqrt()
    Uo, so, Vo, _ = O.svd_of(A, alg, cfg.k, cfg.p, v=v, Omega=Om, l2=cfg.l2, Phi=Phi, transpose=bool(inp))
    U, s, V = host(U), host(s), host(V)
    assert np.max(np.abs(s - so) / so) <= 1e-10
    assert O.projector_distance(U, Uo) <= 1e-9
    assert O.projector_distance(V, Vo) <= 1e-9


def test_c4_normal_mode_full_size(ctx, c4):
    """A^T A ~ V S^2 V^T with the recommended orientation for odd v (input = A^T)."""
    from paper_1804_07531_b200 import rsvd

    cfg, A, _, Omm, _ = c4
    inp = rsvd.recommend_input(rsvd.RSVD_GOAL_NORMAL, 3)
    assert inp == rsvd.RSVD_INPUT_AT
    U, s2, V, _ = ctx.subspace(A, cfg.k, cfg.p, 3, Omm, input=inp, flags=rsvd.RSVD_SQUARED)
    s = np.sqrt(host(s2))
    Vh = host(V)
    np.testing.assert_allclose(Vh.T @ Vh, np.eye(cfg.k), atol=1e-12)
    sig = S.sigma_c4(cfg.rank)[:cfg.k]
    noise = cfg.noise * (np.sqrt(cfg.m) + np.sqrt(cfg.n)) * 1.1
    np.testing.assert_allclose(s[:20], sig[:20], rtol=0, atol=noise + 1e-12)
    # input = A^T with odd v: the algorithm's "A V = U S" identity becomes A^T U = V S
    Uh = host(U)
    cols = [0, 7, 100000, cfg.n - 1]
    AtU = np.stack([A[:, c].cpu().numpy() for c in cols]) @ Uh
    err = np.abs(AtU - Vh[cols] * s) / s[0]
    assert err.max() <= 1e-12


# ------------------------------------------------------------------ C5 at full size (fp32, 40 GB)
@pytest.fixture(scope="module")
def c5():
    free, _ = torch.cuda.mem_get_info()
    if free < 60e9:
        pytest.skip(f"C5 needs ~60 GB of free device memory, have {free / 1e9:.0f}")
    cfg = S.CONFIGS["C5"]
    A = S.make_matrix_torch(cfg, torch.device("cuda", 0), panel_rows=2048)
    Om = S.gaussian_test_matrix_torch(cfg.n, cfg.l, cfg, S.ROLE_OMEGA, torch.device("cuda", 0))
    torch.cuda.synchronize()
    yield cfg, A, Om
    del A
    torch.cuda.empty_cache()


@pytest.mark.parametrize("alg,v", [("subspace", 3), ("krylov", 5)])
def test_c5_full_size(ctx, c5, alg, v):
    """C5 (fp32, tcgen05 3xTF32 views): odd v ends with [Q_c, R_c] = qr(A Q_r), tsvd(R_c), so A V = U S
    row by row (checked in fp64 on sampled rows of the fp32 A, to fp32-accumulation accuracy);
    orthonormal factors; leading values at the construction sigma_i = exp(-i/100) to the noise level."""
    cfg, A, Om = c5
    fn = ctx.subspace if alg == "subspace" else ctx.block_krylov
    U, s, V, info = fn(A, cfg.k, cfg.p, v, Om)
    assert U.dtype == torch.float32 and info.views == v
    U, s, V = host(U).astype(np.float64), host(s).astype(np.float64), host(V).astype(np.float64)
    k = cfg.k
    np.testing.assert_allclose(U.T @ U, np.eye(k), atol=2e-5)
    np.testing.assert_allclose(V.T @ V, np.eye(k), atol=2e-5)
    assert np.all(np.diff(s) <= 1e-7 * s[0])
    sig = S.sigma_c5(cfg.rank)[:k]
    noise = cfg.noise * (np.sqrt(cfg.m) + np.sqrt(cfg.n)) * 1.1
    np.testing.assert_allclose(s[:20], sig[:20], rtol=1e-4, atol=noise)
    rows = [0, 1, 4999, 50000, cfg.m - 1]
    Ar = np.stack([A[r].double().cpu().numpy() for r in rows])
    err = np.abs(Ar @ V - U[rows] * s) / s[0]
    assert err.max() <= 1e-4
