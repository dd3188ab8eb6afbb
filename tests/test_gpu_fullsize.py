"""Parity at BASELINE.json's full sizes (GPU, -m gpu).

C3 (fp64 20000 x 8000): element-wise against the oracle on the same bytes, in the launch
configuration bench.py uses (CUDA graphs).  C4's recipe and widths at 5000 x 20000 against the
oracle.  The 80 GB C4 and the 40 GB C5 are compared element-wise with the oracle at full size in
test_gpu_fullsize_c4.py / test_gpu_fullsize_c5.py (oracle views over row panels of the bytes
copied back from the device).
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


# ------------------------------------------------------------------ C4 recipe and widths, scaled
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
        assert info.views == 1
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
