"""C4 at full size (fp64 50000 x 200000, 80 GB), element-wise against the oracle (north_star:
"GPU U, Sigma, V match the CPU oracle within the stated tolerances on all five configs").

A is built on the GPU (synth.make_matrix_torch, the config's recipe) and copied back to host
memory once; the oracle evaluates every view over row panels of those bytes (oracle.PanelOp,
SURVEY §8(c)), with the same Omega / Phi.  BASELINE C4's runs: block Krylov v = 3 (= Alg. 2 v = 3,
P:930), the single pass with l2 = 240, and the normal-matrix estimate with the recommended
orientation for odd v (input = A^T).  Tolerances (north_star, SURVEY c-14): sigma
1e-10 relative, projectors 1e-9, ||A - U S V^T||_F within 1e-8 relative of the oracle's (explicit
residual pass over A); normal mode sigma^2 at 2e-10 (reading R12).  Also the properties that hold
at any size: A V = U S row by row for the projection methods, orthonormal factors.
"""
import os

import numpy as np
import pytest
import torch

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu

PANEL = 4096


@pytest.fixture(scope="module")
def ctx():
    from paper_1804_07531_b200 import build, rsvd

    build.build()
    c = rsvd.Context(0)
    yield c
    c.close()


def host(t):
    return t.detach().cpu().numpy()


def _host_mem_available():
    try:
        import psutil

        return psutil.virtual_memory().available
    except Exception:
        return os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")


@pytest.fixture(scope="module")
def c4():
    free, _ = torch.cuda.mem_get_info()
    if free < 110e9:
        pytest.skip(f"C4 needs ~110 GB of free device memory, have {free / 1e9:.0f}")
    if _host_mem_available() < 110e9:
        pytest.skip("C4's oracle needs ~110 GB of host memory for the copied-back A")
    cfg = S.CONFIGS["C4"]
    dev = torch.device("cuda", 0)
    A = S.make_matrix_torch(cfg, dev, panel_rows=2048)
    Om = S.gaussian_test_matrix_torch(cfg.n, cfg.l, cfg, S.ROLE_OMEGA, dev)
    Omm = S.gaussian_test_matrix_torch(cfg.m, cfg.l, cfg, S.ROLE_OMEGA_M, dev)
    Phi = S.gaussian_test_matrix_torch(cfg.m, cfg.l2, cfg, S.ROLE_PHI, dev)
    torch.cuda.synchronize()
    Ah = np.empty((cfg.m, cfg.n), dtype=np.float64)          # the same bytes on the host
    for r0 in range(0, cfg.m, PANEL):
        Ah[r0:r0 + PANEL] = A[r0:r0 + PANEL].cpu().numpy()
    yield cfg, A, Ah, Om, Omm, Phi
    del A, Ah
    torch.cuda.empty_cache()


def _compare(Ah, U, s, V, Uo, so, Vo, tol_s=1e-10):
    assert np.max(np.abs(s - so) / so) <= tol_s
    assert O.projector_distance(U, Uo) <= 1e-9
    assert O.projector_distance(V, Vo) <= 1e-9


def _residuals(Ah, U, s, V, Uo, so, Vo):
    r, ro = O.residual_fro(Ah, U, s, V, panel=PANEL), O.residual_fro(Ah, Uo, so, Vo, panel=PANEL)
    assert abs(r - ro) <= 1e-8 * ro


def test_c4_krylov_v3_vs_oracle(ctx, c4):
    cfg, A, Ah, Om, _, _ = c4
    U, s, V, info = ctx.block_krylov(A, cfg.k, cfg.p, 3, Om)
    assert info.views == 3 and info.vectors == (3 + 1 - 1) * cfg.l
    U, s, V = host(U), host(s), host(V)
    Uo, so, Vo, op = O.svd_of(Ah, "krylov", cfg.k, cfg.p, v=3, Omega=host(Om), panel_rows=PANEL)
    assert op.views == 3
    _compare(Ah, U, s, V, Uo, so, Vo)
    # any size: orthonormal factors, A V = U diag(S) row by row (Alg. 9 odd v ends with qr(A Q_r))
    np.testing.assert_allclose(U.T @ U, np.eye(cfg.k), atol=1e-12)
    np.testing.assert_allclose(V.T @ V, np.eye(cfg.k), atol=1e-12)
    rows = [0, 1, 4999, 25000, cfg.m - 1]
    assert np.max(np.abs(Ah[rows] @ V - U[rows] * s) / s[0]) <= 1e-12
    _residuals(Ah, U, s, V, Uo, so, Vo)


def test_c4_single_pass_vs_oracle(ctx, c4):
    cfg, A, Ah, Om, _, Phi = c4
    U, s, V, info = ctx.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Phi)
    assert info.views == 1
    U, s, V = host(U), host(s), host(V)
    Uo, so, Vo, op = O.svd_of(Ah, "single_pass", cfg.k, cfg.p, Omega=host(Om), l2=cfg.l2, Phi=host(Phi),
                              panel_rows=PANEL)
    assert op.views == 1
    _compare(Ah, U, s, V, Uo, so, Vo)
    _residuals(Ah, U, s, V, Uo, so, Vo)


def test_c4_normal_mode_vs_oracle(ctx, c4):
    """A^T A ~ V S^2 V^T from Alg. 2 v = 3 with input = A^T (the recommended orientation for odd v)."""
    from paper_1804_07531_b200 import rsvd

    cfg, A, Ah, _, Omm, _ = c4
    inp = rsvd.recommend_input(rsvd.RSVD_GOAL_NORMAL, 3)
    assert inp == rsvd.RSVD_INPUT_AT
    U, s2, V, info = ctx.subspace(A, cfg.k, cfg.p, 3, Omm, input=inp, flags=rsvd.RSVD_SQUARED)
    U, s2, V = host(U), host(s2), host(V)
    Uo, so, Vo, _ = O.svd_of(Ah, "subspace", cfg.k, cfg.p, v=3, Omega=host(Omm), transpose=True, panel_rows=PANEL)
    assert np.max(np.abs(s2 - so ** 2) / so ** 2) <= 2e-10
    assert O.projector_distance(V, Vo) <= 1e-9
    assert O.projector_distance(U, Uo) <= 1e-9
    # input = A^T with odd v: the algorithm's own "B V = U S" identity is A^T U = V S
    s = np.sqrt(s2)
    cols = [0, 7, 100000, cfg.n - 1]
    assert np.max(np.abs(Ah[:, cols].T @ U - V[cols] * s) / s[0]) <= 1e-12


def test_c4_single_pass_one_read_vs_oracle(ctx, c4):
    """The same single pass from ONE read of the 80 GB A (RSVD_ONE_READ: the cluster kernel, a3)."""
    from paper_1804_07531_b200 import rsvd

    cfg, A, Ah, Om, _, Phi = c4
    U, s, V, info = ctx.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Phi, flags=rsvd.RSVD_ONE_READ)
    assert info.views == 1 and info.view_launches == 1
    assert info.view_bytes == cfg.m * cfg.n * 8.0
    U, s, V = host(U), host(s), host(V)
    Uo, so, Vo, _ = O.svd_of(Ah, "single_pass", cfg.k, cfg.p, Omega=host(Om), l2=cfg.l2, Phi=host(Phi),
                             panel_rows=PANEL)
    _compare(Ah, U, s, V, Uo, so, Vo)
