"""GPU parity of the fp32 path (C5's dtype): tcgen05 kind::tf32 views with the 3xTF32 split,
every step between views in fp64, inputs and outputs in fp32.

Tolerances (BASELINE.json north_star, fp32): singular values 1e-4 relative; projectors
||UU^T - UoUo^T||_F <= 1e-3; residual ||A - U S V^T||_F within 1e-3 relative of the oracle's.
The oracle runs in fp64 on the same fp32 bytes (upcast once).
Small integers are exact in tf32 (hi = a, lo = 0) and their products and fp32 partial sums
stay below 2^24 here, so the integer views are compared bit for bit.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu

TOL_S, TOL_P, TOL_R = 1e-4, 1e-3, 1e-3


@pytest.fixture(scope="module")
def ctx():
    from paper_1804_07531_b200 import build, rsvd

    build.build()
    c = rsvd.Context(0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def colmajor_dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().t()


def host(t):
    return t.detach().cpu().numpy()


VIEW_SHAPES = [(1037, 777), (200, 200), (64, 2000), (3000, 96), (129, 129)]
VIEW_WIDTHS = [1, 7, 16, 20, 100, 250, 256, 257, 300, 500, 512, 600]


@pytest.mark.parametrize("shape", VIEW_SHAPES)
@pytest.mark.parametrize("w", VIEW_WIDTHS)
@pytest.mark.parametrize("trans", [0, 1])
def test_view_f32_bit_exact(ctx, shape, w, trans):
    m, n = shape
    A = S.integer_matrix(m, n, -8, 8, seed=m + n, dtype=np.float32)
    X = S.integer_matrix(m if trans else n, w, -8, 8, seed=w, dtype=np.float32, order="F")
    Y, info = ctx.view(dev(A), colmajor_dev(X), trans=bool(trans))
    A64, X64 = A.astype(np.float64), X.astype(np.float64)
    ref = (A64.T @ X64) if trans else (A64 @ X64)
    assert Y.dtype == torch.float32
    assert np.array_equal(host(Y).astype(np.float64), ref)
    assert info.view_launches == (w + 255) // 256     # column chunks of <= 256 (TMEM: two M tiles)


@pytest.mark.parametrize("shape,w", [((4096, 3000), 250), ((777, 5000), 64), ((6000, 1500), 500)])
@pytest.mark.parametrize("trans", [0, 1])
def test_view_f32_gaussian_accuracy(ctx, shape, w, trans):
    """3xTF32 keeps ~22 bits per operand: the error is fp32-accumulation level, far below 1xTF32's."""
    m, n = shape
    A = S.random_gaussian_matrix(m, n, seed=11, dtype=np.float32)
    X = np.asarray(S.random_gaussian_matrix(m if trans else n, w, seed=12, dtype=np.float32), order="F")
    Y, _ = ctx.view(dev(A), colmajor_dev(X), trans=bool(trans))
    A64, X64 = A.astype(np.float64), X.astype(np.float64)
    ref = (A64.T @ X64) if trans else (A64 @ X64)
    K = m if trans else n
    scale = np.sqrt(K)  # |A| |X| row/column norm scale of each entry for unit Gaussians
    err = np.max(np.abs(host(Y).astype(np.float64) - ref)) / scale
    # fp32 accumulation over K terms: ~sqrt(K) u per entry on average; 1xTF32 would be ~1e-4
    assert err < 3e-5, err


def c5_scaled(m, n):
    cfg = S.CONFIGS["C5"]
    return cfg, S.make_matrix(cfg, m, n)


def check32(U, s, V, Uo, so, Vo, A):
    U, s, V = host(U).astype(np.float64), host(s).astype(np.float64), host(V).astype(np.float64)
    rel = np.max(np.abs(s - so) / np.abs(so))
    pu, pv = O.projector_distance(U, Uo), O.projector_distance(V, Vo)
    r, ro = O.residual_fro(A, U, s, V), O.residual_fro(A, Uo, so, Vo)
    assert rel <= TOL_S, f"sigma rel err {rel:.3e}"
    assert pu <= TOL_P, f"P_U {pu:.3e}"
    assert pv <= TOL_P, f"P_V {pv:.3e}"
    assert abs(r - ro) <= TOL_R * ro, f"residual {r:.6e} vs {ro:.6e}"
    return rel, pu, pv


@pytest.mark.parametrize("alg,v", [("subspace", 2), ("subspace", 3), ("subspace", 4), ("krylov", 4),
                                   ("single_pass", 1)])
@pytest.mark.parametrize("k,p", [(20, 10), (40, 20)])
def test_f32_algorithms_vs_oracle(ctx, alg, v, k, p):
    cfg, A = c5_scaled(3000, 2500)
    l = k + p
    Om = S.gaussian_test_matrix(A.shape[1], l, cfg, S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(A.shape[0], 2 * l, cfg, S.ROLE_PHI)
    Ad = dev(A)
    if alg == "subspace":
        U, s, V, info = ctx.subspace(Ad, k, p, v, colmajor_dev(Om))
    elif alg == "krylov":
        U, s, V, info = ctx.block_krylov(Ad, k, p, v, colmajor_dev(Om))
    else:
        U, s, V, info = ctx.single_pass(Ad, k, p, 2 * l, colmajor_dev(Om), colmajor_dev(Phi))
    assert U.dtype == torch.float32 and s.dtype == torch.float32
    A64 = A.astype(np.float64)
    Uo, so, Vo, _ = O.svd_of(A64, alg, k, p, v=v, Omega=Om.astype(np.float64), l2=2 * l,
                             Phi=Phi.astype(np.float64))
    check32(U, s, V, Uo, so, Vo, A64)


@pytest.mark.parametrize("alg,v", [("subspace", 2), ("subspace", 3), ("krylov", 3), ("krylov", 4)])
def test_f32_c5_widths_vs_oracle(ctx, alg, v):
    """C5's own k = 200, p = 50 (l = 250; Krylov v = 4 -> basis width 500) on a scaled C5 matrix."""
    cfg, A = c5_scaled(2600, 2400)
    k, p = cfg.k, cfg.p
    Om = S.gaussian_test_matrix(A.shape[1], k + p, cfg, S.ROLE_OMEGA)
    fn = ctx.subspace if alg == "subspace" else ctx.block_krylov
    U, s, V, info = fn(dev(A), k, p, v, colmajor_dev(Om))
    A64 = A.astype(np.float64)
    Uo, so, Vo, _ = O.svd_of(A64, alg, k, p, v=v, Omega=Om.astype(np.float64))
    check32(U, s, V, Uo, so, Vo, A64)


def test_f32_host_arguments(ctx):
    """Host fp32 A / Omega and host outputs through the same ABI call."""
    cfg, A = c5_scaled(1500, 1200)
    k, p = 10, 10
    Om = S.gaussian_test_matrix(A.shape[1], k + p, cfg, S.ROLE_OMEGA)
    U, s, V, info = ctx.subspace(torch.from_numpy(A), k, p, 3, torch.from_numpy(np.ascontiguousarray(Om.T)).t())
    assert info.host_staged == 1
    A64 = A.astype(np.float64)
    Uo, so, Vo, _ = O.svd_of(A64, "subspace", k, p, v=3, Omega=Om.astype(np.float64))
    check32(U, s, V, Uo, so, Vo, A64)
