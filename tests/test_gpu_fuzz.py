"""Randomised parity sweep (GPU): 96 seeded draws of shape, rank, oversampling, view count and
algorithm variant, each compared with the oracle on the same inputs.  Fixed seeds keep it
deterministic; sizes stay small so the whole sweep runs in well under a minute."""
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


def draw(seed):
    g = np.random.default_rng(1000 + seed)
    m, n = int(g.integers(40, 600)), int(g.integers(40, 600))
    k = int(g.integers(1, 12))
    p = int(g.integers(0, 10))
    l = k + p
    while l > min(m, n) // 3:       # keep the Krylov bases (up to 3l) inside the matrix
        p = max(0, p - 1)
        k = max(1, k - 1) if p == 0 else k
        l = k + p
    alg = ["subspace", "krylov", "single_pass", "minvar", "woolfe", "extended", "row", "subspace_T"][seed % 8]
    v = int(g.integers(2, 6))
    decay = float(g.uniform(0.05, 0.6))
    return g, m, n, k, p, alg, v, decay


def matrix(g, m, n, decay):
    r = min(m, n)
    X = np.linalg.qr(g.standard_normal((m, r)))[0]
    Y = np.linalg.qr(g.standard_normal((n, r)))[0]
    s = np.exp(-decay * np.arange(r))
    return (X * s) @ Y.T


@pytest.mark.parametrize("seed", range(96))
def test_random_parity(ctx, seed):
    from paper_1804_07531_b200 import rsvd

    g, m, n, k, p, alg, v, decay = draw(seed)
    A = matrix(g, m, n, decay)
    l = k + p
    l2 = min(m, l + int(g.integers(0, l + 1)))
    Om = g.standard_normal((n, l))
    Phi = g.standard_normal((m, l2))
    if alg == "subspace":
        U, s, V, _ = ctx.subspace(dev(A), k, p, v, cm(Om))
        Uo, so, Vo, _ = O.svd_of(A, "subspace", k, p, v=v, Omega=Om)
    elif alg == "subspace_T":
        OmT = g.standard_normal((m, l))
        U, s, V, _ = ctx.subspace(dev(A), k, p, v, cm(OmT), input=rsvd.RSVD_INPUT_AT)
        Uo, so, Vo, _ = O.svd_of(A, "subspace", k, p, v=v, Omega=OmT, transpose=True)
    elif alg == "krylov":
        U, s, V, _ = ctx.block_krylov(dev(A), k, p, v, cm(Om))
        Uo, so, Vo, _ = O.svd_of(A, "krylov", k, p, v=v, Omega=Om)
    elif alg == "single_pass":
        lc = int(g.integers(0, p + 1))
        U, s, V, _ = ctx.single_pass(dev(A), k, p, l2, cm(Om), cm(Phi), lc=lc)
        Uo, so, Vo = O.one_view_tropp(A, k, p, l2 - k, lc, Om, Phi)
    elif alg == "minvar":
        U, s, V, info = ctx.single_pass(dev(A), k, p, l2, cm(Om), cm(Phi), lc="minvar")
        Uo, so, Vo = O.one_view_tropp(A, k, p, l2 - k, info.lc_used, Om, Phi)
    elif alg == "woolfe":
        lc = int(g.integers(0, p + 1))
        U, s, V, _ = ctx.single_pass(dev(A), k, p, l2, cm(Om), cm(Phi), lc=lc, flags=rsvd.RSVD_WOOLFE)
        Uo, so, Vo = O.one_view_woolfe(A, k, p, l2 - k, lc, Om, Phi)
    elif alg == "extended":
        sw = min(m, n, l + int(g.integers(0, 2 * l + 1)))
        Xr, Xc = S.srft_matrix(m, sw, seed), S.srft_matrix(n, sw, seed + 500)
        var = ["bwz", "bwz2"][seed % 2]
        U, s, V, _ = ctx.single_pass_extended(dev(A), k, p, l2, sw, cm(Om), cm(Phi), cm(Xr), cm(Xc), variant=var)
        Uo, so, Vo = O.one_view_extended(A, k, p, l2 - k, Om, Phi, Xr, Xc, variant=var)
    else:
        U, s, V, _ = ctx.row_stream(dev(A), k, p, cm(Om))
        Uo, so, Vo = O.row_stream_qb(A, k, p, Om, panel_rows=64)
    s, U, V = host(s), host(U), host(V)
    # north_star tolerances (fp64): sigma 1e-10 relative, projectors 1e-9
    assert np.max(np.abs(s - so) / np.maximum(so, 1e-300)) <= 1e-10, (alg, m, n, k, p, v)
    assert O.projector_distance(U, Uo) <= 1e-9 and O.projector_distance(V, Vo) <= 1e-9, (alg, m, n, k, p, v)


@pytest.mark.parametrize("seed", range(24))
def test_random_parity_fp32(ctx, seed):
    """fp32 A (tcgen05 3xTF32 views): the oracle runs in fp64 on the same fp32 bytes; north_star
    fp32 tolerances (sigma 1e-4, projectors 1e-3).  Gentle decay keeps the top-k well separated."""
    g, m, n, k, p, alg, v, decay = draw(seed)
    A = matrix(g, m, n, min(decay, 0.2)).astype(np.float32)
    l = k + p
    Om = g.standard_normal((n, l)).astype(np.float32)
    A64, Om64 = A.astype(np.float64), Om.astype(np.float64)
    if seed % 3 == 0:
        U, s, V, _ = ctx.subspace(dev(A), k, p, v, cm(Om))
        Uo, so, Vo, _ = O.svd_of(A64, "subspace", k, p, v=v, Omega=Om64)
    elif seed % 3 == 1:
        U, s, V, _ = ctx.block_krylov(dev(A), k, p, v, cm(Om))
        Uo, so, Vo, _ = O.svd_of(A64, "krylov", k, p, v=v, Omega=Om64)
    else:
        U, s, V, _ = ctx.row_stream(dev(A), k, p, cm(Om))
        Uo, so, Vo = O.row_stream_qb(A64, k, p, Om64, panel_rows=64)
    s, U, V = (host(x).astype(np.float64) for x in (s, U, V))
    assert np.max(np.abs(s - so) / so) <= 1e-4
    assert O.projector_distance(U, Uo) <= 1e-3 and O.projector_distance(V, Vo) <= 1e-3
