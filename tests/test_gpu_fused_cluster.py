"""The one-read single pass for wide sketches (a3; k_view_fused_cl, view_fused_cluster.cu): Alg. 7
line 3 a)+b) from one read of A with the Y_c partials reduced across a 16- or
8-CTA cluster, for l > 72 or l2 > 144 (C4: l = 120, l2 = 240) with flags | RSVD_ONE_READ (the
default takes two view launches there, faster on device-resident A).  Parity of the whole Alg. 7
with the oracle on ragged shapes (rows not a multiple of the 16-row tile, columns not a multiple
of the 64-column strip or of the cluster's strip group, l2 not a multiple of 8), one view launch."""
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


def colmajor_dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().t()


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("m,n,k,p,l2", [(3000, 4000, 100, 20, 240), (2503, 1100, 80, 20, 203),
                                        (1777, 5003, 60, 20, 170), (4100, 2200, 120, 8, 256),
                                        (999, 777, 90, 10, 100),
                                        # narrow widths (C2's 30 / 60, C3's 70 / 140) on the cluster kernel
                                        (4000, 4000, 20, 10, 60), (6001, 2999, 50, 20, 140)])
def test_fused_cluster_single_pass_vs_oracle(ctx, m, n, k, p, l2):
    cfg = S.CONFIGS["C4"]
    A = S.make_matrix(cfg, m, n)
    l = k + p
    Om = S.gaussian_test_matrix(n, l, cfg, S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(m, l2, cfg, S.ROLE_PHI)
    from paper_1804_07531_b200 import rsvd

    U, s, V, info = ctx.single_pass(torch.from_numpy(A).cuda(), k, p, l2, colmajor_dev(Om), colmajor_dev(Phi),
                                    flags=rsvd.RSVD_ONE_READ)
    assert info.views == 1 and info.view_launches == 1      # one read of A
    Uo, so, Vo = O.one_view_tropp(A, k, p, l2 - k, p, Om, Phi)
    U, s, V = host(U), host(s), host(V)
    assert np.max(np.abs(s - so) / so) <= 1e-10
    assert O.projector_distance(U, Uo) <= 1e-9 and O.projector_distance(V, Vo) <= 1e-9
    r, ro = O.residual_fro(A, U, s, V), O.residual_fro(A, Uo, so, Vo)
    assert abs(r - ro) <= 1e-8 * ro


@pytest.mark.parametrize("m,n,l,l2", [(700, 1300, 130 - 10, 200), (2047, 4099, 100, 256), (333, 5000, 73, 150),
                                      (1200, 520, 128, 145)])
def test_fused_cluster_sketches_bitwise_integer(ctx, m, n, l, l2):
    """Integer A, Omega, Phi keep every partial sum exact in fp64, so Y_c = A Omega and Y_r = A^T Phi
    from the one-read cluster kernel (DSMEM reduction of the Y_c partials, group slots summed in
    order) are bit-exact against NumPy, whatever the summation order (rsvd_view_fused)."""
    A = S.integer_matrix(m, n, -3, 3, seed=m)
    Om = S.integer_matrix(n, l, -2, 2, seed=n, order="F")
    Phi = S.integer_matrix(m, l2, -2, 2, seed=l2, order="F")
    Yc, Yr, info = ctx.view_fused(torch.from_numpy(A).cuda(), colmajor_dev(Om), colmajor_dev(Phi))
    assert info.view_launches == 1
    assert np.array_equal(host(Yc), A @ Om)
    assert np.array_equal(host(Yr), A.T @ Phi)
