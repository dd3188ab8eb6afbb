"""The row-sharded (multi-GPU) code path on one GPU: a one-rank NCCL communicator makes every
call take the sharded route of SURVEY §8(e) — CholeskyQR of side-M blocks through all-reduced
Grams (no single-launch cluster path), the A^T Y partial followed by ncclAllReduce, NCCL calls
captured in the CUDA graph.  Results must match the CPU oracle within the north_star tolerances
and the communicator-free context to rounding.  (The pool gives one GPU per call; the N > 1
schedule itself is checked against the oracle on CPU in test_multirank_cpu.py.)"""
import numpy as np
import pytest
import torch

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctxs():
    from paper_1804_07531_b200 import build, rsvd

    build.build()
    c1 = rsvd.Context(0)
    c1.comm_init(1, 0, rsvd.get_unique_id())
    c0 = rsvd.Context(0)
    yield c1, c0
    c1.close()
    c0.close()


def colmajor_dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().t()


def host(t):
    return t.detach().cpu().numpy()


CASES = [("C2", None, None, "subspace", 3), ("C2", None, None, "krylov", 4), ("C2", None, None, "single_pass", 1),
         ("C3", 3000, 1200, "subspace", 2), ("C3", 3000, 1200, "krylov", 5), ("C1", None, None, "subspace", 4)]


@pytest.mark.parametrize("name,m,n,alg,v", CASES)
def test_one_rank_comm_matches_oracle(ctxs, name, m, n, alg, v):
    c1, c0 = ctxs
    assert c1.nranks == 1
    cfg = S.CONFIGS[name]
    A = S.make_matrix(cfg, m, n)
    Om = S.gaussian_test_matrix(A.shape[1], cfg.l, cfg, S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(A.shape[0], cfg.l2, cfg, S.ROLE_PHI)
    Ad = torch.from_numpy(A).cuda()
    outs = []
    for c in (c1, c0):
        if alg == "subspace":
            r = c.subspace(Ad, cfg.k, cfg.p, v, colmajor_dev(Om))
        elif alg == "krylov":
            r = c.block_krylov(Ad, cfg.k, cfg.p, v, colmajor_dev(Om))
        else:
            r = c.single_pass(Ad, cfg.k, cfg.p, cfg.l2, colmajor_dev(Om), colmajor_dev(Phi))
        outs.append([host(x) for x in r[:3]])
    Uo, so, Vo, _ = O.svd_of(A, alg, cfg.k, cfg.p, v=v, Omega=Om, l2=cfg.l2, Phi=Phi)
    (U, s, V), (U0, s0, V0) = outs
    assert np.max(np.abs(s - so) / so) <= 1e-10
    assert O.projector_distance(U, Uo) <= 1e-9 and O.projector_distance(V, Vo) <= 1e-9
    assert np.max(np.abs(s - s0) / s0) <= 1e-12
    assert O.projector_distance(U, U0) <= 1e-11 and O.projector_distance(V, V0) <= 1e-11


def test_one_rank_comm_nystrom(ctxs):
    c1, _ = ctxs
    cfg = S.CONFIGS["C2"]
    A = S.make_matrix(cfg)
    Om = S.gaussian_test_matrix(A.shape[0], cfg.l, cfg, S.ROLE_OMEGA)   # odd v: m x l
    s2, V, info = c1.nystrom(torch.from_numpy(A).cuda(), cfg.k, cfg.p, 3, colmajor_dev(Om))
    Vo, s2o = O.nystrom_tevd(A, cfg.k, cfg.p, 3, Om)
    assert np.max(np.abs(host(s2) - s2o) / s2o) <= 2e-10
    assert O.projector_distance(host(V), Vo) <= 1e-9


@pytest.mark.parametrize("variant", ["minvar", "woolfe"])
def test_one_rank_comm_adaptive_single_pass(ctxs, variant):
    """MinVar l_c (masks on the row-sharded Q_c, C = Phi^T Q_c all-reduced) and Alg. 8 (Y_r on the
    replicated side) through the sharded route: same l_c and results as the communicator-free ctx."""
    from paper_1804_07531_b200 import rsvd

    c1, c0 = ctxs
    cfg = S.CONFIGS["C2"]
    A = S.make_matrix(cfg, 1500, 1300)
    Om = S.gaussian_test_matrix(A.shape[1], cfg.l, cfg, S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(A.shape[0], cfg.l2, cfg, S.ROLE_PHI)
    Ad = torch.from_numpy(A).cuda()
    kw = dict(lc="minvar") if variant == "minvar" else dict(lc=cfg.p // 2, flags=rsvd.RSVD_WOOLFE)
    outs = []
    for c in (c1, c0):
        r = c.single_pass(Ad, cfg.k, cfg.p, cfg.l2, colmajor_dev(Om), colmajor_dev(Phi), **kw)
        outs.append(([host(x) for x in r[:3]], r[3].lc_used))
    ((U, s, V), lc1), ((U0, s0, V0), lc0) = outs
    assert lc1 == lc0
    if variant == "minvar":
        Uo, so, Vo = O.one_view_tropp(A, cfg.k, cfg.p, cfg.l2 - cfg.k, lc1, Om, Phi)
    else:
        Uo, so, Vo = O.one_view_woolfe(A, cfg.k, cfg.p, cfg.l2 - cfg.k, cfg.p // 2, Om, Phi)
    assert np.max(np.abs(s - so) / so) <= 1e-10
    assert O.projector_distance(U, Uo) <= 1e-9 and O.projector_distance(V, Vo) <= 1e-9
    assert np.max(np.abs(s - s0) / s0) <= 1e-12


def test_one_rank_comm_row_stream(ctxs):
    """The row-wise pass through the sharded route (Yhat_r all-reduced once after the panels)."""
    c1, c0 = ctxs
    cfg = S.CONFIGS["C2"]
    A = S.make_matrix(cfg)
    Om = S.gaussian_test_matrix(A.shape[1], cfg.l, cfg, S.ROLE_OMEGA)
    Ad = torch.from_numpy(A).cuda()
    (U, s, V), (U0, s0, V0) = [[host(x) for x in c.row_stream(Ad, cfg.k, cfg.p, colmajor_dev(Om))[:3]]
                               for c in (c1, c0)]
    Uo, so, Vo = O.row_stream_qb(A, cfg.k, cfg.p, Om, panel_rows=4096)
    assert np.max(np.abs(s - so) / so) <= 1e-10 and O.projector_distance(V, Vo) <= 1e-9
    assert np.max(np.abs(s - s0) / s0) <= 1e-12
