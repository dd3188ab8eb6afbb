"""Block Krylov for a matrix read row wise, rsvd_block_krylov_rows: A^T A X from ONE
pass over the rows (row panels kept in L2 between the two products).  Parity with the oracle's
row-wise block Krylov (oracle.row_block_krylov) and with Alg. 9 (rsvd_block_krylov, the explicit
views: the same Krylov subspaces), read counts (half the views), multi-panel runs at C3's
full size, fp32 and the sharded path (loopback, unequal shards)."""
import threading

import numpy as np
import pytest
import torch

import oracle as O
import synth as S
from paper_1804_07531_b200.sharding import shard_rows

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
    return t.detach().cpu().numpy().astype(np.float64)


def check(A, U, s, V, Uo, so, Vo, ts=1e-10, tp=1e-9, tr=1e-8):
    assert np.max(np.abs(s - so) / so) <= ts
    assert O.projector_distance(U, Uo) <= tp and O.projector_distance(V, Vo) <= tp
    r, ro = O.residual_fro(A, U, s, V), O.residual_fro(A, Uo, so, Vo)
    assert abs(r - ro) <= tr * ro


@pytest.mark.parametrize("name,m,n", [("C1", None, None), ("C2", None, None), ("C3", 3000, 1100), ("C2", 777, 555)])
@pytest.mark.parametrize("v", [2, 3, 4, 5, 6])
def test_krylov_rows_vs_oracle(ctx, name, m, n, v):
    cfg = S.CONFIGS[name]
    A = S.make_matrix(cfg, m, n)
    if (v // 2) * cfg.l > min(A.shape):
        pytest.skip("Krylov basis wider than the matrix")
    Om = S.gaussian_test_matrix(A.shape[1], cfg.l, cfg, S.ROLE_OMEGA)
    U, s, V, info = ctx.block_krylov_rows(torch.from_numpy(A).cuda(), cfg.k, cfg.p, v, colmajor_dev(Om))
    (Uo, so, Vo), passes = O.row_block_krylov(A, cfg.k, cfg.p, v, Om, panel_rows=512)
    assert info.views == passes == ((v - 1) // 2 + 1 if v % 2 else v // 2 + 1)
    check(A, host(U), host(s), host(V), Uo, so, Vo)
    # the same Krylov subspaces as Alg. 9 with explicit views
    U9, s9, V9, info9 = ctx.block_krylov(torch.from_numpy(A).cuda(), cfg.k, cfg.p, v, colmajor_dev(Om))
    assert info9.views == v
    check(A, host(U), host(s), host(V), host(U9), host(s9), host(V9))


@pytest.mark.parametrize("v", [3, 4, 5])
def test_krylov_rows_c3_full_size_many_panels(ctx, v):
    """C3 at full size (20000 x 8000, 1.28 GB): 27 row panels of <= 48 MB per pass."""
    cfg = S.CONFIGS["C3"]
    A = S.make_matrix(cfg)
    Om = S.gaussian_test_matrix(cfg.n, cfg.l, cfg, S.ROLE_OMEGA)
    U, s, V, info = ctx.block_krylov_rows(torch.from_numpy(A).cuda(), cfg.k, cfg.p, v, colmajor_dev(Om))
    (Uo, so, Vo), passes = O.row_block_krylov(A, cfg.k, cfg.p, v, Om, panel_rows=4096)
    assert info.views == passes
    check(A, host(U), host(s), host(V), Uo, so, Vo)


@pytest.mark.parametrize("v", [3, 4])
def test_krylov_rows_fp32(ctx, v):
    cfg = S.CONFIGS["C5"]
    A = S.make_matrix(cfg, 2600, 2400)
    k, p = 40, 10
    Om = S.gaussian_test_matrix(A.shape[1], k + p, cfg, S.ROLE_OMEGA)
    U, s, V, info = ctx.block_krylov_rows(torch.from_numpy(A).cuda(), k, p, v, colmajor_dev(Om))
    assert U.dtype == torch.float32
    A64 = A.astype(np.float64)
    (Uo, so, Vo), _ = O.row_block_krylov(A64, k, p, v, Om.astype(np.float64), panel_rows=512)
    check(A64, host(U), host(s), host(V), Uo, so, Vo, ts=1e-4, tp=1e-3, tr=1e-3)


@pytest.mark.parametrize("N", [2, 3])
@pytest.mark.parametrize("v", [4, 5])
def test_krylov_rows_sharded(v, N):
    """Row shards (loopback, unequal 128-aligned shards): A^T A X partials all-reduced."""
    from paper_1804_07531_b200 import rsvd

    cfg = S.CONFIGS["C2"]
    A = S.make_matrix(cfg, 2600, 1200)
    m, n = A.shape
    Om = S.gaussian_test_matrix(n, cfg.l, cfg, S.ROLE_OMEGA)
    Ad, Omd = torch.from_numpy(A).cuda(), colmajor_dev(Om)
    torch.cuda.synchronize()
    group = rsvd.LoopGroup(N)
    streams = [torch.cuda.Stream() for _ in range(N)]
    ctxs = [rsvd.Context(0, stream=s_) for s_ in streams]
    for r, c in enumerate(ctxs):
        c.comm_init_loopback(group, r)
    group.close()
    outs, errs = [None] * N, [None] * N

    def work(r):
        try:
            sh = shard_rows(m, N, r, align=128)
            with torch.cuda.stream(streams[r]):
                outs[r] = ctxs[r].block_krylov_rows(Ad[sh.row0:sh.row0 + sh.m_local], cfg.k, cfg.p, v, Omd, m=m,
                                                    row0=sh.row0)[:3]
            streams[r].synchronize()
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(N)]
    [t.start() for t in th]
    [t.join(300) for t in th]
    for c in ctxs:
        c.close()
    for e in errs:
        if e is not None:
            raise e
    U = np.concatenate([host(o[0]) for o in outs])
    for o in outs[1:]:
        assert np.array_equal(host(o[1]), host(outs[0][1])) and np.array_equal(host(o[2]), host(outs[0][2]))
    (Uo, so, Vo), _ = O.row_block_krylov(A, cfg.k, cfg.p, v, Om, panel_rows=512)
    check(A, U, host(outs[0][1]), host(outs[0][2]), Uo, so, Vo)
