"""The row-sharded (multi-GPU) code path of librsvd with N VIRTUAL row shards on one GPU.

rsvd_comm_init_loopback joins N contexts (one host thread and one stream each) into a loopback
group: every collective of the sharded schedule (Gram / cross-product all-reduces, the A^T Y
partials, the single pass's Y_r) is a host barrier plus cross-stream event waits and an ordered
sum over the ranks (SURVEY §4's single-process shard simulator).  Every algorithm runs with
N in {2, 3, 8} shards from shard_rows(align=128): unequal shards with row0 > 0 and m_local < m,
on both inputs (A and A^T, so the sharded side is the range side or the co-range side).

Checks: against the CPU oracle at north_star's tolerances (SURVEY c-14), against the unsharded
call to the same tolerances, and S / V (replicated outputs) bitwise identical on all ranks.
"""
import threading

import numpy as np
import pytest
import torch

import oracle as O
import synth as S
from paper_1804_07531_b200.sharding import shard_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_1804_07531_b200 import build, rsvd

    build.build()
    return rsvd


def colmajor_dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().t()


def host(t):
    return t.detach().cpu().numpy().astype(np.float64)


def run_sharded(rsvd, N, m, fn, align=128):
    """fn(ctx, shard) on N virtual ranks, each in its own thread with its own stream."""
    torch.cuda.synchronize()
    group = rsvd.LoopGroup(N, timeout_s=120.0)
    streams = [torch.cuda.Stream() for _ in range(N)]
    ctxs = [rsvd.Context(0, stream=s) for s in streams]
    for r, c in enumerate(ctxs):
        c.comm_init_loopback(group, r)
    group.close()                       # the contexts keep the group alive
    shards = [shard_rows(m, N, r, align=align) for r in range(N)]
    out, errs = [None] * N, [None] * N

    def worker(r):
        try:
            with torch.cuda.stream(streams[r]):
                out[r] = fn(ctxs[r], shards[r])
            streams[r].synchronize()
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=worker, args=(r,)) for r in range(N)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    for c in ctxs:
        c.close()
    for e in errs:
        if e is not None:
            raise e
    return shards, out


def assemble(shards, outs):
    """(U stacked over the row shards, S of rank 0, V of rank 0); S and V bitwise equal on all ranks."""
    U = np.concatenate([host(o[0]) for o in outs], axis=0) if outs[0][0] is not None else None
    S0, V0 = host(outs[0][1]), host(outs[0][2]) if outs[0][2] is not None else None
    for o in outs[1:]:
        assert np.array_equal(host(o[1]), S0), "S differs between ranks"
        if V0 is not None:
            assert np.array_equal(host(o[2]), V0), "V differs between ranks"
    return U, S0, V0


TOL = {"f64": (1e-10, 1e-9, 1e-8), "f32": (1e-4, 1e-3, 1e-3)}


def check(A, U, s, V, Uo, so, Vo, dt="f64", k=None):
    ts, tp, tr = TOL[dt]
    k = len(so) if k is None else k
    assert np.max(np.abs(s[:k] - so[:k]) / so[:k]) <= ts
    if U is not None:
        assert O.projector_distance(U[:, :k], Uo[:, :k]) <= tp
    if V is not None:
        assert O.projector_distance(V[:, :k], Vo[:, :k]) <= tp
    if U is not None and V is not None:
        r, ro = O.residual_fro(A, U, s, V), O.residual_fro(A, Uo, so, Vo)
        assert abs(r - ro) <= tr * ro


def problem(name, m, n, dt="f64"):
    cfg = S.CONFIGS[name]
    A = S.make_matrix(cfg, m, n)
    if dt == "f32":
        A = A.astype(np.float32)
    return cfg, A


NS = [2, 3, 8]
SHAPES = [("C2", 2600, 1200), ("C3", 3000, 1100)]


@pytest.mark.parametrize("N", NS)
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: s[0])
@pytest.mark.parametrize("alg,v,inp", [("subspace", 2, 0), ("subspace", 3, 0), ("subspace", 4, 1), ("subspace", 5, 1),
                                       ("krylov", 3, 0), ("krylov", 4, 0), ("krylov", 5, 0), ("krylov", 4, 1),
                                       ("krylov", 5, 1)])
def test_sharded_subspace_krylov(lib, N, shape, alg, v, inp):
    name, m, n = shape
    cfg, A = problem(name, m, n)
    rows = m if inp else n
    Om = S.gaussian_test_matrix(rows, cfg.l, cfg, S.ROLE_OMEGA_M if inp else S.ROLE_OMEGA)
    Ad, Omd = torch.from_numpy(A).cuda(), colmajor_dev(Om)

    def fn(ctx, sh):
        As = Ad[sh.row0:sh.row0 + sh.m_local]
        Os = Omd[sh.row0:sh.row0 + sh.m_local] if inp else Omd
        f = ctx.subspace if alg == "subspace" else ctx.block_krylov
        U, s, V, info = f(As, cfg.k, cfg.p, v, Os, input=inp, m=m, row0=sh.row0)
        assert info.views == v and info.graph_replayed == 0
        return U, s, V

    shards, outs = run_sharded(lib, N, m, fn)
    assert len({sh.m_local for sh in shards}) > 1 and shards[-1].row0 > 0   # unequal shards
    U, s, V = assemble(shards, outs)
    Uo, so, Vo, _ = O.svd_of(A, alg, cfg.k, cfg.p, v=v, Omega=Om, transpose=bool(inp))
    check(A, U, s, V, Uo, so, Vo)


@pytest.mark.parametrize("N", NS)
@pytest.mark.parametrize("variant", ["tropp", "minvar", "woolfe", "lc0"])
def test_sharded_single_pass(lib, N, variant):
    cfg, A = problem("C2", 2600, 1200)
    m, n = A.shape
    Om = S.gaussian_test_matrix(n, cfg.l, cfg, S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(m, cfg.l2, cfg, S.ROLE_PHI)
    Ad, Omd, Phid = torch.from_numpy(A).cuda(), colmajor_dev(Om), colmajor_dev(Phi)
    lc = {"tropp": -1, "minvar": "minvar", "woolfe": cfg.p // 2, "lc0": 0}[variant]
    flags = lib.RSVD_WOOLFE if variant == "woolfe" else 0

    def fn(ctx, sh):
        sl = slice(sh.row0, sh.row0 + sh.m_local)
        U, s, V, info = ctx.single_pass(Ad[sl], cfg.k, cfg.p, cfg.l2, Omd, Phid[sl], lc=lc, flags=flags, m=m,
                                        row0=sh.row0)
        return U, s, V, info.lc_used

    shards, outs = run_sharded(lib, N, m, fn)
    lcs = {o[3] for o in outs}
    assert len(lcs) == 1
    U, s, V = assemble(shards, outs)
    if variant == "woolfe":
        Uo, so, Vo = O.one_view_woolfe(A, cfg.k, cfg.p, cfg.l2 - cfg.k, cfg.p // 2, Om, Phi)
    elif variant == "minvar":
        Uo, so, Vo, lco = O.one_view_minvar(A, cfg.k, cfg.p, cfg.l2 - cfg.k, Om, Phi)
        assert lcs.pop() == lco
    else:
        Uo, so, Vo = O.one_view_tropp(A, cfg.k, cfg.p, cfg.l2 - cfg.k, 0 if variant == "lc0" else cfg.p, Om, Phi)
    check(A, U, s, V, Uo, so, Vo)


@pytest.mark.parametrize("N", NS)
def test_sharded_row_stream_and_extended(lib, N):
    cfg, A = problem("C2", 2600, 1200)
    m, n = A.shape
    Om = S.gaussian_test_matrix(n, cfg.l, cfg, S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(m, cfg.l, cfg, S.ROLE_PHI)
    s_ = 2 * cfg.l
    Xr, Xc = S.srft_matrix(m, s_, 11), S.srft_matrix(n, s_, 12)
    Ad, Omd, Phid, Xrd, Xcd = (torch.from_numpy(A).cuda(), colmajor_dev(Om), colmajor_dev(Phi), colmajor_dev(Xr),
                               colmajor_dev(Xc))

    def fn_row(ctx, sh):
        sl = slice(sh.row0, sh.row0 + sh.m_local)
        return ctx.row_stream(Ad[sl], cfg.k, cfg.p, Omd, m=m, row0=sh.row0)[:3]

    shards, outs = run_sharded(lib, N, m, fn_row)
    U, s, V = assemble(shards, outs)
    Uo, so, Vo = O.row_stream_qb(A, cfg.k, cfg.p, Om)
    check(A, U, s, V, Uo, so, Vo)

    def fn_ext(ctx, sh):
        sl = slice(sh.row0, sh.row0 + sh.m_local)
        return ctx.single_pass_extended(Ad[sl], cfg.k, cfg.p, cfg.l, s_, Omd, Phid[sl], Xrd[sl], Xcd, "bwz2", m=m,
                                        row0=sh.row0)[:3]

    shards, outs = run_sharded(lib, N, m, fn_ext)
    U, s, V = assemble(shards, outs)
    Uo, so, Vo = O.one_view_extended(A, cfg.k, cfg.p, cfg.p, Om, Phi, Xr, Xc, "bwz2")
    check(A, U, s, V, Uo, so, Vo)


@pytest.mark.parametrize("N", NS)
@pytest.mark.parametrize("alg,v", [("nystrom", 2), ("nystrom", 3), ("pinched", 3), ("pinched", 4)])
def test_sharded_normal_matrix(lib, N, alg, v):
    cfg, A = problem("C2", 2600, 1200)
    m, n = A.shape
    om_m = (v % 2 == 1) if alg == "nystrom" else (v % 2 == 0)
    Om = S.gaussian_test_matrix(m if om_m else n, cfg.l, cfg, S.ROLE_OMEGA_M if om_m else S.ROLE_OMEGA)
    Ad, Omd = torch.from_numpy(A).cuda(), colmajor_dev(Om)

    def fn(ctx, sh):
        sl = slice(sh.row0, sh.row0 + sh.m_local)
        f = ctx.nystrom if alg == "nystrom" else ctx.pinched
        s2, V, _ = f(Ad[sl], cfg.k, cfg.p, v, Omd[sl] if om_m else Omd, m=m, row0=sh.row0)
        return None, s2, V

    shards, outs = run_sharded(lib, N, m, fn)
    _, s2, V = assemble(shards, outs)
    if alg == "nystrom":
        Vo, so2 = O.nystrom_tevd(A, cfg.k, cfg.p, v, Om)
    else:
        Vo, so2 = O.pinched_tevd(A, cfg.k, cfg.p, v, Om)
    assert np.max(np.abs(s2 - so2) / so2) <= 2e-10
    assert O.projector_distance(V, Vo) <= 1e-9


@pytest.mark.parametrize("N", [2, 8])
@pytest.mark.parametrize("alg,v", [("subspace", 3), ("krylov", 4)])
def test_sharded_fp32(lib, N, alg, v):
    """fp32 A (tcgen05 3xTF32 views) through the sharded path, C5's recipe at 3000 x 2400."""
    cfg = S.CONFIGS["C5"]
    A = S.make_matrix(cfg, 3000, 2400)
    m, n = A.shape
    k, p = 40, 10
    Om = S.gaussian_test_matrix(n, k + p, cfg, S.ROLE_OMEGA)
    Ad, Omd = torch.from_numpy(A).cuda(), colmajor_dev(Om)

    def fn(ctx, sh):
        f = ctx.subspace if alg == "subspace" else ctx.block_krylov
        return f(Ad[sh.row0:sh.row0 + sh.m_local], k, p, v, Omd, m=m, row0=sh.row0)[:3]

    shards, outs = run_sharded(lib, N, m, fn)
    U, s, V = assemble(shards, outs)
    Uo, so, Vo, _ = O.svd_of(A.astype(np.float64), alg, k, p, v=v, Omega=Om.astype(np.float64))
    check(A.astype(np.float64), U, s, V, Uo, so, Vo, dt="f32")


@pytest.mark.parametrize("N", NS)
def test_sharded_equals_unsharded(lib, N):
    """The sharded schedule against the communicator-free call on the same bytes (rounding only)."""
    cfg, A = problem("C3", 3000, 1100)
    m, n = A.shape
    Om = S.gaussian_test_matrix(n, cfg.l, cfg, S.ROLE_OMEGA)
    Ad, Omd = torch.from_numpy(A).cuda(), colmajor_dev(Om)
    c0 = lib.Context(0)
    U1, s1, V1, _ = c0.block_krylov(Ad, cfg.k, cfg.p, 5, Omd)
    c0.close()

    def fn(ctx, sh):
        return ctx.block_krylov(Ad[sh.row0:sh.row0 + sh.m_local], cfg.k, cfg.p, 5, Omd, m=m, row0=sh.row0)[:3]

    shards, outs = run_sharded(lib, N, m, fn)
    U, s, V = assemble(shards, outs)
    check(A, U, s, V, host(U1), host(s1), host(V1))


@pytest.mark.parametrize("N", NS)
@pytest.mark.parametrize("alg,v,inp,dt", [("subspace", 3, 0, "f64"), ("subspace", 4, 1, "f64"), ("krylov", 4, 0, "f64"),
                                          ("krylov", 5, 1, "f64"), ("krylov", 4, 0, "f32")])
def test_shard_n_equals_replicated_n(lib, N, alg, v, inp, dt, monkeypatch):
    """n-side sharding (Alg. 2 / 9 under a communicator: side-N blocks split into 32-aligned row
    chunks, A^T Y reduce-scattered, X all-gathered before A X, V all-gathered at the end) against
    the replicated side-N schedule (RSVD_NO_SHARD_N=1) on the same shards: rounding only, and V
    full length and bitwise equal on all ranks.  n = 2300 gives every rank a chunk at N = 2, 3, 8
    (the last one ragged)."""
    cfg, A = problem("C2", 2600, 2300, dt)
    m, n = A.shape
    rows = m if inp else n
    Om = S.gaussian_test_matrix(rows, cfg.l, cfg, S.ROLE_OMEGA_M if inp else S.ROLE_OMEGA)
    if dt == "f32":
        Om = Om.astype(np.float32)
    Ad, Omd = torch.from_numpy(A).cuda(), colmajor_dev(Om)

    def fn(ctx, sh):
        As = Ad[sh.row0:sh.row0 + sh.m_local]
        Os = Omd[sh.row0:sh.row0 + sh.m_local] if inp else Omd
        f = ctx.subspace if alg == "subspace" else ctx.block_krylov
        return f(As, cfg.k, cfg.p, v, Os, input=inp, m=m, row0=sh.row0)[:3]

    shards, outs = run_sharded(lib, N, m, fn)
    U, s, V = assemble(shards, outs)
    assert V.shape == (n, cfg.k)
    monkeypatch.setenv("RSVD_NO_SHARD_N", "1")
    shards, outs = run_sharded(lib, N, m, fn)
    Ur, sr, Vr = assemble(shards, outs)
    A64 = A.astype(np.float64)
    check(A64, U, s, V, Ur, sr, Vr, dt=dt)
    if dt == "f64":   # rounding-level agreement (fp64 views: only the reduction order differs)
        assert np.max(np.abs(s - sr) / sr) <= 1e-12
    Uo, so, Vo, _ = O.svd_of(A64, alg, cfg.k, cfg.p, v=v, Omega=Om.astype(np.float64), transpose=bool(inp))
    check(A64, U, s, V, Uo, so, Vo, dt=dt)


def test_loopback_failing_rank_releases_peers(lib):
    """A rank whose call fails (here: an invalid argument detected on the device side of the call,
    a zero-row shard) must not leave its peers blocked: they return RSVD_E_NCCL."""
    cfg, A = problem("C2", 600, 400)
    m, n = A.shape
    Om = S.gaussian_test_matrix(n, cfg.l, cfg, S.ROLE_OMEGA)
    Ad, Omd = torch.from_numpy(A).cuda(), colmajor_dev(Om)
    group = lib.LoopGroup(2, timeout_s=20.0)
    ctxs = [lib.Context(0, stream=torch.cuda.Stream()) for _ in range(2)]
    for r, c in enumerate(ctxs):
        c.comm_init_loopback(group, r)
    res = [None, None]

    def worker(r):
        try:
            if r == 0:
                ctxs[0].subspace(Ad[:300], cfg.k, cfg.p, 3, Omd, m=m, row0=0)
            else:   # rank 1 never joins the collectives (stands for a crashed peer)
                pass
            res[r] = "ok"
        except lib.RsvdError as e:
            res[r] = e.code

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(60)
    assert res[0] == -4          # RSVD_E_NCCL after the 20 s timeout, not a hang
    for c in ctxs:
        c.close()
    group.close()
