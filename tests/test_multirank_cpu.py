"""Multi-rank (N > 1) host logic on CPU: world_size-2 gloo process groups on 127.0.0.1.

* shard planning, unique-id broadcast and max-over-ranks timing (paper_1804_07531_b200.sharding);
* the row-sharded SCHEDULE (include/rsvd.h MULTI-GPU) as a NumPy emulation with
  gloo collectives: A X local, A^T Y and every Gram / cross product of a row-sharded block
  all-reduced, column-side blocks replicated.  Each rank runs Alg. 2 / 9 / 7 / 8, the extended
  sketch and the row-wise single pass on its row block;
* the n-side sharding of Alg. 2 / 9 (rsvd_api.cu Exec::plan_shard_n): side-N blocks in 32-aligned
  row chunks, A^T Y reduced and scattered to the chunks, X all-gathered before A X, side-N Grams
  all-reduced, the shifted CholeskyQR3 shift from the global length n, V all-gathered at the end;
  the gathered result must equal the single-process oracle (the schedule is exact algebra, so the
  same 1e-10 / 1e-9 tolerances as GPU parity apply).
  This checks the decomposition, not librsvd: the library's own sharded code path (unequal shards,
  row0 > 0, the CholeskyQR3 shift from the global row count) runs on one GPU with N virtual
  ranks in tests/test_gpu_loopback.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth as S
from paper_1804_07531_b200.sharding import broadcast_uid, max_over_ranks, shard_rows, weak_scaled


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ------------------------------------------------------------------ pure shard planning
@pytest.mark.parametrize("m,world,align", [(4000, 2, 1), (4001, 2, 1), (50000, 8, 128), (9, 8, 1), (1037, 3, 32)])
def test_shard_rows_tile_in_rank_order(m, world, align):
    shards = [shard_rows(m, world, r, align) for r in range(world)]
    assert shards[0].row0 == 0
    for a, b in zip(shards, shards[1:]):
        assert a.row0 + a.m_local == b.row0
    assert shards[-1].row0 + shards[-1].m_local == m
    assert all(s.m_local >= 1 for s in shards)
    assert max(s.m_local for s in shards) - min(s.m_local for s in shards) <= 2 * align  # one chunk + ragged tail


def test_weak_scaled():
    sh = [weak_scaled(4000, 4, r) for r in range(4)]
    assert [s.row0 for s in sh] == [0, 4000, 8000, 12000] and all(s.m == 16000 for s in sh)


def test_shard_rows_errors():
    with pytest.raises(ValueError):
        shard_rows(3, 4, 0)
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)


# ------------------------------------------------------------------ the sharded schedule (emulated)
class ShardedOps:
    """NumPy emulation of the row-sharded schedule: side M (rows of A) is sharded, side N is
    replicated.  All reductions go through dist.all_reduce (sum)."""

    def __init__(self, A_local):
        self.A = A_local

    @staticmethod
    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x))
        dist.all_reduce(t)
        return t.numpy()

    def sharded(self, side):
        return side == "M"

    def local_n(self, X):                     # a caller's n-long array -> this rank's side-N block
        return X

    def finish_n(self, X):                    # this rank's side-N block -> the full n-long output
        return X

    def view(self, from_side, X):             # from N: A X (local, side M); from M: A^T X (all-reduced)
        return self.A @ X if from_side == "N" else self.allreduce(self.A.T @ X)

    def cross(self, side, Xa, Xb):
        G = Xa.T @ Xb
        return self.allreduce(G) if self.sharded(side) else G


    def orth(self, side, Y, shifted=False):
        """CholeskyQR2 (shifted CholeskyQR3 if `shifted`) with the Gram all-reduced on the sharded
        side; R replicated.  Mirrors Exec::orth / orth_fused."""
        R = np.eye(Y.shape[1])
        if shifted:
            rows = self.allreduce(np.array([float(Y.shape[0])]))[0] if self.sharded(side) else Y.shape[0]
            G = self.cross(side, Y, Y)
            w = Y.shape[1]
            G = G + 11.0 * (rows * w + w * (w + 1)) * 1.1102230246251565e-16 * np.trace(G) * np.eye(w)
            L = np.linalg.cholesky(G)
            Y = np.linalg.solve(L, Y.T).T
            R = L.T                            # R0 folded into R (Y_in = Q R2 R1 R0)
        for _ in range(2):
            G = self.cross(side, Y, Y)
            L = np.linalg.cholesky(G)
            Y = np.linalg.solve(L, Y.T).T      # Y L^-T
            R = L.T @ R
        return Y, R


class ShardedOpsN(ShardedOps):
    """ShardedOps with the n-long side sharded too (Alg. 2 / 9 under N > 1 ranks): chunk size
    cs = round_up(ceil(n / N), 32), rank r owns rows [r cs, min((r + 1) cs, n)) of every side-N block."""

    def __init__(self, A_local, n, world, rank):
        super().__init__(A_local)
        self.n, self.world = n, world
        self.cs = -(-(-(-n // world)) // 32) * 32
        assert (world - 1) * self.cs < n          # every rank owns a chunk (as plan_shard_n requires)
        self.n0 = rank * self.cs
        self.n_loc = min(self.cs, n - self.n0)

    def sharded(self, side):
        return True

    def local_n(self, X):
        return X[self.n0:self.n0 + self.n_loc]

    def finish_n(self, X):
        pad = np.zeros((self.cs, X.shape[1]))
        pad[:X.shape[0]] = X
        parts = [torch.zeros(self.cs, X.shape[1], dtype=torch.float64) for _ in range(self.world)]
        dist.all_gather(parts, torch.from_numpy(pad))
        return np.vstack([t.numpy() for t in parts])[:self.n]

    def view(self, from_side, X):
        if from_side == "N":                      # all-gather X's chunks, then A X (local rows)
            return self.A @ self.finish_n(X)
        full = self.allreduce(self.A.T @ X)       # reduce (gloo has no reduce-scatter) ...
        return full[self.n0:self.n0 + self.n_loc]   # ... and keep this rank's chunk


def _alg2_sharded(ops, k, p, v, Om):
    Qr = ops.local_n(Om).copy()
    Qc = Rc = Rr = None
    for j in range(1, v + 1):
        if j % 2:
            Qc, Rc = ops.orth("M", ops.view("N", Qr))
        else:
            Qr, Rr = ops.orth("N", ops.view("M", Qc))
    if v % 2 == 0:
        Vw, lam, Uwt = np.linalg.svd(Rr)
        return Qc @ Uwt.T[:, :k], lam[:k], ops.finish_n(Qr @ Vw[:, :k])
    Uw, lam, Vwt = np.linalg.svd(Rc)
    return Qc @ Uw[:, :k], lam[:k], ops.finish_n(Qr @ Vwt.T[:, :k])


def _alg9_sharded(ops, k, p, v, Om):
    l = Om.shape[1]
    blocks, prev = [], ops.local_n(Om)
    for j in range(1, v):
        B = ops.view("N", prev) if j % 2 else ops.view("M", prev)
        side = "M" if j % 2 else "N"
        if j < v - 1:
            B, _ = ops.orth(side, B)
        if (v % 2 == 0 and j % 2 == 1) or (v % 2 == 1 and j % 2 == 0):
            blocks.append(B)
        prev = B
    side_K = "M" if v % 2 == 0 else "N"
    Q = None
    for B in blocks:                            # BCGS2 with all-reduced cross products
        W = B
        if Q is not None:
            W = W - Q @ ops.cross(side_K, Q, W)
            W, _ = ops.orth(side_K, W, shifted=True)
            W = W - Q @ ops.cross(side_K, Q, W)
        W, _ = ops.orth(side_K, W)
        Q = W if Q is None else np.hstack([Q, W])
    if v % 2 == 0:
        Qr, Rr = ops.orth("N", ops.view("M", Q))
        Vw, lam, Uwt = np.linalg.svd(Rr)
        return Q @ Uwt.T[:, :k], lam[:k], ops.finish_n(Qr @ Vw[:, :k])
    Qc, Rc = ops.orth("M", ops.view("N", Q))
    Uw, lam, Vwt = np.linalg.svd(Rc)
    return Qc @ Uw[:, :k], lam[:k], ops.finish_n(Q @ Vwt.T[:, :k])


def _alg7_sharded(ops, k, p, Om, Phi_local):
    Yc = ops.view("N", Om)                      # local
    Yr = ops.view("M", Phi_local)               # all-reduced (fused kernel's Y_r partial)
    Qc, _ = ops.orth("M", Yc)
    C = ops.cross("M", Phi_local, Qc)           # Phi^T Q_c, all-reduced
    Qh, Rh = np.linalg.qr(C)
    X = np.linalg.solve(Rh, Qh.T @ Yr.T)
    Uw, lam, Vwt = np.linalg.svd(X, full_matrices=False)
    return Qc @ Uw[:, :k], lam[:k], Vwt[:k].T


def _row_sharded(ops, k, p, Om):
    """Single pass over the rows: the local panels give Y_c rows and a partial
    A_local^T Y_c; Yhat_r is all-reduced once (include/rsvd.h rsvd_row_stream)."""
    Yc = ops.view("N", Om)
    Yh = ops.allreduce(ops.A.T @ Yc)
    Qc, Rc = ops.orth("M", Yc)
    Bt = Yh @ np.linalg.pinv(Rc, rcond=1e-12)
    Qb, Rb = ops.orth("N", Bt)
    Uh, lam, Vht = np.linalg.svd(Rb.T)
    return Qc @ Uh[:, :k], lam[:k], Qb @ Vht.T[:, :k]


def _woolfe_sharded(ops, k, p, lc, Om, Phi_local):
    """Alg. 8: Y_r all-reduced, Phi^T Q_c all-reduced, everything on side N replicated."""
    Yc = ops.view("N", Om)
    Yr = ops.view("M", Phi_local)
    Qc, Rc = ops.orth("M", Yc)
    Qr, Rr = ops.orth("N", Yr, shifted=True)
    w = k + lc
    Qc = Qc @ np.linalg.svd(Rc)[0][:, :w]
    Ur = np.linalg.svd(Rr)[0][:, :w]
    Qr = Qr @ Ur
    Qh, Rh = np.linalg.qr(ops.cross("M", Phi_local, Qc))
    Xh = np.linalg.solve(Rh, Qh.T @ (Yr.T @ Qr))
    Ux, lam, Vxt = np.linalg.svd(Xh)
    return Qc @ Ux[:, :k], lam[:k], Qr @ Vxt.T[:, :k]


def _extended_sharded(ops, k, p, Om, Phi_local, Xr_local, Xc, variant):
    """Extended sketch: [A Omega | A Xi_c] local, Y_r all-reduced, Z = Xi_r^T (A Xi_c)
    and Xi_r^T Q_c all-reduced; the small algebra replicated."""
    Yc = ops.view("N", Om)
    W = ops.view("N", Xc)
    Yr = ops.view("M", Phi_local)
    Z = ops.cross("M", Xr_local, W)
    Qc, _ = ops.orth("M", Yc)
    Qr, _ = ops.orth("N", Yr, shifted=True)
    Uc, Tc = np.linalg.qr(ops.cross("M", Xr_local, Qc))
    Ur, Tr = np.linalg.qr(Xc.T @ Qr)
    Tcp, Trp = np.linalg.pinv(Tc, rcond=1e-12), np.linalg.pinv(Tr, rcond=1e-12)
    X = Uc.T @ Z @ Ur
    if variant == "bwz2":
        core = Tcp @ X @ Trp.T
    else:
        Ux, sx, Vxt = np.linalg.svd(X)
        core = (Tcp @ Ux[:, :k]) @ np.diag(sx[:k]) @ (Trp @ Vxt.T[:, :k]).T
    Uk, lam, Vkt = np.linalg.svd(core)
    return Qc @ Uk[:, :k], lam[:k], Qr @ Vkt.T[:, :k]


CASES = [("subspace", "C1", 2, None, None), ("subspace", "C1", 3, None, None),
         ("subspace", "C2", 4, 1200, 900), ("krylov", "C1", 4, None, None),
         ("krylov", "C2", 5, 1200, 900), ("single_pass", "C1", 1, None, None),
         ("single_pass", "C3", 1, 1500, 700), ("row", "C2", 1, 1200, 900), ("row", "C1", 1, None, None),
         ("woolfe", "C2", 1, 1200, 900), ("bwz", "C1", 1, None, None), ("bwz2", "C2", 1, 1200, 900),
         ("subspace_n", "C2", 4, 1200, 900), ("subspace_n", "C1", 3, None, None), ("krylov_n", "C2", 5, 1200, 900),
         ("krylov_n", "C2", 4, 1200, 901)]


def _one_case(rank, world, case):
    alg, name, v, mm, nn = case
    cfg = S.CONFIGS[name]
    A = S.make_matrix(cfg, mm, nn)
    Om = S.gaussian_test_matrix(A.shape[1], cfg.l, cfg, S.ROLE_OMEGA)
    Phi = S.gaussian_test_matrix(A.shape[0], cfg.l2, cfg, S.ROLE_PHI)
    sh = shard_rows(A.shape[0], world, rank)
    nshard = alg.endswith("_n")
    alg = alg[:-2] if nshard else alg
    A_l = A[sh.row0:sh.row0 + sh.m_local]
    ops = ShardedOpsN(A_l, A.shape[1], world, rank) if nshard else ShardedOps(A_l)
    Phi_l = Phi[sh.row0:sh.row0 + sh.m_local]
    s_ext = min(A.shape[0], A.shape[1], 2 * cfg.l)
    Xr, Xc = S.srft_matrix(A.shape[0], s_ext, 7), S.srft_matrix(A.shape[1], s_ext, 8)
    lc = cfg.p // 2
    if alg == "subspace":
        U, s, V = _alg2_sharded(ops, cfg.k, cfg.p, v, Om)
    elif alg == "krylov":
        U, s, V = _alg9_sharded(ops, cfg.k, cfg.p, v, Om)
    elif alg == "row":
        U, s, V = _row_sharded(ops, cfg.k, cfg.p, Om)
    elif alg == "woolfe":
        U, s, V = _woolfe_sharded(ops, cfg.k, cfg.p, lc, Om, Phi_l)
    elif alg in ("bwz", "bwz2"):
        U, s, V = _extended_sharded(ops, cfg.k, cfg.p, Om, Phi_l, Xr[sh.row0:sh.row0 + sh.m_local], Xc, alg)
    else:
        U, s, V = _alg7_sharded(ops, cfg.k, cfg.p, Om, Phi_l)
    parts = [None] * world
    dist.all_gather_object(parts, U)
    res = {}
    if rank == 0:
        Ug = np.vstack(parts)
        if alg == "row":
            Uo, so, Vo = O.row_stream_qb(A, cfg.k, cfg.p, Om, panel_rows=256)
        elif alg == "woolfe":
            Uo, so, Vo = O.one_view_woolfe(A, cfg.k, cfg.p, cfg.l2 - cfg.k, lc, Om, Phi)
        elif alg in ("bwz", "bwz2"):
            Uo, so, Vo = O.one_view_extended(A, cfg.k, cfg.p, cfg.l2 - cfg.k, Om, Phi, Xr, Xc, variant=alg)
        else:
            Uo, so, Vo, _ = O.svd_of(A, alg, cfg.k, cfg.p, v=v, Omega=Om, l2=cfg.l2, Phi=Phi)
        res["sig"] = float(np.max(np.abs(s - so) / so))
        res["pu"] = O.projector_distance(Ug, Uo)
        res["pv"] = O.projector_distance(V, Vo)
    sv = [None] * world                         # replicated outputs: bitwise identical on all ranks
    dist.all_gather_object(sv, (s.tobytes(), V.tobytes()))
    res["replicated_equal"] = all(x == sv[0] for x in sv)
    return res


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        uid = os.urandom(128) if rank == 0 else None
        got = broadcast_uid(uid, rank)
        t = torch.tensor(list(got), dtype=torch.float64)
        lst = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(lst, t)
        res["uid_equal"] = all(torch.equal(lst[0], x) for x in lst)
        res["max"] = max_over_ranks(float(rank + 1) * 1.5)
        res["cases"] = [_one_case(rank, world, c) for c in CASES]
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def gloo_results():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return res


def test_gloo_uid_broadcast_and_max(gloo_results):
    assert gloo_results[0]["uid_equal"] and gloo_results[1]["uid_equal"]
    assert gloo_results[0]["max"] == gloo_results[1]["max"] == 3.0


@pytest.mark.parametrize("idx", range(len(CASES)), ids=[f"{c[0]}-{c[1]}-v{c[2]}" for c in CASES])
def test_row_sharded_schedule_matches_oracle(gloo_results, idx):
    r0 = gloo_results[0]["cases"][idx]
    assert r0["sig"] <= 1e-10 and r0["pu"] <= 1e-9 and r0["pv"] <= 1e-9, r0
    assert r0["replicated_equal"] and gloo_results[1]["cases"][idx]["replicated_equal"]
