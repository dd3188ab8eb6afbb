"""Thin ctypes binding of librsvd.so (include/rsvd.h).  Argument marshalling only: every step
of the randomized-SVD path runs in the library's CUDA kernels.  There is no CPU fallback — if
the shared library cannot be loaded, every entry point raises.

Tensors: A is a row-major (m, n) float64 tensor (CUDA or CPU/pinned).  Tall-skinny arguments are
(rows, w) tensors; they are passed column-major (each column contiguous) — a tensor with
stride (1, ld) is passed as is, anything else is copied to that layout first.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librsvd.so")

RSVD_F32, RSVD_F64 = 1, 2
RSVD_INPUT_A, RSVD_INPUT_AT = 0, 1
RSVD_GOAL_SVD, RSVD_GOAL_LEFT, RSVD_GOAL_RIGHT, RSVD_GOAL_NORMAL = 0, 1, 2, 3
RSVD_SQUARED, RSVD_NO_GRAPH, RSVD_PROFILE, RSVD_CORE_NO_J, RSVD_ASYNC, RSVD_WOOLFE = 1, 2, 4, 16, 32, 64
RSVD_ORTH_SHIFTED = 128
RSVD_ONE_READ = 256
RSVD_LC_MINVAR = -2
RSVD_EXT_BWZ, RSVD_EXT_BWZ2 = 0, 1
RSVD_PLAN_FLAT, RSVD_PLAN_DECAY, RSVD_PLAN_RAPID, RSVD_PLAN_BALANCED = 0, 1, 2, 3
ERR = {0: "RSVD_OK", -1: "RSVD_E_ARG", -2: "RSVD_E_DTYPE", -3: "RSVD_E_CUDA", -4: "RSVD_E_NCCL",
       -5: "RSVD_E_NOMEM", -6: "RSVD_E_NUMERIC", -7: "RSVD_E_STATE"}

EXPORTS = ["rsvd_create", "rsvd_destroy", "rsvd_wait", "rsvd_strerror", "rsvd_last_error", "rsvd_version", "rsvd_sm_count",
           "rsvd_recommend_input", "rsvd_probe_peaks", "rsvd_get_unique_id", "rsvd_comm_init", "rsvd_comm_nranks", "rsvd_subspace",
           "rsvd_block_krylov", "rsvd_single_pass", "rsvd_nystrom", "rsvd_pinched", "rsvd_view", "rsvd_view_fused",
           "rsvd_orth", "rsvd_core_svd", "rsvd_plan", "rsvd_single_pass_extended",
           "rsvd_row_stream", "rsvd_set_sm_limit", "rsvd_loop_create", "rsvd_loop_destroy",
           "rsvd_comm_init_loopback", "rsvd_block_krylov_rows"]


class RsvdMat(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int32), ("reserved", ctypes.c_int32), ("m", ctypes.c_int64),
                ("n", ctypes.c_int64), ("m_local", ctypes.c_int64), ("row0", ctypes.c_int64),
                ("lda", ctypes.c_int64), ("data", ctypes.c_void_p)]


class RsvdInfo(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("views", ctypes.c_int32), ("vectors", ctypes.c_int64),
                ("rank_deficient_cols", ctypes.c_int32), ("jacobi_sweeps", ctypes.c_int32),
                ("lc_used", ctypes.c_int32), ("host_staged", ctypes.c_int32), ("graph_replayed", ctypes.c_int32),
                ("nondeterministic", ctypes.c_int32), ("view_launches", ctypes.c_int32),
                ("kernel_launches", ctypes.c_int32), ("view_ms", ctypes.c_double), ("view_bytes", ctypes.c_double),
                ("view_flops", ctypes.c_double), ("total_ms", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "reserved"}


class RsvdError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERR.get(code, code)}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load librsvd.so (fail loudly if it is missing: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -m paper_1804_07531_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint
    pinfo = ctypes.POINTER(RsvdInfo)
    pmat = ctypes.POINTER(RsvdMat)
    L.rsvd_create.argtypes = [ctypes.POINTER(vp), i32, vp]
    L.rsvd_destroy.argtypes = [vp]
    L.rsvd_strerror.argtypes = [i32]
    L.rsvd_strerror.restype = ctypes.c_char_p
    L.rsvd_last_error.argtypes = [vp]
    L.rsvd_last_error.restype = ctypes.c_char_p
    L.rsvd_sm_count.argtypes = [vp]
    L.rsvd_set_sm_limit.argtypes = [vp, i32]
    L.rsvd_wait.argtypes = [vp, pinfo]
    L.rsvd_recommend_input.argtypes = [i32, i32]
    L.rsvd_get_unique_id.argtypes = [vp]
    L.rsvd_probe_peaks.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    L.rsvd_comm_init.argtypes = [vp, i32, i32, vp]
    L.rsvd_comm_nranks.argtypes = [vp]
    L.rsvd_loop_create.argtypes = [i32, ctypes.c_double, ctypes.POINTER(vp)]
    L.rsvd_loop_destroy.argtypes = [vp]
    L.rsvd_comm_init_loopback.argtypes = [vp, vp, i32]
    alg = [vp, pmat, i32, i32, i32, i32, vp, i64, vp, i64, vp, vp, i64, u32, pinfo]
    L.rsvd_subspace.argtypes = alg
    L.rsvd_block_krylov.argtypes = alg
    L.rsvd_plan.argtypes = [i32, i32, i32, ctypes.c_double, ctypes.POINTER(i32), ctypes.POINTER(i32),
                            ctypes.POINTER(i32)]
    L.rsvd_single_pass_extended.argtypes = [vp, pmat, i32, i32, i32, i32, vp, i64, vp, i64, vp, i64, vp, i64, i32,
                                            vp, i64, vp, vp, i64, u32, pinfo]
    L.rsvd_row_stream.argtypes = [vp, pmat, i32, i32, vp, i64, vp, i64, vp, vp, i64, u32, pinfo]
    L.rsvd_block_krylov_rows.argtypes = [vp, pmat, i32, i32, i32, vp, i64, vp, i64, vp, vp, i64, u32, pinfo]
    L.rsvd_single_pass.argtypes = [vp, pmat, i32, i32, i32, i32, vp, i64, vp, i64, vp, i64, vp, vp, i64, u32, pinfo]
    L.rsvd_nystrom.argtypes = [vp, pmat, i32, i32, i32, vp, i64, vp, vp, i64, u32, pinfo]
    L.rsvd_pinched.argtypes = [vp, pmat, i32, i32, i32, vp, i64, vp, vp, i64, u32, pinfo]
    L.rsvd_view.argtypes = [vp, pmat, i32, vp, i64, i32, vp, i64, u32, pinfo]
    L.rsvd_view_fused.argtypes = [vp, pmat, vp, i64, i32, vp, i64, i32, vp, i64, vp, i64, u32, pinfo]
    L.rsvd_orth.argtypes = [vp, i64, i32, vp, i64, vp, u32, pinfo]
    L.rsvd_core_svd.argtypes = [vp, i32, i32, vp, i64, vp, vp, vp, u32, pinfo]
    _lib = L
    return L


def recommend_input(goal: int, v: int) -> int:
    return lib().rsvd_recommend_input(goal, v)


def plan(scheme: int, k: int, T: int, alpha: float = 0.5):
    """rsvd_plan: single-pass oversampling from the budget T = 2k + l_1 + l_2.
    Returns the ABI arguments (p, l2, lc) of rsvd_single_pass."""
    p, l2, lc = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    rc = lib().rsvd_plan(scheme, k, T, alpha, ctypes.byref(p), ctypes.byref(l2), ctypes.byref(lc))
    if rc != 0:
        raise RsvdError(rc, "rsvd_plan: T >= 2k + 6, k >= 1 and 0 <= alpha <= 1 required")
    return p.value, l2.value, lc.value


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = lib().rsvd_get_unique_id(buf)
    if rc:
        raise RsvdError(rc, "rsvd_get_unique_id")
    return buf.raw


def _colmajor(t: torch.Tensor) -> torch.Tensor:
    """(rows, w) tensor in column-major layout (stride (1, ld))."""
    if t.dim() == 1:
        t = t[:, None]
    if t.stride(0) == 1 and (t.shape[1] == 1 or t.stride(1) >= t.shape[0]):
        return t
    return t.t().contiguous().t()


def _ld(t: torch.Tensor) -> int:
    return t.stride(1) if t.shape[1] > 1 else max(t.shape[0], 1)


def _new_colmajor(rows, cols, like: torch.Tensor, pin=False):
    if like.is_cuda:
        return torch.empty((cols, rows), dtype=like.dtype, device=like.device).t()
    return torch.empty((cols, rows), dtype=like.dtype, pin_memory=pin).t()


class LoopGroup:
    """rsvd_loop: N virtual row shards of one A on one GPU (the sharded path without N GPUs).
    Each member Context joins with ``ctx.comm_init_loopback(group, rank)`` and must be driven by
    its own thread (every rank makes the same calls, as with NCCL)."""

    def __init__(self, nranks: int, timeout_s: float = 120.0):
        h = ctypes.c_void_p()
        rc = lib().rsvd_loop_create(nranks, timeout_s, ctypes.byref(h))
        if rc:
            raise RsvdError(rc, "rsvd_loop_create: 1 <= nranks <= 16")
        self._h = h
        self.nranks = nranks

    def close(self):
        if getattr(self, "_h", None):
            lib().rsvd_loop_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One rsvd_ctx bound to a CUDA device and a stream.

    By default the stream is torch's current stream.  When that is the legacy default stream
    (handle 0), the library creates its own BLOCKING stream, which the CUDA runtime orders with
    the default stream in both directions (rsvd_create), so inputs produced on torch's default
    stream are complete before a call starts and later default-stream work waits for the call.
    With an explicit torch stream the caller orders it (``wait_stream``) against producers."""

    def __init__(self, device: int | None = None, stream: torch.cuda.Stream | None = None):
        L = lib()
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = ctypes.c_void_p()
        rc = L.rsvd_create(ctypes.byref(h), device, ctypes.c_void_p(self.stream.cuda_stream))
        if rc:
            raise RsvdError(rc, "rsvd_create")
        self._h = h
        self.nranks = 1
        self.rank = 0

    def close(self):
        if getattr(self, "_h", None):
            lib().rsvd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def sm_count(self) -> int:
        return lib().rsvd_sm_count(self._h)

    def set_sm_limit(self, n: int):
        """Cap the SMs this context's persistent kernels are sized for (rsvd_set_sm_limit)."""
        self._check(lib().rsvd_set_sm_limit(self._h, n), "rsvd_set_sm_limit")

    def probe_peaks(self):
        """(FP64 DMMA TFLOP/s, HBM read GB/s) measured on this device."""
        t, g = ctypes.c_double(), ctypes.c_double()
        self._check(lib().rsvd_probe_peaks(self._h, ctypes.byref(t), ctypes.byref(g)), "rsvd_probe_peaks")
        return t.value, g.value

    def wait(self, info=None):
        """Complete an RSVD_ASYNC call on this context (synchronises its stream)."""
        inf = info if info is not None else RsvdInfo()
        self._check(lib().rsvd_wait(self._h, ctypes.byref(inf)), "rsvd_wait")
        return inf

    def _check(self, rc, what):
        if rc:
            raise RsvdError(rc, f"{what}: {lib().rsvd_last_error(self._h).decode()}")

    def comm_init_loopback(self, group: LoopGroup, rank: int):
        """Join a loopback group as virtual rank `rank` (rsvd_comm_init_loopback)."""
        self._check(lib().rsvd_comm_init_loopback(self._h, group._h, rank), "rsvd_comm_init_loopback")
        self.nranks, self.rank = group.nranks, rank

    def comm_init(self, nranks: int, rank: int, uid: bytes):
        """Collective: all ranks pass the same 128-byte id (rank 0's get_unique_id())."""
        buf = ctypes.create_string_buffer(uid, 128)
        self._check(lib().rsvd_comm_init(self._h, nranks, rank, buf), "rsvd_comm_init")
        self.nranks, self.rank = nranks, rank

    # ------------------------------------------------------------------ helpers
    @staticmethod
    def mat(A: torch.Tensor, m: int | None = None, row0: int = 0) -> RsvdMat:
        if A.dtype != torch.float64:
            dt = RSVD_F32 if A.dtype == torch.float32 else 0
        else:
            dt = RSVD_F64
        if A.stride(1) != 1:
            raise ValueError("A must be row-major (stride(1) == 1)")
        ml, n = A.shape
        return RsvdMat(dt, 0, m if m is not None else ml, n, ml, row0, A.stride(0), A.data_ptr())

    def _out_like(self, A, rows, cols, host_out):
        # at least one column: an invalid k must reach the C ABI, which reports RSVD_E_ARG
        cols = max(cols, 1)
        if host_out or not A.is_cuda:
            return _new_colmajor(rows, cols, A.cpu() if A.is_cuda else A, pin=True)
        return _new_colmajor(rows, cols, A)

    # ------------------------------------------------------------------ algorithms
    def _alg(self, fn, name, A, k, p, v, Omega, input=RSVD_INPUT_A, flags=0, m=None, row0=0,
             want_u=True, want_v=True, host_out=False):
        Om = _colmajor(Omega)
        M = self.mat(A, m, row0)
        U = self._out_like(A, A.shape[0], k, host_out) if want_u else None
        V = self._out_like(A, A.shape[1], k, host_out) if want_v else None
        S = (torch.empty(max(k, 1), dtype=A.dtype, pin_memory=True) if (host_out or not A.is_cuda)
             else torch.empty(max(k, 1), dtype=A.dtype, device=A.device))
        info = RsvdInfo()
        rc = fn(self._h, ctypes.byref(M), k, p, v, input, Om.data_ptr(), _ld(Om),
                U.data_ptr() if U is not None else None, _ld(U) if U is not None else 0, S.data_ptr(),
                V.data_ptr() if V is not None else None, _ld(V) if V is not None else 0, flags, ctypes.byref(info))
        self._check(rc, name)
        return U, S, V, info

    def subspace(self, A, k, p, v, Omega, input=RSVD_INPUT_A, flags=0, **kw):
        """Alg. 2.  Returns (U, S, V, info) of A."""
        return self._alg(lib().rsvd_subspace, "rsvd_subspace", A, k, p, v, Omega, input, flags, **kw)

    def block_krylov(self, A, k, p, v, Omega, input=RSVD_INPUT_A, flags=0, **kw):
        """Alg. 9."""
        return self._alg(lib().rsvd_block_krylov, "rsvd_block_krylov", A, k, p, v, Omega, input, flags, **kw)

    def single_pass(self, A, k, p, l2, Omega, Phi, lc=-1, flags=0, m=None, row0=0, host_out=False):
        """Alg. 7.  lc = -1 -> lc = p (Tropp baseline); lc = "minvar" (RSVD_LC_MINVAR) ->
        minimum-variance l_c chosen on the device, returned in info.lc_used.
        flags | RSVD_WOOLFE -> Alg. 8."""
        if lc == "minvar":
            lc = RSVD_LC_MINVAR
        Om, Ph = _colmajor(Omega), _colmajor(Phi)
        M = self.mat(A, m, row0)
        U = self._out_like(A, A.shape[0], k, host_out)
        V = self._out_like(A, A.shape[1], k, host_out)
        S = (torch.empty(max(k, 1), dtype=A.dtype, pin_memory=True) if (host_out or not A.is_cuda)
             else torch.empty(max(k, 1), dtype=A.dtype, device=A.device))
        info = RsvdInfo()
        rc = lib().rsvd_single_pass(self._h, ctypes.byref(M), k, p, l2, lc, Om.data_ptr(), _ld(Om), Ph.data_ptr(),
                                    _ld(Ph), U.data_ptr(), _ld(U), S.data_ptr(), V.data_ptr(), _ld(V), flags,
                                    ctypes.byref(info))
        self._check(rc, "rsvd_single_pass")
        return U, S, V, info

    def single_pass_extended(self, A, k, p, l2, s, Omega, Phi, Xi_r, Xi_c, variant="bwz2", flags=0, m=None,
                             row0=0, host_out=False):
        """Extended 1-view sketch: Xi_r (m x s), Xi_c (n x s) are the SRFT test matrices;
        variant "bwz" (Eq. bwz) or "bwz2" (Eq. bwzimproved)."""
        var = {"bwz": RSVD_EXT_BWZ, "bwz2": RSVD_EXT_BWZ2}[variant] if isinstance(variant, str) else variant
        Om, Ph, Xr, Xc = _colmajor(Omega), _colmajor(Phi), _colmajor(Xi_r), _colmajor(Xi_c)
        M = self.mat(A, m, row0)
        U = self._out_like(A, A.shape[0], k, host_out)
        V = self._out_like(A, A.shape[1], k, host_out)
        S = (torch.empty(max(k, 1), dtype=A.dtype, pin_memory=True) if (host_out or not A.is_cuda)
             else torch.empty(max(k, 1), dtype=A.dtype, device=A.device))
        info = RsvdInfo()
        rc = lib().rsvd_single_pass_extended(self._h, ctypes.byref(M), k, p, l2, s, Om.data_ptr(), _ld(Om),
                                             Ph.data_ptr(), _ld(Ph), Xr.data_ptr(), _ld(Xr), Xc.data_ptr(), _ld(Xc),
                                             var, U.data_ptr(), _ld(U), S.data_ptr(), V.data_ptr(), _ld(V), flags,
                                             ctypes.byref(info))
        self._check(rc, "rsvd_single_pass_extended")
        return U, S, V, info

    def block_krylov_rows(self, A, k, p, v, Omega, flags=0, m=None, row0=0, host_out=False):
        """Block Krylov with A^T A X from one pass over the rows; info.views = reads of A."""
        Om = _colmajor(Omega)
        M = self.mat(A, m, row0)
        U = self._out_like(A, A.shape[0], k, host_out)
        V = self._out_like(A, A.shape[1], k, host_out)
        S = (torch.empty(max(k, 1), dtype=A.dtype, pin_memory=True) if (host_out or not A.is_cuda)
             else torch.empty(max(k, 1), dtype=A.dtype, device=A.device))
        info = RsvdInfo()
        rc = lib().rsvd_block_krylov_rows(self._h, ctypes.byref(M), k, p, v, Om.data_ptr(), _ld(Om), U.data_ptr(),
                                          _ld(U), S.data_ptr(), V.data_ptr(), _ld(V), flags, ctypes.byref(info))
        self._check(rc, "rsvd_block_krylov_rows")
        return U, S, V, info

    def row_stream(self, A, k, p, Omega, flags=0, m=None, row0=0, host_out=False):
        """Single pass over the rows of A; equals subspace(v=2) when R_c is invertible."""
        Om = _colmajor(Omega)
        M = self.mat(A, m, row0)
        U = self._out_like(A, A.shape[0], k, host_out)
        V = self._out_like(A, A.shape[1], k, host_out)
        S = (torch.empty(max(k, 1), dtype=A.dtype, pin_memory=True) if (host_out or not A.is_cuda)
             else torch.empty(max(k, 1), dtype=A.dtype, device=A.device))
        info = RsvdInfo()
        rc = lib().rsvd_row_stream(self._h, ctypes.byref(M), k, p, Om.data_ptr(), _ld(Om), U.data_ptr(), _ld(U),
                                   S.data_ptr(), V.data_ptr(), _ld(V), flags, ctypes.byref(info))
        self._check(rc, "rsvd_row_stream")
        return U, S, V, info

    def _normal(self, fn, name, A, k, p, v, Omega, flags=0, m=None, row0=0, host_out=False):
        Om = _colmajor(Omega)
        M = self.mat(A, m, row0)
        V = self._out_like(A, A.shape[1], k, host_out)
        S = (torch.empty(max(k, 1), dtype=A.dtype, pin_memory=True) if (host_out or not A.is_cuda)
             else torch.empty(max(k, 1), dtype=A.dtype, device=A.device))
        info = RsvdInfo()
        self._check(fn(self._h, ctypes.byref(M), k, p, v, Om.data_ptr(), _ld(Om), S.data_ptr(), V.data_ptr(), _ld(V),
                       flags, ctypes.byref(info)), name)
        return S, V, info

    def nystrom(self, A, k, p, v, Omega, **kw):
        """Alg. 4: A^T A ~ V diag(S) V^T.  Omega: n x (k+p) for even v, m x (k+p) for odd v."""
        return self._normal(lib().rsvd_nystrom, "rsvd_nystrom", A, k, p, v, Omega, **kw)

    def pinched(self, A, k, p, v, Omega, **kw):
        """Alg. 5: A^T A ~ V diag(S) V^T.  Omega: m x (k+p) for even v, n x (k+p) for odd v."""
        return self._normal(lib().rsvd_pinched, "rsvd_pinched", A, k, p, v, Omega, **kw)

    # ------------------------------------------------------------------ primitives
    def view(self, A, X, trans=False, flags=0):
        X = _colmajor(X)
        M = self.mat(A)
        rows = A.shape[1] if trans else A.shape[0]
        Y = _new_colmajor(rows, X.shape[1], A) if A.is_cuda else _new_colmajor(rows, X.shape[1], A, pin=True)
        info = RsvdInfo()
        self._check(lib().rsvd_view(self._h, ctypes.byref(M), int(trans), X.data_ptr(), _ld(X), X.shape[1],
                                    Y.data_ptr(), _ld(Y), flags, ctypes.byref(info)), "rsvd_view")
        return Y, info

    def view_fused(self, A, Omega, Phi, flags=0):
        Om, Ph = _colmajor(Omega), _colmajor(Phi)
        M = self.mat(A)
        Yc = _new_colmajor(A.shape[0], Om.shape[1], A)
        Yr = _new_colmajor(A.shape[1], Ph.shape[1], A)
        info = RsvdInfo()
        self._check(lib().rsvd_view_fused(self._h, ctypes.byref(M), Om.data_ptr(), _ld(Om), Om.shape[1],
                                          Ph.data_ptr(), _ld(Ph), Ph.shape[1], Yc.data_ptr(), _ld(Yc),
                                          Yr.data_ptr(), _ld(Yr), flags, ctypes.byref(info)), "rsvd_view_fused")
        return Yc, Yr, info

    def orth(self, Y, flags=0):
        """CholeskyQR2, or shifted CholeskyQR3 with flags | RSVD_ORTH_SHIFTED (returns a new Q and
        R; the input is not modified)."""
        Q = _colmajor(Y).clone() if _colmajor(Y).data_ptr() == Y.data_ptr() else _colmajor(Y)
        Q = Q.t().contiguous().t()
        w = Q.shape[1]
        R = torch.empty((w, w), dtype=Q.dtype, device=Q.device).t()
        info = RsvdInfo()
        self._check(lib().rsvd_orth(self._h, Q.shape[0], w, Q.data_ptr(), _ld(Q), R.data_ptr(), flags,
                                    ctypes.byref(info)), "rsvd_orth")
        return Q, R, info

    def core_svd(self, Mx, flags=0):
        Mx = _colmajor(Mx)
        r, c = Mx.shape
        U = torch.empty((c, r), dtype=Mx.dtype, device=Mx.device).t()
        S = torch.empty(c, dtype=Mx.dtype, device=Mx.device)
        V = torch.empty((c, c), dtype=Mx.dtype, device=Mx.device).t()
        info = RsvdInfo()
        self._check(lib().rsvd_core_svd(self._h, r, c, Mx.data_ptr(), _ld(Mx), U.data_ptr(), S.data_ptr(),
                                        V.data_ptr(), flags, ctypes.byref(info)), "rsvd_core_svd")
        return U, S, V, info
