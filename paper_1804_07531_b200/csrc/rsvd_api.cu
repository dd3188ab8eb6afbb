// C-ABI driver of librsvd: context, workspace arena, CUDA-graph cache, NCCL row-sharding and
// the algorithms of arXiv 1804.07531 expressed as sequences of device kernels.
//
//   Alg. 2  generalized subspace iteration
//   Alg. 9  generalized block Krylov
//   Alg. 7  1-view (Tropp variant, l_c)
//
// Every algorithm is enqueued on the ctx stream with no host round trip; the first call with a
// given signature is captured into a CUDA graph, later calls replay it.  The workspace is sized
// by running the same enqueue code in "dry" mode (allocations only, no launches).
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "comm.h"
#include "internal.h"

namespace rsvd {
bool chol_reads_upper_only(int w);
int launch_chol_ref(const double* G, const double* ref, int w, double tol, double* R, double* Rinv,
                    DevStatus* status, cudaStream_t st, double shift_coef = 0.0);
int launch_jacobi_t(const double* M, int64_t ldm, int trans, int r, int c, double* Ul, double* S, double* Vr,
                    double* scratch, DevStatus* status, cudaStream_t st, int want_j);
int launch_diag(const double* G, int w, double* d, cudaStream_t st);
int probe_peaks(int sms, cudaStream_t st, double* dmma_tflops, double* read_gbs);
int cholqr_pass_ctas(int64_t rows);
bool orth_cluster_fits(int64_t rows, int w);
int launch_orth_cluster(double* Y, int64_t ldy, int64_t rows, int w, int shifted, double shift_coef, double* Rout,
                        double* Rw /* 3 w*w scratch */, DevStatus* status, cudaStream_t st);
int launch_cholqr_pass(const double* Yin, int64_t ldi, double* Yout, int64_t ldo, int64_t rows, int w,
                       const double* Rin, double* slots, unsigned* counter, double tol, double shift_coef,
                       int second_pass, double* R, double* Rinv, DevStatus* status, cudaStream_t st);
}  // namespace rsvd

using namespace rsvd;

// ================================================================ context
struct rsvd_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  Comm* comm = nullptr;        // rsvd_comm_init (NCCL) or rsvd_comm_init_loopback; null: single GPU
  int nranks = 1, rank = 0;
  char* arena = nullptr;
  size_t arena_size = 0;
  DevStatus* dstat = nullptr;
  DevStatus* hstat = nullptr;  // pinned
  unsigned* counter = nullptr; // arrival counter of the last-CTA finisher kernels (self-resetting)
  std::map<std::string, cudaGraphExec_t> graphs;
  std::map<std::string, int> graph_kernels;  // kernel nodes per cached graph
  std::vector<cudaEvent_t> events;
  std::string err;
  // RSVD_ASYNC: the call's host-side results, completed by rsvd_wait
  bool pending = false;
  rsvd_info pending_info;
};

namespace {

void set_err(rsvd_ctx* c, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
}

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// debug / A-B switches read once from the environment (e.g. RSVD_NO_ORTH_CLUSTER=1)
bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && v[0] && v[0] != '0';
}

enum Side { SIDE_M = 0, SIDE_N = 1 };

struct TS {  // column-major tall-skinny block: w columns of `rows`, leading dim ld
  double* p = nullptr;
  int64_t rows = 0, ld = 0;
  int w = 0;
};

enum PtrKind { PTR_NULL = 0, PTR_DEVICE = 1, PTR_HOST = 2 };

PtrKind ptr_kind(const void* p, int device) {
  if (!p) return PTR_NULL;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return PTR_HOST;
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return PTR_DEVICE;
  (void)device;
  return PTR_HOST;
}

// ---------------------------------------------------------------- call description
struct Call {
  int alg = 0;  // 0 subspace, 1 krylov, 2 single pass, 10 view, 11 fused view, 12 orth, 13 core svd
  const rsvd_mat* A = nullptr;
  int k = 0, p = 0, v = 0, input = 0, l2 = 0, lc = 0, trans = 0, w = 0;
  int64_t rows = 0;  // orth / core
  int cols = 0;
  const void* Om = nullptr;
  int64_t ldom = 0;
  const void* Phi = nullptr;
  int64_t ldphi = 0;
  void* U = nullptr;
  int64_t ldu = 0;
  void* S = nullptr;
  void* V = nullptr;
  int64_t ldv = 0;
  void* R = nullptr;
  unsigned flags = 0;
  // extended 1-view sketch (alg 5): SRFT test matrices Xi_r (m_local x s), Xi_c (n x s), variant
  int s = 0, variant = 0;
  const void* Xr = nullptr;
  int64_t ldxr = 0;
  const void* Xc = nullptr;
  int64_t ldxc = 0;
  // info fields known at enqueue time (also what rsvd_wait reports for RSVD_ASYNC calls)
  int info_views = 0, info_lc = 0;
  int64_t info_vectors = 0;
  // resolved kinds
  PtrKind kA = PTR_NULL, kOm = PTR_NULL, kPhi = PTR_NULL, kU = PTR_NULL, kS = PTR_NULL, kV = PTR_NULL,
          kR = PTR_NULL, kXr = PTR_NULL, kXc = PTR_NULL;
};

// ---------------------------------------------------------------- executor
struct Exec {
  rsvd_ctx* ctx;
  const Call& call;
  bool dry;
  char* base;
  size_t off = 0, peak = 0;
  cudaStream_t st;
  int rc = RSVD_OK;
  bool profile = false;
  bool launch_off = false;  // real addresses, record transfers, launch nothing
  int a_restaged = 0;
  int nondet = 0;
  bool live() const { return !dry && !launch_off && rc == RSVD_OK; }
  std::vector<std::pair<int, int>> ev_pairs;  // indices into ctx->events
  int ev_used = 0;
  double view_bytes = 0, view_flops = 0;
  int view_launches = 0;
  // device views of the caller's arrays (resolved in prepare)
  const double* A = nullptr;
  const float* A32 = nullptr;   // dtype == RSVD_F32: A itself (every internal block stays fp64)
  int dtype = RSVD_F64;
  int64_t lda = 0, m = 0, n = 0;
  int64_t m_glob = 0;   // global row count of A (m = this rank's rows)
  // n-side sharding (Alg. 2 / 9 under a communicator of N > 1 ranks): side-N blocks
  // hold only this rank's chunk of rows [n0, n0 + n_loc) of the n-long side, stored with ld = n_cs
  // (the chunk size, a multiple of 32, equal on every rank).  A^T Y is a local full-length partial
  // followed by a reduce-scatter; A X first all-gathers X; Grams of side-N blocks are all-reduced.
  bool shard_n = false;
  int64_t n_cs = 0, n0 = 0, n_loc = 0;
  // host-transfer plan (executed outside the graph); esz = element bytes (8, or 4 for fp32)
  struct H2D { void* dst; int64_t ldd; const void* src; int64_t lds; int64_t rows; int64_t cols; int esz = 8; };
  struct D2H { void* dst; int64_t ldd; const void* src; int64_t lds; int64_t rows; int64_t cols; int esz = 8; };
  std::vector<H2D> h2d;
  std::vector<D2H> d2h;
  // fp32 outputs: fp64 result block -> fp32 staging block, converted at the end of the algorithm
  struct Narrow { const double* src; int64_t lds; float* dst; int64_t ldd; int64_t rows; int cols; };
  std::vector<Narrow> narrow;
  float* alloc_f(int64_t n_el) { return reinterpret_cast<float*>(alloc((n_el + 1) / 2)); }
  void flush_outputs() {
    for (auto& t : narrow)
      if (live()) chk(launch_f64_to_f32(t.src, t.lds, t.dst, t.ldd, t.rows, t.cols, st));
    narrow.clear();
  }

  Exec(rsvd_ctx* c, const Call& cl, bool d, char* b) : ctx(c), call(cl), dry(d), base(b), st(c->stream) {}

  double* alloc(int64_t n_el) {
    const size_t bytes = (size_t)round_up(std::max<int64_t>(n_el, 1) * 8, 256);
    char* p = (dry ? (char*)(uintptr_t)0x100000 : base) + off;
    off += bytes;
    peak = std::max(peak, off);
    return reinterpret_cast<double*>(p);
  }
  size_t mark() const { return off; }
  void release(size_t m_) { off = m_; }
  void chk(int r) {
    if (rc == RSVD_OK && r != RSVD_OK) rc = r;
  }
  int64_t side_rows(Side s) const { return s == SIDE_M ? m : (shard_n ? n_loc : n); }
  // global length of a side (sharded or not)
  int64_t side_rows_glob(Side s) const { return s == SIDE_M ? m_glob : n; }
  TS new_ts(Side s, int w) {
    TS t;
    t.rows = side_rows(s);
    t.ld = (s == SIDE_N && shard_n) ? n_cs : round_up(std::max<int64_t>(t.rows, 1), 32);
    t.w = w;
    t.p = alloc(t.ld * w);
    return t;
  }
  TS slice(const TS& t, int c0, int wc) const {
    TS s = t;
    s.p = t.p + (int64_t)c0 * t.ld;
    s.w = wc;
    return s;
  }
  // a communicator exists (rsvd_comm_init; also with one rank, which runs the sharded code path
  // on one GPU: sharded CholeskyQR, all-reduced Grams and A^T Y partials, NCCL in the graph)
  bool collective() const { return ctx->comm != nullptr; }
  bool sharded(Side s) const { return s == SIDE_M ? collective() : shard_n; }
  // enable n-side sharding for this call (after bind_A): every rank must own >= 1 row of side N
  void plan_shard_n() {
    shard_n = false;
    if (!collective() || ctx->nranks < 2 || getenv_flag("RSVD_NO_SHARD_N")) return;
    const int N = ctx->nranks;
    const int64_t cs = round_up((n + N - 1) / N, 32);
    if ((N - 1) * cs >= n) return;
    shard_n = true;
    n_cs = cs;
    n0 = (int64_t)ctx->rank * cs;
    n_loc = std::min<int64_t>(cs, n - n0);
  }
  // full (n x w) copy of an n-sharded side-N block: all-gather of the chunks
  TS gather_n(const TS& X) {
    TS F;
    F.rows = n;
    F.ld = round_up(n, 32);
    F.w = X.w;
    F.p = alloc(F.ld * X.w);
    gather_n_into(X, F.p, F.ld);
    return F;
  }
  void gather_n_into(const TS& X, double* dst, int64_t ldd) {
    double* buf = alloc(n_cs * X.w * ctx->nranks);
    if (!live()) return;
    std::string e;
    const int r = ctx->comm->allgather(X.p, buf, (size_t)(n_cs * X.w), st, &e);
    if (r != RSVD_OK) {
      set_err(ctx, "%s", e.c_str());
      chk(r);
      return;
    }
    chk(launch_rows_chunk(dst, ldd, n, buf, n_cs, ctx->nranks, X.w, 0, st));
  }
  // Y (this rank's chunk, ld n_cs) = sum over ranks of the full-length partials F, chunk n0
  void reduce_scatter_n(const TS& F, const TS& Y) {
    double* buf = alloc(n_cs * F.w * ctx->nranks);
    if (!live()) return;
    chk(launch_rows_chunk(F.p, F.ld, n, buf, n_cs, ctx->nranks, F.w, 1, st));
    std::string e;
    const int r = ctx->comm->reduce_scatter(buf, Y.p, (size_t)(n_cs * F.w), st, &e);
    if (r != RSVD_OK) {
      set_err(ctx, "%s", e.c_str());
      chk(r);
    }
  }

  void allreduce(double* p, int64_t count) {
    if (!live()) return;
    std::string e;
    const int r = ctx->comm->allreduce(p, (size_t)count, st, &e);
    if (r != RSVD_OK) {
      set_err(ctx, "%s", e.c_str());
      chk(r);
    }
  }
  void ev_record(int* idx) {
    if (!live() || !profile) return;
    if (ev_used >= (int)ctx->events.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ctx->events.push_back(e);
    }
    *idx = ev_used++;
    cudaEventRecord(ctx->events[*idx], st);
  }

  // ------------------------------------------------------------ matrix views (hot path)
  // from == SIDE_N: Y (side M) = A X;  from == SIDE_M: Y (side N) = A^T X (+ all-reduce)
  // One view of A (or, with nr >= 0, of its row panel [r0, r0 + nr): then Y / X are the panel's
  // row slices, nothing is all-reduced, and a_keep loads the panel with evict_last for a re-read).
  void view(Side from, const TS& X, const TS& Y, int64_t r0 = 0, int64_t nr = -1, int a_keep = 0) {
    if (shard_n && nr < 0) {
      const size_t mk = mark();
      if (from == SIDE_N) {                  // A X: X all-gathered to full length first
        TS F = gather_n(X);
        view_local(from, F, Y, 0, -1, 0, false);
      } else {                               // A^T Y: full-length local partial, reduce-scatter
        TS F;
        F.rows = n;
        F.ld = round_up(n, 32);
        F.w = Y.w;
        F.p = alloc(F.ld * Y.w);
        view_local(from, X, F, 0, -1, 0, false);
        reduce_scatter_n(F, Y);
      }
      release(mk);
      return;
    }
    view_local(from, X, Y, r0, nr, a_keep, true);
  }
  void view_local(Side from, const TS& X, const TS& Y, int64_t r0, int64_t nr, int a_keep, bool reduce) {
    const bool panel = nr >= 0;
    const int64_t rows_v = panel ? nr : m;
    if (dtype == RSVD_F32) {
      view32(from, X, Y, r0, nr, reduce);
      return;
    }
    const int w = X.w;
    // balanced column chunks of <= kMaxWT * 8 (each chunk streams A once: w = 140 as 72 + 68, two
    // tensor-bound launches, not 128 + an HBM-bound 12)
    const int nchunk = (w + kMaxWT * 8 - 1) / (kMaxWT * 8);
    const int cw = std::min(kMaxWT * 8, ((w + nchunk - 1) / nchunk + 7) / 8 * 8);
    for (int c0 = 0; c0 < w; c0 += cw) {
      const int wc = std::min(cw, w - c0);
      const size_t mk = mark();
      ViewArgs a;
      a.A = A + (panel ? r0 * lda : 0);
      a.rows = rows_v;
      a.n = n;
      a.lda = lda;
      a.a_keep = a_keep;
      a.X = X.p + (int64_t)c0 * X.ld;
      a.ldx = X.ld;
      a.w = wc;
      a.grid_cap = ctx->sms;
      const int kind = (from == SIDE_N) ? VIEW_AX : VIEW_ATY;
      plan_view(kind, rows_v, n, wc, ctx->sms, &a.S, &a.KTS);
      double* dst = Y.p + (int64_t)c0 * Y.ld;
      double* slots = (a.S == 1) ? dst : alloc((int64_t)a.S * Y.ld * wc);
      a.out = slots;
      a.ldo = Y.ld;
      a.slot_stride = (int64_t)Y.ld * wc;
      view_bytes += (double)rows_v * n * 8.0;
      view_flops += 2.0 * rows_v * n * wc;
      ++view_launches;
      if (live()) {
        int e0 = -1, e1 = -1;
        nvtxRangePushA(kind == VIEW_AX ? "view A*X" : "view A^T*Y");
        ev_record(&e0);
        chk(kind == VIEW_AX ? launch_view_ax(a, st) : launch_view_aty(a, st));
        nvtxRangePop();
        ev_record(&e1);
        if (e0 >= 0) ev_pairs.push_back({e0, e1});
        if (a.S > 1) chk(launch_slot_sum(slots, Y.ld, a.slot_stride, a.S, Y.rows, wc, dst, Y.ld, st));
      }
      release(mk);
    }
    if (from == SIDE_M && collective() && !panel && reduce) allreduce(Y.p, Y.ld * Y.w);
  }

  // fp32 A: split X into tf32 hi / lo parts, tcgen05 3xTF32 view into fp64 partial slots
  void view32(Side from, const TS& X, const TS& Y, int64_t r0, int64_t nr, bool reduce) {
    const bool panel = nr >= 0;
    const int64_t rows_v = panel ? nr : m;
    const int w = X.w;
    // column chunks of <= 256: a chunk of up to 256 columns keeps two 128-row M tiles per CTA
    // (TMEM 2 x 256 columns); one 512-wide launch has one M tile and twice the X traffic per A
    // byte (C5 Krylov v = 4, w = 500 co-range view: 58.7 ms as one launch, 2 x 21.4 as two)
    const int nchunk = (w + 255) / 256;
    const int cw = ((w + nchunk - 1) / nchunk + 7) / 8 * 8;
    for (int c0 = 0; c0 < w; c0 += cw) {
      const int wc = std::min(cw, w - c0);
      const size_t mk = mark();
      ViewArgs32 a;
      a.kind = (from == SIDE_N) ? VIEW_AX : VIEW_ATY;
      a.A = A32 + (panel ? r0 * lda : 0);
      a.rows = rows_v;
      a.n = n;
      a.lda = lda;
      float* xh = alloc_f(X.ld * wc);
      float* xl = alloc_f(X.ld * wc);
      a.Xhi = xh;
      a.Xlo = xl;
      a.ldx = X.ld;
      a.w = wc;
      a.grid_cap = ctx->sms;
      plan_view_tf32(a.kind, rows_v, n, wc, ctx->sms, &a.S, &a.KTS);
      double* dst = Y.p + (int64_t)c0 * Y.ld;
      const int ns = tf32_slots(a.S, a.KTS);                 // fp32 chunk partials, summed in fp64
      float* slots = alloc_f((int64_t)ns * Y.ld * wc);
      a.out = slots;
      a.ldo = Y.ld;
      a.slot_stride = (int64_t)Y.ld * wc;
      view_bytes += (double)rows_v * n * 4.0;
      view_flops += 2.0 * rows_v * n * wc;
      ++view_launches;
      if (live()) {
        chk(launch_split_tf32(X.p + (int64_t)c0 * X.ld, X.ld, X.rows, wc, xh, xl, X.ld, st));
        int e0 = -1, e1 = -1;
        ev_record(&e0);
        chk(launch_view_tf32(a, st));
        ev_record(&e1);
        if (e0 >= 0) ev_pairs.push_back({e0, e1});
        chk(launch_slot_sum_f32(slots, Y.ld, a.slot_stride, ns, Y.rows, wc, dst, Y.ld, st));
      }
      release(mk);
    }
    if (from == SIDE_M && collective() && !panel && reduce) allreduce(Y.p, Y.ld * Y.w);
  }

  // G (a x b, col-major ld a) = Xa^T Xb over the side's rows (+ all-reduce when sharded)
  void cross(Side s, const TS& Xa, const TS& Xb, double* G) {
    const size_t mk = mark();
    if (big_skinny(Xa.rows, Xa.w, Xb.w) && Xa.w >= 8) {
      gram_dmma(Xa, Xb, G);
    } else {
      const int ns = gram_slots(Xa.rows);
      double* slots = alloc((int64_t)ns * Xa.w * Xb.w);
      if (live()) {
        chk(launch_cross_gram(Xa.p, Xa.ld, Xa.w, Xb.p, Xb.ld, Xb.w, Xa.rows, slots, ns, st));
        chk(launch_slots_reduce_small(slots, ns, (int64_t)Xa.w * Xb.w, G, st));
      }
    }
    release(mk);
    if (sharded(s)) allreduce(G, (int64_t)Xa.w * Xb.w);
  }

  // ---- tall-skinny products on the FP64 tensor cores, as views of a transposed operand.
  // A column-major rows x w block Q is, byte for byte, a row-major w x rows matrix Q^T, so
  //   Q^T X  = view A X   with A = Q^T   (k_view_ax; reduction over the long dimension)
  //   Q M    = view A^T M with A = Q^T   (k_view_aty; reduction over w)
  // Used where the product is large enough for the view kernels' fixed costs (C3-C5 blocks).
  static bool big_skinny(int64_t rows, int w, int c) { return (double)rows * w * c >= 5.0e7 && rows >= 8192; }

  // one view launch (fp64) on the row-major matrix Ar (ar x nr, lda), X column-major (kdim x w, ldx);
  // result column-major (out_rows x w) into dst (ldd), split-K partial slots summed in order
  // tri: only the upper triangle of the result is needed (a Gram for the cluster Cholesky, VIEW_AX:
  // rows < c0 + wc of column chunk c0) or X is upper triangular (R^-1 applies, VIEW_ATY: the
  // reduction stops at row c0 + wc of X): the chunk's A rows are cut to c0 + wc
  void view_raw(int kind, const double* Ar, int64_t ar, int64_t nr, int64_t lda_r, const double* X, int64_t ldx,
                int w, double* dst, int64_t ldd, bool tri = false) {
    for (int c0 = 0; c0 < w; c0 += kMaxWT * 8) {
      const int wc = std::min(kMaxWT * 8, w - c0);
      const size_t mk = mark();
      const int64_t ar_c = tri ? std::min<int64_t>(ar, c0 + wc) : ar;
      ViewArgs a;
      a.A = Ar;
      a.rows = ar_c;
      a.n = nr;
      a.lda = lda_r;
      a.X = X + (int64_t)c0 * ldx;
      a.ldx = ldx;
      a.w = wc;
      a.grid_cap = ctx->sms;
      plan_view(kind, ar_c, nr, wc, ctx->sms, &a.S, &a.KTS);
      const int64_t orows = (kind == VIEW_AX) ? ar_c : nr;
      double* d = dst + (int64_t)c0 * ldd;
      double* slots = (a.S == 1) ? d : alloc((int64_t)a.S * ldd * wc);
      a.out = slots;
      a.ldo = ldd;
      a.slot_stride = ldd * wc;
      if (live()) {
        chk(kind == VIEW_AX ? launch_view_ax(a, st) : launch_view_aty(a, st));
        if (a.S > 1) chk(launch_slot_sum(slots, ldd, a.slot_stride, a.S, orows, wc, d, ldd, st));
      }
      release(mk);
    }
  }

  // G (a x b, col-major ld a) = Xa^T Xb over the rows (no all-reduce here); upper: only the upper
  // triangle of a square Gram is formed (the rest of G is undefined)
  void gram_dmma(const TS& Xa, const TS& Xb, double* G, bool upper = false) {
    view_raw(VIEW_AX, Xa.p, Xa.w, Xa.rows, Xa.ld, Xb.p, Xb.ld, Xb.w, G, Xa.w, upper);
  }
  // Gram G = Y^T Y for a Cholesky: the upper triangle only when the Cholesky that consumes it
  // reads nothing else (k_chol_cl), on the DMMA views (w >= 65 and a large block)
  void gram_chol(Side s, const TS& Y, double* G) {
    if (chol_reads_upper_only(Y.w) && big_skinny(Y.rows, Y.w, Y.w) && Y.w >= 8) {
      const size_t mk = mark();
      gram_dmma(Y, Y, G, true);
      release(mk);
      if (sharded(s)) allreduce(G, (int64_t)Y.w * Y.w);
      return;
    }
    cross(s, Y, Y, G);
  }

  // out (rows x c, ldo) = in (rows x w, ldi) M (w x c, ldm); mode 1: out -= in M
  void tsmm(const double* in, int64_t ldi, int64_t rows, int w, const double* M, int64_t ldm, int c, double* out,
            int64_t ldo, int mode, bool m_upper = false) {
    if (!big_skinny(rows, w, c) || w < 8 || ((ldm * 8) & 15) || (reinterpret_cast<uintptr_t>(M) & 15)) {
      if (live()) chk(launch_ts_gemm(in, ldi, rows, w, M, ldm, c, out, ldo, mode, st));
      return;
    }
    if (mode == 0) {
      view_raw(VIEW_ATY, in, w, rows, ldi, M, ldm, c, out, ldo, m_upper && c == w);
      return;
    }
    const size_t mk = mark();
    const int64_t ldt = round_up(rows, 32);
    double* T = alloc(ldt * c);
    view_raw(VIEW_ATY, in, w, rows, ldi, M, ldm, c, T, ldt);
    if (live()) chk(launch_sub_cols(T, ldt, out, ldo, rows, c, st));
    release(mk);
  }

  // CholeskyQR2 in place: Y <- Q, R_out (w x w) = R2 R1 if requested.  `ref` (w) optional
  // reference squared column norms for the first pass's rank guard.
  // With `shifted`, a first shifted-Cholesky pass (G + sI, s = 11 (rows w + w(w+1)) u ||Y||_F^2)
  // makes any Y with kappa(Y) < 1/u well enough conditioned for the two CholeskyQR passes
  // (shifted CholeskyQR3, Fukaya et al. 2020); used for the projected Krylov blocks.
  void orth(Side s, const TS& Y, double* R_out, const double* ref, bool shifted = false) {
    const int w = Y.w;
    if (w <= 64 && !sharded(s) && ref == nullptr) {
      orth_fused(s, Y, R_out, shifted);
      return;
    }
    const size_t mk = mark();
    double* G = alloc((int64_t)w * w);
    double* R1 = alloc((int64_t)w * w);
    double* R1i = alloc((int64_t)w * w);
    double* R2 = alloc((int64_t)w * w);
    double* R2i = alloc((int64_t)w * w);
    TS T = new_ts(s, w);
    double* R0s = nullptr;
    if (shifted) {
      double* R0 = alloc((int64_t)w * w);
      R0s = R0;
      double* R0i = alloc((int64_t)w * w);
      // the shift must be identical on every rank: the GLOBAL row count of a sharded side
      const double rows_all = (double)(sharded(s) ? side_rows_glob(s) : Y.rows);
      const double coef = 11.0 * (rows_all * w + (double)w * (w + 1)) * 1.1102230246251565e-16;
      gram_chol(s, Y, G);
      if (live()) chk(launch_chol_ref(G, nullptr, w, 0.0, R0, R0i, nullptr, st, coef));
      tsmm(Y.p, Y.ld, Y.rows, w, R0i, w, w, T.p, T.ld, 0, true);
      if (live()) chk(launch_copy_cols(T.p, T.ld, Y.p, Y.ld, Y.rows, w, st));
    }
    gram_chol(s, Y, G);
    if (live()) chk(launch_chol_ref(G, ref, w, 1e-12, R1, R1i, ctx->dstat, st));
    tsmm(Y.p, Y.ld, Y.rows, w, R1i, w, w, T.p, T.ld, 0, true);
    gram_chol(s, T, G);
    if (live()) chk(launch_chol_ref(G, nullptr, w, 1e-12, R2, R2i, nullptr, st));
    tsmm(T.p, T.ld, T.rows, w, R2i, w, w, Y.p, Y.ld, 0, true);
    if (live() && R_out) {
      if (shifted) {  // R = R2 R1 R0 (R1i is free now)
        chk(launch_small_gemm(0, 0, w, w, w, R1, w, R0s, w, R1i, w, st));
        chk(launch_small_gemm(0, 0, w, w, w, R2, w, R1i, w, R_out, w, st));
      } else {
        chk(launch_small_gemm(0, 0, w, w, w, R2, w, R1, w, R_out, w, st));
      }
    }
    release(mk);
  }

  // CholeskyQR2 (or shifted CholeskyQR3) for w <= 64 on an unsharded side: every pass is one
  // launch of k_cholqr_pass (apply previous R^-1, Gram, last-CTA Cholesky + inverse).
  void orth_fused(Side s, const TS& Y, double* R_out, bool shifted) {
    (void)s;
    const int w = Y.w;
    const size_t mk = mark();
    if (orth_cluster_fits(Y.rows, w) && !getenv_flag("RSVD_NO_ORTH_CLUSTER")) {
      // the whole CholeskyQR2 / shifted CholeskyQR3 in one cluster launch (Y resident in smem)
      double* Rw = alloc(3 * (int64_t)w * w);
      const double coef = 11.0 * ((double)Y.rows * w + (double)w * (w + 1)) * 1.1102230246251565e-16;
      if (live()) chk(launch_orth_cluster(Y.p, Y.ld, Y.rows, w, shifted ? 1 : 0, coef, R_out, Rw, ctx->dstat, st));
      release(mk);
      return;
    }
    const int G = cholqr_pass_ctas(Y.rows);
    double* slots = alloc((int64_t)G * w * w);
    double* R0 = alloc((int64_t)w * w);
    double* R0i = alloc((int64_t)w * w);
    double* R1 = alloc((int64_t)w * w);
    double* R1i = alloc((int64_t)w * w);
    double* R2 = alloc((int64_t)w * w);
    double* R2i = alloc((int64_t)w * w);
    TS T = new_ts(s, w);
    if (live()) {
      const double coef = 11.0 * ((double)Y.rows * w + (double)w * (w + 1)) * 1.1102230246251565e-16;
      if (!shifted) {
        chk(launch_cholqr_pass(Y.p, Y.ld, nullptr, 0, Y.rows, w, nullptr, slots, ctx->counter, 1e-12, 0.0, 0, R1,
                               R1i, ctx->dstat, st));
        chk(launch_cholqr_pass(Y.p, Y.ld, T.p, T.ld, Y.rows, w, R1i, slots, ctx->counter, 1e-12, 0.0, 1, R2, R2i,
                               nullptr, st));
        chk(launch_ts_gemm(T.p, T.ld, T.rows, w, R2i, w, w, Y.p, Y.ld, 0, st));   // w <= 64: FMA kernel
        if (R_out) chk(launch_small_gemm(0, 0, w, w, w, R2, w, R1, w, R_out, w, st));
      } else {
        chk(launch_cholqr_pass(Y.p, Y.ld, nullptr, 0, Y.rows, w, nullptr, slots, ctx->counter, 0.0, coef, 0, R0,
                               R0i, nullptr, st));
        chk(launch_cholqr_pass(Y.p, Y.ld, T.p, T.ld, Y.rows, w, R0i, slots, ctx->counter, 1e-12, 0.0, 0, R1, R1i,
                               ctx->dstat, st));
        chk(launch_cholqr_pass(T.p, T.ld, Y.p, Y.ld, Y.rows, w, R1i, slots, ctx->counter, 1e-12, 0.0, 1, R2, R2i,
                               nullptr, st));
        chk(launch_ts_gemm(Y.p, Y.ld, Y.rows, w, R2i, w, w, T.p, T.ld, 0, st));
        chk(launch_copy_cols(T.p, T.ld, Y.p, Y.ld, Y.rows, w, st));
        if (R_out) {  // R = R2 R1 R0
          chk(launch_small_gemm(0, 0, w, w, w, R1, w, R0, w, R1i, w, st));
          chk(launch_small_gemm(0, 0, w, w, w, R2, w, R1i, w, R_out, w, st));
        }
      }
    }
    release(mk);
  }

  // block classical Gram-Schmidt, twice, over blocks of width bw, then CholeskyQR2 per block.
  // first_orthonormal: block 0 is already an orth's Q (an intermediate Krylov block, v >= 4).
  // Rank guard of the projected blocks (reading R11): a column whose projected remainder is at
  // the rounding level of the projection, |w_j - Q Q^T w_j|^2 <= (64 u)^2 |w_j|^2 with the norm
  // taken BEFORE projecting, lies in the span of the previous blocks and is zeroed; the guarded
  // Cholesky passes keep exact zero columns at zero.  (A self-referenced guard, judged on the
  // remainder alone, would renormalise that rounding noise into a spurious direction.)
  void bcgs2(Side s, const TS& K, int bw, bool first_orthonormal) {
    const int nb = (K.w + bw - 1) / bw;
    for (int b = 0; b < nb; ++b) {
      const int c0 = b * bw, wc = std::min(bw, K.w - c0);
      TS Wb = slice(K, c0, wc);
      const size_t mk = mark();
      if (b > 0) {
        // BCGS2 (Barlow & Smoktunowicz): project, normalise (shifted CholeskyQR: the projected
        // remainder of a raw Krylov block can be tiny and nearly rank deficient), project again
        // (removes the components the normalisation amplified), then CholeskyQR2.
        TS Qp = slice(K, 0, c0);
        double* C = alloc((int64_t)c0 * wc);
        double* ref = alloc(wc);
        double* nrm = alloc(wc);
        colnorm2(s, Wb, ref);                               // |w_j|^2 before the projection
        cross(s, Qp, Wb, C);
        tsmm(Qp.p, Qp.ld, Qp.rows, c0, C, c0, wc, Wb.p, Wb.ld, 1);
        colnorm2(s, Wb, nrm);                               // ... and after it
        constexpr double kDepTol = (64.0 * 1.1102230246251565e-16) * (64.0 * 1.1102230246251565e-16);
        if (live()) chk(launch_zero_dep_cols(Wb.p, Wb.ld, Wb.rows, wc, nrm, ref, kDepTol, ctx->dstat, st, 1));
        orth(s, Wb, nullptr, nullptr, /*shifted=*/true);
        cross(s, Qp, Wb, C);
        tsmm(Qp.p, Qp.ld, Qp.rows, c0, C, c0, wc, Wb.p, Wb.ld, 1);
        orth(s, Wb, nullptr, nullptr);
      } else if (!first_orthonormal) {
        orth(s, Wb, nullptr, nullptr);
      }
      release(mk);
    }
  }

  // d[j] = |X_j|^2 over the side's rows (+ all-reduce when sharded): the diagonal of X^T X alone
  void colnorm2(Side s, const TS& X, double* d) {
    if (live()) chk(launch_colnorm2(X.p, X.ld, X.rows, X.w, d, st));
    if (sharded(s)) allreduce(d, X.w);
  }

  // out (rows x k, ldo) = Q (rows x w) * Mk (w x k, ld w)
  void lift(const TS& Q, const double* Mk, int k, double* out, int64_t ldo) {
    tsmm(Q.p, Q.ld, Q.rows, Q.w, Mk, Q.w, k, out, ldo, 0);
  }

  // want_j: 0 = right vectors as B^T U S^-1 (the leading triplets the algorithms keep); 2 = accumulate
  // J in the 64 < w <= 128 kernel (cores whose trailing vectors are used or must stay orthonormal)
  void core_svd(const double* M, int w, int trans, double* Ul, double* Sv, double* Vr, int want_j = 0) {
    const size_t mk = mark();
    double* scratch = alloc(2 * 512 * 512 + 4096);
    if (live()) chk(launch_jacobi_t(M, w, trans, w, w, Ul, Sv, Vr, scratch, ctx->dstat, st, want_j));
    release(mk);
  }

  // ------------------------------------------------------------ staging of caller arrays
  // device TS copy of a caller array (rows x w, column-major, ld_user)
  // (host or device) caller arrays are copied in by cudaMemcpy2DAsync before the graph launch,
  // and outputs are copied out after it, so the captured graph never references caller memory
  // other than A: one graph serves every call with the same A, shapes and flags.
  TS stage_in(Side s, const void* src, int64_t ld_user, int w, PtrKind kind) {
    (void)kind;
    TS t = new_ts(s, w);
    if (s == SIDE_N && shard_n && src)   // this rank's chunk of the caller's n-long array
      src = static_cast<const char*>(src) + n0 * (dtype == RSVD_F32 ? 4 : 8);
    if (dtype == RSVD_F32) {
      float* f = alloc_f(t.ld * w);
      h2d.push_back({f, t.ld, src, ld_user, t.rows, w, 4});
      if (live()) chk(launch_f32_to_f64(f, t.ld, t.p, t.ld, t.rows, w, st));
    } else {
      h2d.push_back({t.p, t.ld, src, ld_user, t.rows, w});
    }
    return t;
  }
  // stage a caller array (rows of dst x w) into columns [col0, col0 + w) of an existing block
  void stage_into(const TS& dst, int col0, const void* src, int64_t ld_user, int w) {
    double* d = dst.p + (int64_t)col0 * dst.ld;
    if (dtype == RSVD_F32) {
      float* f = alloc_f(dst.ld * w);
      h2d.push_back({f, dst.ld, src, ld_user, dst.rows, w, 4});
      if (live()) chk(launch_f32_to_f64(f, dst.ld, d, dst.ld, dst.rows, w, st));
    } else {
      h2d.push_back({d, dst.ld, src, ld_user, dst.rows, w});
    }
  }
  // where to write a caller output of rows x cols (col-major, ld): direct if device, else staging
  double* out_ptr(void* user, int64_t ld_user, int64_t rows, int cols, PtrKind kind, int64_t* ld_out) {
    const int64_t ld = round_up(std::max<int64_t>(rows, 1), 32);
    double* p = alloc(ld * cols);
    *ld_out = ld;
    if (kind != PTR_NULL && user) {
      if (dtype == RSVD_F32) {
        float* f = alloc_f(ld * cols);
        narrow.push_back({p, ld, f, ld, rows, cols});
        d2h.push_back({user, ld_user, f, ld, rows, cols, 4});
      } else {
        d2h.push_back({user, ld_user, p, ld, rows, cols});
      }
    }
    return p;
  }
};

// ================================================================ algorithms
// Each takes the resolved Exec; sides: the algorithm's input B = A (input 0) or A^T (input 1).
// range side of B  (rows of B): side_c;  co-range side (cols of B): side_r.

void write_outputs(Exec& E, Side side_c, Side side_r, const TS& Qc, const TS& Qr, const double* Uh,
                   const double* Vh, const double* lam, int w, int k) {
  const Call& c = E.call;
  // B's U = Qc Uh (side_c), B's V = Qr Vh (side_r); A's U lives on side M, A's V on side N
  auto emit = [&](Side s, const TS& Q, const double* M) {
    if (s == SIDE_M) {
      if (c.kU == PTR_NULL) return;
      int64_t ld;
      double* o = E.out_ptr(c.U, c.ldu, Q.rows, k, c.kU, &ld);
      E.lift(Q, M, k, o, ld);
    } else {
      if (c.kV == PTR_NULL) return;
      int64_t ld;
      double* o = E.out_ptr(c.V, c.ldv, E.n, k, c.kV, &ld);
      if (E.shard_n) {   // lift this rank's chunk, all-gather the full V
        const size_t mk = E.mark();
        TS L = E.new_ts(SIDE_N, k);
        E.lift(Q, M, k, L.p, L.ld);
        E.gather_n_into(L, o, ld);
        E.release(mk);
      } else {
        E.lift(Q, M, k, o, ld);
      }
    }
  };
  emit(side_c, Qc, Uh);
  emit(side_r, Qr, Vh);
  if (c.kS != PTR_NULL) {
    int64_t ld;
    double* so = E.out_ptr(c.S, k, k, 1, c.kS, &ld);
    if (E.live()) {
      E.chk(launch_copy_cols(lam, w, so, k, k, 1, E.st));
      if (c.flags & RSVD_SQUARED) E.chk(launch_square(so, k, E.st));
    }
  }
}

void alg_subspace(Exec& E) {
  const Call& c = E.call;
  const int l = c.k + c.p;
  const Side side_c = c.input == RSVD_INPUT_A ? SIDE_M : SIDE_N;
  const Side side_r = c.input == RSVD_INPUT_A ? SIDE_N : SIDE_M;
  TS Qr = E.stage_in(side_r, c.Om, c.ldom, l, c.kOm);   // line 1: Q_r = Omega
  TS Qc = E.new_ts(side_c, l);
  double* Rlast = E.alloc((int64_t)l * l);
  for (int j = 1; j <= c.v; ++j) {                       // lines 2-8
    if (j % 2 == 1) {
      E.view(side_r, Qr, Qc);                            // A Q_r
      E.orth(side_c, Qc, j == c.v ? Rlast : nullptr, nullptr);
    } else {
      E.view(side_c, Qc, Qr);                            // A^* Q_c
      E.orth(side_r, Qr, j == c.v ? Rlast : nullptr, nullptr);
    }
  }
  double* Ul = E.alloc((int64_t)l * l);
  double* Vr = E.alloc((int64_t)l * l);
  double* lam = E.alloc(l);
  E.core_svd(Rlast, l, 1, Vr, lam, Ul, (c.flags & RSVD_SQUARED) ? 2 : 0);  // Jacobi on R^T: left(R^T) = right(R)
  // v even: R_r = Vh Lam Uh^T -> left = Vh, right = Uh;  v odd: R_c = Uh Lam Vh^T
  if (c.v % 2 == 0)
    write_outputs(E, side_c, side_r, Qc, Qr, /*Uh=*/Vr, /*Vh=*/Ul, lam, l, c.k);
  else
    write_outputs(E, side_c, side_r, Qc, Qr, /*Uh=*/Ul, /*Vh=*/Vr, lam, l, c.k);
}

void alg_krylov(Exec& E) {
  const Call& c = E.call;
  const int l = c.k + c.p, v = c.v;
  const Side side_c = c.input == RSVD_INPUT_A ? SIDE_M : SIDE_N;
  const Side side_r = c.input == RSVD_INPUT_A ? SIDE_N : SIDE_M;
  const bool even = (v % 2 == 0);
  const int nb = even ? v / 2 : (v - 1) / 2;
  const int W = nb * l;
  const Side side_K = even ? side_c : side_r;
  TS K = E.new_ts(side_K, W);
  TS Q0 = E.stage_in(side_r, c.Om, c.ldom, l, c.kOm);   // line 1: Q_r^0 = Omega
  TS tmp_c = E.new_ts(side_c, l), tmp_r = E.new_ts(side_r, l);
  TS prev = Q0;
  for (int j = 1; j <= v - 1; ++j) {                    // lines 2-7
    const bool odd = (j % 2 == 1);
    const bool in_K = even ? odd : !odd;                 // K_c = odd blocks (v even), K_r = even blocks
    TS dst;
    if (in_K) {
      const int b = even ? (j - 1) / 2 : (j / 2 - 1);
      dst = E.slice(K, b * l, l);
    } else {
      dst = odd ? tmp_c : tmp_r;
    }
    E.view(odd ? side_r : side_c, prev, dst);
    if (j < v - 1) E.orth(odd ? side_c : side_r, dst, nullptr, nullptr);  // last block stays raw
    prev = dst;
  }
  if (v == 1) return;
  E.bcgs2(side_K, K, l, /*first_orthonormal=*/nb > 1);   // qr(K_c) / qr(K_r)  (lines 9 / 14)
  TS Qo = E.new_ts(even ? side_r : side_c, W);
  double* Rw = E.alloc((int64_t)W * W);
  E.view(side_K, K, Qo);                                  // one more view (lines 10 / 15)
  E.orth(even ? side_r : side_c, Qo, Rw, nullptr);
  double* Ul = E.alloc((int64_t)W * W);
  double* Vr = E.alloc((int64_t)W * W);
  double* lam = E.alloc(W);
  E.core_svd(Rw, W, 1, Vr, lam, Ul, (c.flags & RSVD_SQUARED) ? 2 : 0);
  if (even)  // Q_c = K, Q_r = Qo, R_r = Vh Lam Uh^T
    write_outputs(E, side_c, side_r, K, Qo, Vr, Ul, lam, W, c.k);
  else       // Q_r = K, Q_c = Qo, R_c = Uh Lam Vh^T
    write_outputs(E, side_c, side_r, Qo, K, Ul, Vr, lam, W, c.k);
}

constexpr double kYcSlotBudget = 4.0e9;  // bytes of deterministic Y_c partial slots

// One view of A for the 1-view methods (Alg. 7 line 3; the extended sketch):
// Yc = A Om and Yr = A^* Phi from one read of every A tile (k_view_fused), or two view launches
// when the widths exceed the fused kernel's register budget or A is fp32 (info.view_launches = 2).
constexpr double kYcClusterSlotBudget = 24.0e9;  // bytes of the cluster kernel's Y_c group slots

// Wide sketches (C4: l = 120, l2 = 240): k_view_fused_cl, one read of A with the Y_c partials
// reduced across a thread-block cluster (view_fused_cluster.cu).  Returns false when not applicable.
bool sketch_view_cluster(Exec& E, const TS& Om, const TS& Phi, const TS& Yc, const TS& Yr, bool wanted) {
  const int l = Om.w, l2 = Phi.w;
  // with RSVD_ONE_READ the cluster kernel also takes the narrow widths: its Y_c partial traffic is
  // l / (64 CL) of A's bytes against l / 64 for the one-CTA kernel (C3, l = 70: 3.2x A's bytes of
  // DRAM traffic in all with the one-CTA kernel)
  if (!wanted || E.dtype != RSVD_F64 || !fused_cl_supported(l, l2)) return false;
  FusedClArgs a;
  plan_fused_cl(E.m, E.n, l, l2, E.ctx->sms, &a);
  a.ldys = round_up(l, 8);
  a.yc_slot_stride = round_up(std::max<int64_t>(E.m, 1), 32) * a.ldys;
  if ((double)a.NG * a.yc_slot_stride * 8.0 > kYcClusterSlotBudget) return false;
  const size_t mk = E.mark();
  a.A = E.A;
  a.rows = E.m;
  a.n = E.n;
  a.lda = E.lda;
  a.Om = Om.p;
  a.ldom = Om.ld;
  a.l = l;
  a.Phi = Phi.p;
  a.ldphi = Phi.ld;
  a.l2 = l2;
  a.yc_slots = E.alloc((int64_t)a.NG * a.yc_slot_stride);
  double* yrs = (a.S == 1) ? Yr.p : E.alloc((int64_t)a.S * Yr.ld * l2);
  a.yr = yrs;
  a.ldyr = Yr.ld;
  a.yr_slot_stride = (int64_t)Yr.ld * l2;
  E.view_bytes += (double)E.m * E.n * 8.0;
  E.view_flops += 2.0 * E.m * E.n * (l + l2);
  ++E.view_launches;
  if (E.live()) {
    int e0 = -1, e1 = -1;
    E.ev_record(&e0);
    E.chk(launch_view_fused_cl(a, E.st));
    E.ev_record(&e1);
    if (e0 >= 0) E.ev_pairs.push_back({e0, e1});
    E.chk(launch_slot_sum_rows(a.yc_slots, a.ldys, a.yc_slot_stride, a.NG, Yc.rows, l, Yc.p, Yc.ld, E.st));
    if (a.S > 1) E.chk(launch_slot_sum(yrs, Yr.ld, a.yr_slot_stride, a.S, Yr.rows, l2, Yr.p, Yr.ld, E.st));
  }
  if (E.collective()) E.allreduce(Yr.p, Yr.ld * l2);
  E.release(mk);
  return true;
}

// Sketch widths beyond the one-CTA fused kernel (C4: l = 120, l2 = 240) take two view launches by
// default: on device-resident A both products are DMMA-bound, and the one-read cluster kernel runs
// at 0.62 of the per-SM DMMA rate on the 112 SMs that seven 16-CTA clusters occupy (C4: 416 ms
// against 204 ms for the two views).  flags & RSVD_ONE_READ selects the one-read path (A is read
// from memory once: the paper's single-pass premise, for when reading A is the cost).
void sketch_view(Exec& E, const TS& Om, const TS& Phi, const TS& Yc, const TS& Yr) {
  const int l = Om.w, l2 = Phi.w;
  if (sketch_view_cluster(E, Om, Phi, Yc, Yr, (E.call.flags & RSVD_ONE_READ) != 0)) return;
  const bool fused_ok = (E.dtype == RSVD_F64) && (l <= kFusedMaxL) && ((l2 + 7) / 8 <= kFusedMaxL2T);
  if (fused_ok) {
    const size_t mk = E.mark();
    FusedArgs a;
    a.A = E.A;
    a.rows = E.m;
    a.n = E.n;
    a.lda = E.lda;
    a.Om = Om.p;
    a.ldom = Om.ld;
    a.l = l;
    a.Phi = Phi.p;
    a.ldphi = Phi.ld;
    a.l2 = l2;
    a.grid_cap = E.ctx->sms;
    plan_view(VIEW_FUSED, E.m, E.n, l2, E.ctx->sms, &a.S, &a.KTS);
    const int nsb = fused_strips(E.n);
    const double slot_bytes = (double)nsb * Yc.ld * l * 8.0;
    a.yc_atomic = slot_bytes > kYcSlotBudget ? 1 : 0;
    E.nondet |= a.yc_atomic;
    double* ycs = a.yc_atomic ? Yc.p : E.alloc((int64_t)nsb * Yc.ld * l);
    a.yc = ycs;
    a.ldyc = Yc.ld;
    a.yc_slot_stride = (int64_t)Yc.ld * l;
    double* yrs = (a.S == 1) ? Yr.p : E.alloc((int64_t)a.S * Yr.ld * l2);
    a.yr = yrs;
    a.ldyr = Yr.ld;
    a.yr_slot_stride = (int64_t)Yr.ld * l2;
    E.view_bytes += (double)E.m * E.n * 8.0;
    E.view_flops += 2.0 * E.m * E.n * (l + l2);
    ++E.view_launches;
    if (E.live()) {
      if (a.yc_atomic) E.chk(launch_fill(Yc.p, Yc.ld * l, 0.0, E.st));
      int e0 = -1, e1 = -1;
      E.ev_record(&e0);
      E.chk(launch_view_fused(a, E.st));
      E.ev_record(&e1);
      if (e0 >= 0) E.ev_pairs.push_back({e0, e1});
      if (!a.yc_atomic) E.chk(launch_slot_sum(ycs, Yc.ld, a.yc_slot_stride, nsb, Yc.rows, l, Yc.p, Yc.ld, E.st));
      if (a.S > 1) E.chk(launch_slot_sum(yrs, Yr.ld, a.yr_slot_stride, a.S, Yr.rows, l2, Yr.p, Yr.ld, E.st));
    }
    if (E.collective()) E.allreduce(Yr.p, Yr.ld * l2);
    E.release(mk);
  } else {
    // widths beyond the fused kernel's register budget: two views (documented; info->view_launches = 2)
    E.view(SIDE_N, Om, Yc);
    E.view(SIDE_M, Phi, Yr);
  }
}

void alg_single_pass(Exec& E) {
  const Call& c = E.call;
  const int l = c.k + c.p, l2 = c.l2;
  const bool minvar = (c.lc == RSVD_LC_MINVAR);
  const bool woolfe = (c.flags & RSVD_WOOLFE) != 0;
  const int lc = minvar ? c.p : c.lc;
  const int lp = c.k + lc;  // width of Q_c after the optional truncation; MinVar: l, masked
  TS Om = E.stage_in(SIDE_N, c.Om, c.ldom, l, c.kOm);
  TS Phi = E.stage_in(SIDE_M, c.Phi, c.ldphi, l2, c.kPhi);
  TS Yc = E.new_ts(SIDE_M, l);
  TS Yr = E.new_ts(SIDE_N, l2);
  // ---- line 3: a) Y_c = A Omega  and  b) Y_r = A^* Phi  from one read of A
  sketch_view(E, Om, Phi, Yc, Yr);
  // ---- lines 4-10: Q_c (optionally truncated to the top k+l_c left singular vectors of R_c)
  double* Rc = E.alloc((int64_t)l * l);
  E.orth(SIDE_M, Yc, Rc, nullptr);
  TS Qc = Yc;
  if (lc < c.p || minvar || woolfe) {
    double* Ul = E.alloc((int64_t)l * l);
    double* Vr = E.alloc((int64_t)l * l);
    double* sv = E.alloc(l);
    E.core_svd(Rc, l, 1, Vr, sv, Ul, 2);   // truncation / MinVar use trailing left vectors of R_c
    TS Q2 = E.new_ts(SIDE_M, lp);
    E.tsmm(Yc.p, Yc.ld, Yc.rows, l, Ul, l, lp, Q2.p, Q2.ld, 0);
    Qc = Q2;
  }
  // ---- line 11: C = Phi^* Q_c   (l2 x lp, tiny; replicated)
  TS C;
  C.rows = l2;
  C.ld = round_up(l2, 32);
  C.w = lp;
  C.p = E.alloc(C.ld * lp);
  {
    double* Cg = E.alloc((int64_t)l2 * lp);
    E.cross(SIDE_M, Phi, Qc, Cg);
    if (E.live()) E.chk(launch_copy_cols(Cg, l2, C.p, C.ld, l2, lp, E.st));
  }
  // [Qh, Rh] = qr(X) for an l2 x lp block X (ld ldx) by CholeskyQR2: Qh overwrites X, Rh^-1 =
  // R1^-1 R2^-1 into Rhi (lp x lp).  The guarded Cholesky zeroes exactly-zero columns.
  double* G = E.alloc((int64_t)lp * lp);
  double* R1 = E.alloc((int64_t)lp * lp);
  double* R1i = E.alloc((int64_t)lp * lp);
  double* R2 = E.alloc((int64_t)lp * lp);
  double* R2i = E.alloc((int64_t)lp * lp);
  double* Cq = E.alloc((int64_t)l2 * lp);
  double* Rw = E.alloc(3 * (int64_t)lp * lp);
  static const bool qr_small_chain = getenv_flag("RSVD_QR_SMALL_CHAIN");
  auto qr_small = [&](double* X, int64_t ldx, double* Rhi_out) {
    if (!E.live()) return;
    if (!qr_small_chain && orth_cluster_fits(l2, lp)) {
      // the same CholeskyQR2 (guarded passes, closed-form second pass) in one cluster launch,
      // Qh over X and Rh = R2 R1; Rh^-1 by back substitution (zero pivots -> zero rows/columns)
      E.chk(launch_orth_cluster(X, ldx, l2, lp, 0, 0.0, R1, Rw, E.ctx->dstat, E.st));
      E.chk(launch_tri_inv(R1, lp, Rhi_out, nullptr, E.st));
      return;
    }
    E.chk(launch_small_gemm(1, 0, lp, lp, l2, X, ldx, X, ldx, G, lp, E.st));
    E.chk(launch_chol_ref(G, nullptr, lp, 1e-12, R1, R1i, E.ctx->dstat, E.st));
    E.chk(launch_small_gemm(0, 0, l2, lp, lp, X, ldx, R1i, lp, Cq, l2, E.st));
    E.chk(launch_small_gemm(1, 0, lp, lp, l2, Cq, l2, Cq, l2, G, lp, E.st));
    E.chk(launch_chol_ref(G, nullptr, lp, 1e-12, R2, R2i, nullptr, E.st));
    E.chk(launch_small_gemm(0, 0, l2, lp, lp, Cq, l2, R2i, lp, X, ldx, E.st));        // Qh
    E.chk(launch_small_gemm(0, 0, lp, lp, lp, R1i, lp, R2i, lp, Rhi_out, lp, E.st));  // Rh^-1
  };
  double* Rhi = E.alloc((int64_t)lp * lp);
  if (woolfe) {
    // ---- Alg. 8 lines 4b-6b: Y_r = Q_r R_r, tsvd(R_r, k + l_c), Q_r <- Q_r Qh_r
    double* Rr = E.alloc((int64_t)l2 * l2);
    E.orth(SIDE_N, Yr, Rr, nullptr, /*shifted=*/true);  // Y_r can be far worse conditioned than Y_c
    double* Ur = E.alloc((int64_t)l2 * l2);
    double* Vrr = E.alloc((int64_t)l2 * l2);
    double* svr = E.alloc(l2);
    E.core_svd(Rr, l2, 1, Vrr, svr, Ur, 2);                  // R_r = Ur S Vrr^T
    TS Qr = E.new_ts(SIDE_N, lp);
    E.tsmm(Yr.p, Yr.ld, Yr.rows, l2, Ur, l2, lp, Qr.p, Qr.ld, 0);
    // ---- line 7: (Phi^* Q_c) Xh = Y_r^* Q_r = R_r^T Ur[:, :lp]   (l2 x lp)
    double* RHS = E.alloc((int64_t)l2 * lp);
    double* T1 = E.alloc((int64_t)lp * lp);
    double* Xh = E.alloc((int64_t)lp * lp);
    if (E.live()) E.chk(launch_small_gemm(1, 0, l2, lp, l2, Rr, l2, Ur, l2, RHS, l2, E.st));
    qr_small(C.p, C.ld, Rhi);
    if (E.live()) {
      E.chk(launch_small_gemm(1, 0, lp, lp, l2, C.p, C.ld, RHS, l2, T1, lp, E.st));  // Qh^T RHS
      E.chk(launch_small_gemm(0, 0, lp, lp, lp, Rhi, lp, T1, lp, Xh, lp, E.st));     // Rh^-1 (.)
    }
    // ---- line 8: tsvd(Xh, k) = Uh Lam Vh^T;  line 9: U = Q_c Uh, V = Q_r Vh
    double* Ux = E.alloc((int64_t)lp * lp);
    double* Vx = E.alloc((int64_t)lp * lp);
    double* lam = E.alloc(lp);
    E.core_svd(Xh, lp, 0, Ux, lam, Vx);
    write_outputs(E, SIDE_M, SIDE_N, Qc, Qr, Ux, Vx, lam, lp, c.k);
    return;
  }
  if (minvar && c.p > 0) {
    // ---- minimum-variance l_c: trial spectra from one QR of M = C (all l columns)
    double* Cm = E.alloc((int64_t)l2 * lp);
    double* Rhm = E.alloc((int64_t)lp * lp);
    TS Yq = E.new_ts(SIDE_N, l2);                             // Y_r = Q_y R_y (copy: Y_r is kept)
    double* Ry = E.alloc((int64_t)l2 * l2);
    double* Z = E.alloc((int64_t)l2 * lp);
    double* lamt = E.alloc((int64_t)(c.p + 1) * c.k);
    double* scr = E.alloc(minvar_scratch(l2, lp, c.p));
    if (E.live()) {
      E.chk(launch_copy_cols(C.p, C.ld, Cm, l2, l2, lp, E.st));
      E.chk(launch_copy_cols(Yr.p, Yr.ld, Yq.p, Yq.ld, Yr.rows, l2, E.st));
    }
    qr_small(Cm, l2, Rhm);
    E.orth(SIDE_N, Yq, Ry, nullptr);
    if (E.live()) {
      E.chk(launch_small_gemm(0, 0, l2, lp, l2, Ry, l2, Cm, l2, Z, l2, E.st));       // Z = R_y Qh
      E.chk(launch_minvar_trials(Z, l2, lp, Rhm, c.k, c.p, lamt, scr, E.st));
      int* lc_dev = &E.ctx->dstat->minvar_lc;
      E.chk(launch_minvar_select(lamt, c.k, c.p, lc_dev, E.st));
      E.chk(launch_mask_cols(Qc.p, Qc.ld, Qc.rows, lp, c.k, lc_dev, E.st));
      E.chk(launch_mask_cols(C.p, C.ld, l2, lp, c.k, lc_dev, E.st));
    }
  }
  // ---- line 11: [Qh, Rh] = qr(Phi^* Q_c);  line 12: X = Rh^-1 Qh^* Y_r^*  ->  X^T = Y_r (Qh Rh^-T)
  double* T = E.alloc((int64_t)l2 * lp);
  qr_small(C.p, C.ld, Rhi);
  if (E.live()) E.chk(launch_small_gemm(0, 1, l2, lp, lp, C.p, C.ld, Rhi, lp, T, l2, E.st));
  TS Xt = E.new_ts(SIDE_N, lp);
  E.tsmm(Yr.p, Yr.ld, Yr.rows, l2, T, l2, lp, Xt.p, Xt.ld, 0);
  // ---- line 13: tsvd(X, k) via X^T = Qx Rx  ->  X = Rx^T Qx^T,  svd(Rx^T) = Uh Lam Wh^T
  double* Rx = E.alloc((int64_t)lp * lp);
  E.orth(SIDE_N, Xt, Rx, nullptr);
  double* Ul = E.alloc((int64_t)lp * lp);
  double* Vr = E.alloc((int64_t)lp * lp);
  double* lam = E.alloc(lp);
  E.core_svd(Rx, lp, /*trans=*/0, Vr, lam, Ul);  // svd(Rx^T) from Jacobi on Rx
  // U = Q_c Uh (side M), V = Qx Wh (side N)           (line 14)
  write_outputs(E, SIDE_M, SIDE_N, Qc, Xt, Ul, Vr, lam, lp, c.k);
}

// [Q, R] = qr(X) of a small replicated block (rows x w, col-major ld rows) by CholeskyQR2 with
// the rank guard: Q overwrites X, R = R2 R1 (w x w).
void small_qr(Exec& E, double* X, int rows, int w, double* R) {
  double* G = E.alloc((int64_t)w * w);
  double* R1 = E.alloc((int64_t)w * w);
  double* R1i = E.alloc((int64_t)w * w);
  double* R2 = E.alloc((int64_t)w * w);
  double* R2i = E.alloc((int64_t)w * w);
  double* T = E.alloc((int64_t)rows * w);
  double* Rw = E.alloc(3 * (int64_t)w * w);
  if (!E.live()) return;
  if (!getenv_flag("RSVD_QR_SMALL_CHAIN") && orth_cluster_fits(rows, w)) {
    // the same guarded CholeskyQR2 in one cluster launch (R = R2 R1 written by the kernel)
    E.chk(launch_orth_cluster(X, rows, rows, w, 0, 0.0, R, Rw, nullptr, E.st));
    return;
  }
  E.chk(launch_small_gemm(1, 0, w, w, rows, X, rows, X, rows, G, w, E.st));
  E.chk(launch_chol_ref(G, nullptr, w, 1e-12, R1, R1i, nullptr, E.st));
  E.chk(launch_small_gemm(0, 0, rows, w, w, X, rows, R1i, w, T, rows, E.st));
  E.chk(launch_small_gemm(1, 0, w, w, rows, T, rows, T, rows, G, w, E.st));
  E.chk(launch_chol_ref(G, nullptr, w, 1e-12, R2, R2i, nullptr, E.st));
  E.chk(launch_small_gemm(0, 0, rows, w, w, T, rows, R2i, w, X, rows, E.st));
  E.chk(launch_small_gemm(0, 0, w, w, w, R2, w, R1, w, R, w, E.st));
}

// T^+ (w x w) with singular values below 1e-12 sigma_max dropped (reading R24): one-sided Jacobi
// with J accumulated (every singular pair is used), then V S^+ U^T.
void small_pinv(Exec& E, const double* T, int w, double* Tp) {
  double* Ul = E.alloc((int64_t)w * w);
  double* Vr = E.alloc((int64_t)w * w);
  double* sv = E.alloc(w);
  E.core_svd(T, w, 0, Ul, sv, Vr, 1);
  if (E.live()) E.chk(launch_pinv_svd(Ul, sv, Vr, w, 1e-12, Tp, E.st));
}

// Extended 1-view sketch, bwz (Eq. bwz) or bwz2 (Eq. bwzimproved).  Xi_r / Xi_c are
// the paper's SRFT matrices Phi_r (m x s) and Phi_c (n x s), materialised by the caller (R3, R23).
void alg_extended(Exec& E) {
  const Call& c = E.call;
  const int l = c.k + c.p, l2 = c.l2, s = c.s, k = c.k;
  // one view: [Y_c | A Xi_c] = A [Omega | Xi_c] and Y_r = A^* Phi
  TS OmX = E.new_ts(SIDE_N, l + s);
  E.stage_into(OmX, 0, c.Om, c.ldom, l);
  E.stage_into(OmX, l, c.Xc, c.ldxc, s);
  TS Phi = E.stage_in(SIDE_M, c.Phi, c.ldphi, l2, c.kPhi);
  TS Xr = E.stage_in(SIDE_M, c.Xr, c.ldxr, s, c.kXr);
  TS YW = E.new_ts(SIDE_M, l + s);
  TS Yr = E.new_ts(SIDE_N, l2);
  sketch_view(E, OmX, Phi, YW, Yr);
  TS Yc = E.slice(YW, 0, l), W = E.slice(YW, l, s), Xc = E.slice(OmX, l, s);
  double* Z = E.alloc((int64_t)s * s);
  E.cross(SIDE_M, Xr, W, Z);                      // Z = Xi_r^* A Xi_c      (s x s)
  E.orth(SIDE_M, Yc, nullptr, nullptr);           // Q_c R_c := Y_c
  E.orth(SIDE_N, Yr, nullptr, nullptr, true);     // Q_r R_r := Y_r (shifted CholeskyQR3, R22)
  double* Uc = E.alloc((int64_t)s * l);
  double* Ur = E.alloc((int64_t)s * l2);
  E.cross(SIDE_M, Xr, Yc, Uc);                    // Xi_r^* Q_c            (s x l)
  E.cross(SIDE_N, Xc, Yr, Ur);                    // Xi_c^* Q_r            (s x l2)
  double* Tc = E.alloc((int64_t)l * l);
  double* Tr = E.alloc((int64_t)l2 * l2);
  small_qr(E, Uc, s, l, Tc);                      // U_c T_c := Xi_r^* Q_c
  small_qr(E, Ur, s, l2, Tr);                     // U_r T_r := Xi_c^* Q_r
  double* Tcp = E.alloc((int64_t)l * l);
  double* Trp = E.alloc((int64_t)l2 * l2);
  small_pinv(E, Tc, l, Tcp);
  small_pinv(E, Tr, l2, Trp);
  double* M1 = E.alloc((int64_t)l * s);
  double* X = E.alloc((int64_t)l * l2);
  double* C1 = E.alloc((int64_t)l * l2);
  double* core = E.alloc((int64_t)l * l2);
  double* scratch = E.alloc(2 * 512 * 512 + 4096);
  double* Ux = E.alloc((int64_t)l2 * l);
  double* Vx = E.alloc((int64_t)l * l);
  double* sx = E.alloc(l);
  double* A1 = E.alloc((int64_t)l * k);
  double* B1 = E.alloc((int64_t)l2 * k);
  double* Ul = E.alloc((int64_t)l2 * l);
  double* Vr = E.alloc((int64_t)l * l);
  double* lam = E.alloc(l);
  if (E.live()) {
    E.chk(launch_small_gemm(1, 0, l, s, s, Uc, s, Z, s, M1, l, E.st));         // U_c^* Z
    E.chk(launch_small_gemm(0, 0, l, l2, s, M1, l, Ur, s, X, l, E.st));        // U_c^* Z U_r   (l x l2)
    if (c.variant == RSVD_EXT_BWZ2) {
      E.chk(launch_small_gemm(0, 0, l, l2, l, Tcp, l, X, l, C1, l, E.st));     // T_c^+ (.)
      E.chk(launch_small_gemm(0, 1, l, l2, l2, C1, l, Trp, l2, core, l, E.st)); // (.) (T_r^*)^+
    } else {
      // [[X]]_k = Vx diag(sx) Ux^T from Jacobi on X^T (l2 x l): X^T = Ux S Vx^T
      E.chk(launch_jacobi_t(X, l, 1, l2, l, Ux, sx, Vx, scratch, E.ctx->dstat, E.st, 0));
      E.chk(launch_small_gemm(0, 0, l, k, l, Tcp, l, Vx, l, A1, l, E.st));      // T_c^+ U_x
      E.chk(launch_scale_cols(A1, l, l, k, sx, E.st));                           //   diag(sigma_x)
      E.chk(launch_small_gemm(0, 0, l2, k, l2, Trp, l2, Ux, l2, B1, l2, E.st)); // T_r^+ V_x
      E.chk(launch_small_gemm(0, 1, l, l2, k, A1, l, B1, l2, core, l, E.st));   // rank-k core
    }
    // tsvd(core, k): Jacobi on core^T (l2 x l): core^T = Ul S Vr^T  ->  core = Vr S Ul^T
    E.chk(launch_jacobi_t(core, l, 1, l2, l, Ul, lam, Vr, scratch, E.ctx->dstat, E.st, 0));
  }
  write_outputs(E, SIDE_M, SIDE_N, Yc, Yr, Vr, Ul, lam, l, k);
}

// One pass over the rows of A: Y = A X (side M, written panel by panel) and,
// with Z, Z = A^T (A X) = sum over row panels of A[panel]^T Y[panel] (side N, accumulated in panel
// order, then all-reduced over the row shards).  The panels are small enough to stay in L2
// between the two products: each panel is read from HBM once by the range view (A loaded
// evict_last) and re-read from L2 by the co-range view.  T: side-N scratch of X's width.
constexpr double kRowPanelBytes = 48.0 * 1024 * 1024;
void row_pass(Exec& E, const TS& X, const TS& Y, const TS* Z, const TS& T) {
  const double esz = (E.dtype == RSVD_F32) ? 4.0 : 8.0;
  static const double panel_bytes = [] {
    const char* e = getenv("RSVD_ROW_PANEL_MB");   // A/B experiments only
    return e ? atof(e) * 1024 * 1024 : kRowPanelBytes;
  }();
  int64_t P = (int64_t)(panel_bytes / (esz * (double)E.n));
  P = std::max<int64_t>(128, P / 128 * 128);
  const int w = X.w;
  for (int64_t r0 = 0; r0 < E.m; r0 += P) {
    const int64_t nr = std::min<int64_t>(P, E.m - r0);
    TS Yp;
    Yp.p = Y.p + r0;
    Yp.rows = nr;
    Yp.ld = Y.ld;
    Yp.w = w;
    E.view(SIDE_N, X, Yp, r0, nr, /*a_keep=*/Z != nullptr);   // Y[panel] = A[panel] X
    if (!Z) continue;
    const bool first = (r0 == 0);
    E.view(SIDE_M, Yp, first ? *Z : T, r0, nr);                // A[panel]^T Y[panel]
    if (!first && E.live()) E.chk(launch_add_cols(T.p, T.ld, Z->p, Z->ld, Z->rows, w, E.st));
  }
  if (!Z) return;
  if (E.m == 0 && E.live()) E.chk(launch_fill(Z->p, Z->ld * w, 0.0, E.st));
  if (E.collective()) E.allreduce(Z->p, Z->ld * w);             // over the row shards
}

// Single pass over the rows of A: Y_c = A Omega and Yhat_r = A^T Y_c from one
// row pass, then Q_c R_c := Y_c, B^* = Yhat_r R_c^+ (TSVD pseudo-inverse) and the rank-k
// SVD of Q_c B through qr(B^*).  With R_c invertible this is Alg. 2, v = 2.
void alg_row_stream(Exec& E) {
  const Call& c = E.call;
  const int l = c.k + c.p;
  TS Om = E.stage_in(SIDE_N, c.Om, c.ldom, l, c.kOm);
  TS Yc = E.new_ts(SIDE_M, l);
  TS Yh = E.new_ts(SIDE_N, l);
  TS T = E.new_ts(SIDE_N, l);
  row_pass(E, Om, Yc, &Yh, T);
  double* Rc = E.alloc((int64_t)l * l);
  E.orth(SIDE_M, Yc, Rc, nullptr);                           // Q_c R_c := Y_c
  // R_c^+: guarded triangular inverse — equal to the TSVD pseudo-inverse for an invertible R_c and
  // for the guard-zeroed rows / columns of an exactly rank-deficient one (reading R26)
  double* Rcp = E.alloc((int64_t)l * l);
  if (E.live()) E.chk(launch_tri_inv(Rc, l, Rcp, nullptr, E.st));
  TS Bt = E.new_ts(SIDE_N, l);
  E.tsmm(Yh.p, Yh.ld, Yh.rows, l, Rcp, l, l, Bt.p, Bt.ld, 0); // B^* = Yhat_r R_c^+
  double* Rb = E.alloc((int64_t)l * l);
  E.orth(SIDE_N, Bt, Rb, nullptr);                           // B^* = Q_b R_b
  double* Ul = E.alloc((int64_t)l * l);
  double* Vr = E.alloc((int64_t)l * l);
  double* lam = E.alloc(l);
  E.core_svd(Rb, l, 1, Vr, lam, Ul);                         // R_b = Ul S Vr^T -> Q_c B = Q_c Vr S Ul^T Q_b^T
  write_outputs(E, SIDE_M, SIDE_N, Yc, Bt, /*Uh=*/Vr, /*Vh=*/Ul, lam, l, c.k);
}

// Block Krylov method for a matrix read row wise: A^T A X in ONE row pass, so the
// Krylov blocks of Alg. 9 need about half the reads of A (oracle.row_block_krylov).
//   v odd : K_r = [A^TA Omega, (A^TA)^2 Omega, ...] ((v-1)/2 row passes; intermediate blocks
//           orthonormalised, the last raw, as Alg. 9 lines 3-6), qr(K_r) by BCGS2, Q_c R_c = A Q_r
//           (one range view), tsvd(R_c): (v-1)/2 + 1 reads instead of v.
//   v even: the same passes also give the range blocks A Q^i: K_c = [A Omega, A Q^1, ...]
//           (the last one a plain range view), qr(K_c), Q_r R_r = A^T Q_c, tsvd(R_r): v/2 + 1 reads.
void alg_krylov_rows(Exec& E) {
  const Call& c = E.call;
  const int l = c.k + c.p, v = c.v;
  const bool even = (v % 2 == 0);
  const int nb = even ? v / 2 : (v - 1) / 2;
  const int W = nb * l;
  TS X = E.stage_in(SIDE_N, c.Om, c.ldom, l, c.kOm);         // Q^0 = Omega
  TS T = E.new_ts(SIDE_N, l);
  double* Rw = E.alloc((int64_t)W * W);
  double* Ul = E.alloc((int64_t)W * W);
  double* Vr = E.alloc((int64_t)W * W);
  double* lam = E.alloc(W);
  const int want_j = (c.flags & RSVD_SQUARED) ? 2 : 0;
  if (!even) {
    TS K = E.new_ts(SIDE_N, W);
    TS Y = E.new_ts(SIDE_M, l);
    for (int b = 0; b < nb; ++b) {
      TS Kb = E.slice(K, b * l, l);
      row_pass(E, X, Y, &Kb, T);                               // K_b = A^T A Q^{b}
      if (b < nb - 1) {
        E.orth(SIDE_N, Kb, nullptr, nullptr);                  // Q^{b+1} = qr(K_b).Q
        X = Kb;
      }
    }
    E.bcgs2(SIDE_N, K, l, /*first_orthonormal=*/nb > 1);      // Q_r = qr(K_r)   (line 15)
    TS Qc = E.new_ts(SIDE_M, W);
    E.view(SIDE_N, K, Qc);                                     // A Q_r           (line 16)
    E.orth(SIDE_M, Qc, Rw, nullptr);
    E.core_svd(Rw, W, 1, Vr, lam, Ul, want_j);                 // R_c = Ul S Vr^T (line 17)
    write_outputs(E, SIDE_M, SIDE_N, Qc, K, Ul, Vr, lam, W, c.k);
  } else {
    TS K = E.new_ts(SIDE_M, W);
    TS Z[2] = {E.new_ts(SIDE_N, l), E.new_ts(SIDE_N, l)};
    for (int b = 0; b < nb; ++b) {
      TS Kb = E.slice(K, b * l, l);
      if (b < nb - 1) {
        row_pass(E, X, Kb, &Z[b & 1], T);                      // K_b = A Q^b, Z = A^T A Q^b
        E.orth(SIDE_N, Z[b & 1], nullptr, nullptr);            // Q^{b+1}
        X = Z[b & 1];
      } else {
        E.view(SIDE_N, X, Kb);                                 // last block: range view only
      }
    }
    E.bcgs2(SIDE_M, K, l, /*first_orthonormal=*/false);       // Q_c = qr(K_c)   (line 10)
    TS Qr = E.new_ts(SIDE_N, W);
    E.view(SIDE_M, K, Qr);                                     // A^T Q_c         (line 11)
    E.orth(SIDE_N, Qr, Rw, nullptr);
    E.core_svd(Rw, W, 1, Vr, lam, Ul, want_j);                 // R_r = Vh S Uh^T (line 12)
    write_outputs(E, SIDE_M, SIDE_N, K, Qr, Vr, Ul, lam, W, c.k);
  }
}

// Alg. 3 QrQc on B = A (tr = false) or B = A^T (tr = true), v >= 0 views, starting
// from the staged test matrix Q (on B's co-range side).  Returns the final basis: Q_r of B
// (B's co-range side, in Q) for even v, Q_c of B (B's range side, new block) for odd v.
TS qrqc(Exec& E, bool tr, TS Q, int v, int l) {
  const Side side_c = tr ? SIDE_N : SIDE_M;
  const Side side_r = tr ? SIDE_M : SIDE_N;
  TS Qc = E.new_ts(side_c, l);
  for (int j = 1; j <= v; ++j) {
    if (j % 2 == 1) {
      E.view(side_r, Q, Qc);                 // B Q_r
      E.orth(side_c, Qc, nullptr, nullptr);
    } else {
      E.view(side_c, Qc, Q);                 // B^* Q_c
      E.orth(side_r, Q, nullptr, nullptr);
    }
  }
  return (v % 2 == 0) ? Q : Qc;
}

// tsvd(F, k) of the wide F = Ft^T (l x n) and its right vectors / values:
// Ft = Q_f R_f (CholeskyQR2) -> F = R_f^T Q_f^T; Jacobi on R_f: R_f = Lf S Rf^T
// -> F = Rf S (Q_f Lf)^T: right vectors Q_f Lf, values S.  Writes V (n x k) and S (k).
void tsvd_wide_right(Exec& E, const TS& Ft, int l, int k, double* lam_out, TS* Qf_out, double** Lf_out) {
  double* Rf = E.alloc((int64_t)l * l);
  E.orth(SIDE_N, Ft, Rf, nullptr);
  double* Lf = E.alloc((int64_t)l * l);
  double* Rr = E.alloc((int64_t)l * l);
  E.core_svd(Rf, l, /*trans=*/0, Lf, lam_out, Rr, 2);
  *Qf_out = Ft;
  *Lf_out = Lf;
  (void)k;
}

// emit V = Q W[:, :k] (side N) and S = lam2 (k) to the caller
void write_normal_outputs(Exec& E, const TS& Q, const double* W, const double* lam2, int k) {
  const Call& c = E.call;
  if (c.kV != PTR_NULL) {
    int64_t ld;
    double* o = E.out_ptr(c.V, c.ldv, Q.rows, k, c.kV, &ld);
    E.lift(Q, W, k, o, ld);
  }
  if (c.kS != PTR_NULL) {
    int64_t ld;
    double* so = E.out_ptr(c.S, k, k, 1, c.kS, &ld);
    if (E.live()) E.chk(launch_copy_cols(lam2, k, so, k, k, 1, E.st));
  }
}

// Alg. 4: modified prolonged (Nystrom) TEVD of the normal matrix A^T A with v views
void alg_nystrom(Exec& E) {
  const Call& c = E.call;
  const int l = c.k + c.p, v = c.v;
  // lines 1-7: Q_r (side N) from orth(Omega) (v = 2), QrQc(A, v-2) (even), QrQc(A^T, v-2) (odd)
  const bool tr = (v % 2 == 1);
  TS Q0 = E.stage_in(tr ? SIDE_M : SIDE_N, c.Om, c.ldom, l, c.kOm);
  TS Qr;
  if (v == 2) {
    E.orth(SIDE_N, Q0, nullptr, nullptr);
    Qr = Q0;
  } else {
    Qr = qrqc(E, tr, Q0, v - 2, l);
  }
  // line 8: Y_r = A^T (A Q_r)   (two views)
  TS Yc = E.new_ts(SIDE_M, l);
  TS Yr = E.new_ts(SIDE_N, l);
  E.view(SIDE_N, Qr, Yc);
  E.view(SIDE_M, Yc, Yr);
  // lines 9-10: nu = 2.2e-16 ||Y_r||_2, Y_r += nu Q_r
  double* G = E.alloc((int64_t)l * l);
  double* nu = E.alloc(1);
  E.cross(SIDE_N, Yr, Yr, G);
  if (E.live()) {
    E.chk(launch_nys_nu(G, l, nu, E.st));
    E.chk(launch_axpy_dev(Yr.p, Yr.ld, Qr.p, Qr.ld, Yr.rows, l, nu, E.st));
  }
  // lines 11-12: B = Q_r^T Y_r, C_L = chol((B + B^T)/2, LOWER) = R^T
  double* B = E.alloc((int64_t)l * l);
  double* Bs = E.alloc((int64_t)l * l);
  double* R = E.alloc((int64_t)l * l);
  double* Ri = E.alloc((int64_t)l * l);
  E.cross(SIDE_N, Qr, Yr, B);
  if (E.live()) {
    E.chk(launch_symmetrize(B, l, Bs, E.st));
    E.chk(launch_chol_ref(Bs, nullptr, l, 0.0, R, Ri, E.ctx->dstat, E.st));
  }
  // line 13: F = C_L^-1 Y_r^T  ->  F^T = Y_r R^-1
  TS Ft = E.new_ts(SIDE_N, l);
  E.tsmm(Yr.p, Yr.ld, Yr.rows, l, Ri, l, l, Ft.p, Ft.ld, 0);
  // line 14: [~, Lam_hat, V] = tsvd(F, k)
  double* lam = E.alloc(l);
  TS Qf;
  double* Lf = nullptr;
  tsvd_wide_right(E, Ft, l, c.k, lam, &Qf, &Lf);
  // line 15: Lambda^2 = Lam_hat^2 - nu, negatives -> 0
  double* lam2 = E.alloc(l);
  if (E.live()) E.chk(launch_nys_eig(lam, c.k, nu, lam2, E.st));
  write_normal_outputs(E, Qf, Lf, lam2, c.k);
}

// Alg. 5: modified pinched TEVD of A^T A with v views
void alg_pinched(Exec& E) {
  const Call& c = E.call;
  const int l = c.k + c.p, v = c.v;
  // lines 1-5: Q_r = QrQc(A^T, v-1) (even v) or QrQc(A, v-1) (odd v): a basis on side N
  const bool tr = (v % 2 == 0);
  TS Q0 = E.stage_in(tr ? SIDE_M : SIDE_N, c.Om, c.ldom, l, c.kOm);
  TS Qr = qrqc(E, tr, Q0, v - 1, l);
  // line 6: B_c = A Q_r (one view)
  TS Bc = E.new_ts(SIDE_M, l);
  E.view(SIDE_N, Qr, Bc);
  // line 7: tevd(B_c^T B_c, k) through B_c = Q_b R_b: eigenvectors = right singular vectors of
  // R_b, eigenvalues = sigma(R_b)^2 (the same TEVD without forming the Gram)
  double* Rb = E.alloc((int64_t)l * l);
  E.orth(SIDE_M, Bc, Rb, nullptr);
  double* Ul = E.alloc((int64_t)l * l);
  double* Vr = E.alloc((int64_t)l * l);
  double* lam = E.alloc(l);
  E.core_svd(Rb, l, /*trans=*/1, Vr, lam, Ul, 2);  // Jacobi on R_b^T: its left vectors = right(R_b)
  if (E.live()) E.chk(launch_square(lam, l, E.st));
  // line 8: V_p = Q_r Vhat_p
  write_normal_outputs(E, Qr, Vr, lam, c.k);
}

// primitives -------------------------------------------------------------------------------
void prim_view(Exec& E) {
  const Call& c = E.call;
  const Side from = c.trans ? SIDE_M : SIDE_N;
  const Side to = c.trans ? SIDE_N : SIDE_M;
  TS X = E.stage_in(from, c.Om, c.ldom, c.w, c.kOm);
  TS Y = E.new_ts(to, c.w);
  E.view(from, X, Y);
  int64_t ld;
  double* o = E.out_ptr(c.U, c.ldu, Y.rows, c.w, c.kU, &ld);
  if (E.live()) E.chk(launch_copy_cols(Y.p, Y.ld, o, ld, Y.rows, c.w, E.st));
}

void prim_orth(Exec& E) {
  const Call& c = E.call;
  TS Y;
  Y.rows = c.rows;
  Y.ld = round_up(std::max<int64_t>(c.rows, 1), 32);
  Y.w = c.w;
  Y.p = E.alloc(Y.ld * c.w);
  E.h2d.push_back({Y.p, Y.ld, c.U, c.ldu, Y.rows, c.w});
  // orth on a local (unsharded) side of arbitrary length: emulate with m = rows
  double* R = E.alloc((int64_t)c.w * c.w);
  const int64_t n_save = E.n;
  E.n = c.rows;
  E.orth(SIDE_N, Y, R, nullptr, (c.flags & RSVD_ORTH_SHIFTED) != 0);  // SIDE_N: never all-reduced
  E.n = n_save;
  int64_t ld;
  double* o = E.out_ptr(c.U, c.ldu, Y.rows, c.w, c.kU, &ld);
  if (E.live()) E.chk(launch_copy_cols(Y.p, Y.ld, o, ld, Y.rows, c.w, E.st));
  if (c.kR != PTR_NULL) {
    double* ro = E.out_ptr(c.R, c.w, c.w, c.w, c.kR, &ld);
    if (E.live()) E.chk(launch_copy_cols(R, c.w, ro, ld, c.w, c.w, E.st));
  }
}

void prim_fused(Exec& E) {
  const Call& c = E.call;
  const int l = c.w, l2 = c.l2;
  if (E.dtype != RSVD_F64) {  // the fused fp32 sketch is not built: Alg. 7 runs it as two views
    E.chk(RSVD_E_DTYPE);
    return;
  }
  TS Om = E.stage_in(SIDE_N, c.Om, c.ldom, l, c.kOm);
  TS Phi = E.stage_in(SIDE_M, c.Phi, c.ldphi, l2, c.kPhi);
  TS Yc = E.new_ts(SIDE_M, l), Yr = E.new_ts(SIDE_N, l2);
  if (l > kFusedMaxL || (l2 + 7) / 8 > kFusedMaxL2T || (c.flags & RSVD_ONE_READ)) {
    // wide sketches (or RSVD_ONE_READ): the cluster kernel (one read of A)
    if (!sketch_view_cluster(E, Om, Phi, Yc, Yr, true)) {
      E.chk(RSVD_E_ARG);
      return;
    }
    int64_t ld;
    double* o1 = E.out_ptr(c.U, c.ldu, Yc.rows, l, c.kU, &ld);
    if (E.live()) E.chk(launch_copy_cols(Yc.p, Yc.ld, o1, ld, Yc.rows, l, E.st));
    double* o2 = E.out_ptr(c.V, c.ldv, Yr.rows, l2, c.kV, &ld);
    if (E.live()) E.chk(launch_copy_cols(Yr.p, Yr.ld, o2, ld, Yr.rows, l2, E.st));
    return;
  }
  FusedArgs a;
  a.A = E.A;
  a.rows = E.m;
  a.n = E.n;
  a.lda = E.lda;
  a.Om = Om.p;
  a.ldom = Om.ld;
  a.l = l;
  a.Phi = Phi.p;
  a.ldphi = Phi.ld;
  a.l2 = l2;
  a.grid_cap = E.ctx->sms;
  plan_view(VIEW_FUSED, E.m, E.n, l2, E.ctx->sms, &a.S, &a.KTS);
  const int nsb = fused_strips(E.n);
  a.yc_atomic = ((double)nsb * Yc.ld * l * 8.0 > kYcSlotBudget) ? 1 : 0;
  E.nondet |= a.yc_atomic;
  double* ycs = a.yc_atomic ? Yc.p : E.alloc((int64_t)nsb * Yc.ld * l);
  a.yc = ycs;
  a.ldyc = Yc.ld;
  a.yc_slot_stride = (int64_t)Yc.ld * l;
  double* yrs = (a.S == 1) ? Yr.p : E.alloc((int64_t)a.S * Yr.ld * l2);
  a.yr = yrs;
  a.ldyr = Yr.ld;
  a.yr_slot_stride = (int64_t)Yr.ld * l2;
  E.view_bytes += (double)E.m * E.n * 8.0;
  E.view_flops += 2.0 * E.m * E.n * (l + l2);
  ++E.view_launches;
  if (E.live()) {
    if (a.yc_atomic) E.chk(launch_fill(Yc.p, Yc.ld * l, 0.0, E.st));
    int e0 = -1, e1 = -1;
    E.ev_record(&e0);
    E.chk(launch_view_fused(a, E.st));
    E.ev_record(&e1);
    if (e0 >= 0) E.ev_pairs.push_back({e0, e1});
    if (!a.yc_atomic) E.chk(launch_slot_sum(ycs, Yc.ld, a.yc_slot_stride, nsb, Yc.rows, l, Yc.p, Yc.ld, E.st));
    if (a.S > 1) E.chk(launch_slot_sum(yrs, Yr.ld, a.yr_slot_stride, a.S, Yr.rows, l2, Yr.p, Yr.ld, E.st));
  }
  int64_t ld;
  double* o1 = E.out_ptr(c.U, c.ldu, Yc.rows, l, c.kU, &ld);
  if (E.live()) E.chk(launch_copy_cols(Yc.p, Yc.ld, o1, ld, Yc.rows, l, E.st));
  double* o2 = E.out_ptr(c.V, c.ldv, Yr.rows, l2, c.kV, &ld);
  if (E.live()) E.chk(launch_copy_cols(Yr.p, Yr.ld, o2, ld, Yr.rows, l2, E.st));
}

void prim_core(Exec& E) {
  const Call& c = E.call;
  const int r = (int)c.rows, cc = c.cols;
  double* M = E.alloc((int64_t)r * cc);
  E.h2d.push_back({M, r, c.Om, c.ldom, r, cc});
  int64_t ldU, ldV, ldS;
  double* Uo = E.out_ptr(c.U, r, r, cc, c.kU == PTR_NULL ? PTR_DEVICE : c.kU, &ldU);
  double* So = E.out_ptr(c.S, cc, cc, 1, c.kS, &ldS);
  double* Vo = E.out_ptr(c.V, cc, cc, cc, c.kV, &ldV);
  // jacobi writes Ul with ld r and Vr with ld c: route through arena buffers
  double* Ul = E.alloc((int64_t)r * cc);
  double* Vr = E.alloc((int64_t)cc * cc);
  double* sv = E.alloc(cc);
  double* scratch = E.alloc(2 * 512 * 512 + 4096);
  if (E.live()) {
    E.chk(launch_jacobi_t(M, r, 0, r, cc, Ul, sv, Vr, scratch, E.ctx->dstat, E.st,
                           (c.flags & RSVD_CORE_NO_J) ? 0 : 1));
    if (c.kU != PTR_NULL) E.chk(launch_copy_cols(Ul, r, Uo, ldU, r, cc, E.st));
    if (c.kS != PTR_NULL) E.chk(launch_copy_cols(sv, cc, So, ldS, cc, 1, E.st));
    if (c.kV != PTR_NULL) E.chk(launch_copy_cols(Vr, cc, Vo, ldV, cc, cc, E.st));
  }
}

void run_alg(Exec& E) {
  switch (E.call.alg) {
    case 0: alg_subspace(E); break;
    case 1: alg_krylov(E); break;
    case 2: alg_single_pass(E); break;
    case 3: alg_nystrom(E); break;
    case 4: alg_pinched(E); break;
    case 5: alg_extended(E); break;
    case 6: alg_row_stream(E); break;
    case 7: alg_krylov_rows(E); break;
    case 10: prim_view(E); break;
    case 11: prim_fused(E); break;
    case 12: prim_orth(E); break;
    case 13: prim_core(E); break;
    default: E.chk(RSVD_E_ARG);
  }
  E.flush_outputs();
}

std::string call_key(const Call& c, const Exec& E, const rsvd_ctx* ctx) {
  char buf[1024];
  snprintf(buf, sizeof buf,
           "a%d k%d p%d v%d in%d l2%d lc%d t%d w%d r%lld c%d f%u dt%d A%p m%lld n%lld lda%lld U%d S%d V%d R%d ar%p nr%d "
           "s%d x%d sm%d",
           c.alg, c.k, c.p, c.v, c.input, c.l2, c.lc, c.trans, c.w, (long long)c.rows, c.cols, c.flags, E.dtype,
           // the captured graph reads A in place: the device A (fp64 or fp32) is part of the key
           E.dtype == RSVD_F32 ? (const void*)E.A32 : (const void*)E.A, (long long)E.m, (long long)E.n,
           (long long)E.lda, c.kU != PTR_NULL, c.kS != PTR_NULL,
           c.kV != PTR_NULL, c.kR != PTR_NULL, (void*)ctx->arena, ctx->nranks + (ctx->comm ? 1000 : 0), c.s,
           c.variant, ctx->sms);
  return std::string(buf);
}

// Stage A (host memory -> first arena allocation) and bind the executor to the device A.
void bind_A(Exec& E, const Call& call) {
  if (!call.A) return;
  E.m = call.A->m_local;
  E.m_glob = call.A->m;
  E.n = call.A->n;
  E.lda = call.A->lda;
  E.dtype = call.A->dtype;
  const int esz = E.dtype == RSVD_F32 ? 4 : 8;
  const bool misaligned = call.kA == PTR_DEVICE &&
                         ((reinterpret_cast<uintptr_t>(call.A->data) & 15) || ((call.A->lda * esz) & 15));
  if (call.kA == PTR_HOST || misaligned) {
    // host A, or a device A whose base / row stride violates TMA's 16-byte rule: copy into an
    // aligned workspace block (row-major copy: width n elements, height m rows)
    E.lda = round_up(call.A->n, 32);
    void* Ad = E.alloc(E.m * E.lda * esz / 8);
    E.h2d.push_back({Ad, E.lda, call.A->data, call.A->lda, E.n, E.m, esz});
    E.A = static_cast<const double*>(Ad);
    E.a_restaged = 1;
  } else {
    E.A = static_cast<const double*>(call.A->data);
  }
  if (E.dtype == RSVD_F32) {
    E.A32 = reinterpret_cast<const float*>(E.A);
    E.A = nullptr;
  }
  // the n-long side is sharded too for the generalized subspace iteration and block Krylov
  if (call.alg == 0 || call.alg == 1) E.plan_shard_n();
}

// Wait for the ctx stream.  With a communicator: its wait (NCCL polls ncclCommGetAsyncError and
// aborts after RSVD_COMM_TIMEOUT_S seconds, default 600, instead of hanging on a dead peer).
int wait_stream(rsvd_ctx* ctx) {
  std::string e;
  int r;
  if (ctx->comm) {
    static const double timeout_s = [] {
      const char* v = getenv("RSVD_COMM_TIMEOUT_S");
      return v ? atof(v) : 600.0;
    }();
    r = ctx->comm->wait(ctx->stream, timeout_s, &e);
  } else {
    cudaError_t se = cudaStreamSynchronize(ctx->stream);
    r = se == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
    if (r) e = std::string("CUDA error: ") + cudaGetErrorString(se);
  }
  if (r) set_err(ctx, "%s", e.c_str());
  return r;
}

int execute_impl(rsvd_ctx* ctx, Call& call, rsvd_info* info);

// A rank whose call fails before its collectives complete would leave its peers blocked in them:
// abort the communicator (loopback: release the peers' host barriers; NCCL: ncclCommAbort).
// Numerical failures are detected after the whole call completed and leave the comm intact.
// NVTX range per API call (visible in Nsight timelines; a no-op without a tool attached)
const char* alg_name(int alg) {
  switch (alg) {
    case 0: return "rsvd_subspace";
    case 1: return "rsvd_block_krylov";
    case 2: return "rsvd_single_pass";
    case 3: return "rsvd_nystrom";
    case 4: return "rsvd_pinched";
    case 5: return "rsvd_single_pass_extended";
    case 6: return "rsvd_row_stream";
    case 7: return "rsvd_block_krylov_rows";
    case 10: return "rsvd_view";
    case 11: return "rsvd_view_fused";
    case 12: return "rsvd_orth";
    case 13: return "rsvd_core_svd";
    default: return "rsvd";
  }
}

int execute(rsvd_ctx* ctx, Call& call, rsvd_info* info) {
  nvtxRangePushA(alg_name(call.alg));
  const int r = execute_impl(ctx, call, info);
  nvtxRangePop();
  if (r != RSVD_OK && r != RSVD_E_NUMERIC && ctx->comm) ctx->comm->abort();
  return r;
}

int execute_impl(rsvd_ctx* ctx, Call& call, rsvd_info* info) {
  if (info) memset(info, 0, sizeof(*info));
  cudaSetDevice(ctx->device);
  call.kA = call.A ? ptr_kind(call.A->data, ctx->device) : PTR_NULL;
  call.kOm = ptr_kind(call.Om, ctx->device);
  call.kPhi = ptr_kind(call.Phi, ctx->device);
  call.kU = ptr_kind(call.U, ctx->device);
  call.kS = ptr_kind(call.S, ctx->device);
  call.kV = ptr_kind(call.V, ctx->device);
  call.kR = ptr_kind(call.R, ctx->device);
  call.kXr = ptr_kind(call.Xr, ctx->device);
  call.kXc = ptr_kind(call.Xc, ctx->device);
  const bool profile = (call.flags & RSVD_PROFILE) != 0;
  if (ctx->pending) {
    set_err(ctx, "a RSVD_ASYNC call on this ctx has not been completed by rsvd_wait");
    return RSVD_E_STATE;
  }
  if (profile && (call.flags & RSVD_ASYNC)) {
    set_err(ctx, "RSVD_PROFILE cannot be combined with RSVD_ASYNC");
    return RSVD_E_ARG;
  }
  // ---- 1. sizing pass (fake base)
  Exec sz(ctx, call, true, nullptr);
  bind_A(sz, call);
  run_alg(sz);
  if (sz.rc) {
    set_err(ctx, "invalid configuration (planning failed, code %d)", sz.rc);
    return sz.rc;
  }
  const size_t need = sz.peak + 4096;
  if (need > ctx->arena_size) {
    cudaStreamSynchronize(ctx->stream);
    for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
    ctx->graphs.clear();
    ctx->graph_kernels.clear();
    if (ctx->arena) cudaFree(ctx->arena);
    ctx->arena = nullptr;
    ctx->arena_size = 0;
    const size_t bytes = (size_t)round_up((int64_t)(need * 1.25), 1 << 20);
    if (cudaMalloc(&ctx->arena, bytes) != cudaSuccess) {
      cudaGetLastError();
      set_err(ctx, "cudaMalloc of %zu bytes of workspace failed", bytes);
      return RSVD_E_NOMEM;
    }
    ctx->arena_size = bytes;
  }
  // ---- 2. enqueue (or record-only) pass at real addresses
  Exec E(ctx, call, false, ctx->arena);
  E.profile = profile;
  bind_A(E, call);
  cudaStream_t st = ctx->stream;
  // the loopback communicator synchronises ranks on the host: not capturable, enqueue directly
  const bool use_graph = !(call.flags & RSVD_NO_GRAPH) && !profile && (!ctx->comm || ctx->comm->graph_ok());
  const std::string key = call_key(call, E, ctx);
  auto it = use_graph ? ctx->graphs.find(key) : ctx->graphs.end();
  const bool replay = use_graph && it != ctx->graphs.end();

  auto do_h2d = [&](const std::vector<Exec::H2D>& lst) -> int {
    for (auto& t : lst)
      if (cudaMemcpy2DAsync(t.dst, t.ldd * t.esz, t.src, t.lds * t.esz, t.rows * t.esz, t.cols, cudaMemcpyDefault,
                            st) != cudaSuccess)
        return RSVD_E_CUDA;
    return RSVD_OK;
  };
  int rc = RSVD_OK;
  if (use_graph) {
    cudaGraphExec_t ge = nullptr;
    if (replay) {
      E.launch_off = true;  // record transfers only
      run_alg(E);
      ge = it->second;
    } else {
      cudaGraph_t g;
      if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        set_err(ctx, "cudaStreamBeginCapture failed");
        return RSVD_E_CUDA;
      }
      cudaMemsetAsync(ctx->dstat, 0, sizeof(DevStatus), st);
      cudaMemsetAsync(ctx->counter, 0, 256, st);
      run_alg(E);
      cudaError_t ce = cudaStreamEndCapture(st, &g);
      if (E.rc || ce != cudaSuccess) {
        cudaGetLastError();
        if (ce == cudaSuccess) cudaGraphDestroy(g);
        set_err(ctx, "enqueue failed during capture (rc %d, %s)", E.rc, cudaGetErrorString(ce));
        return E.rc ? E.rc : RSVD_E_CUDA;
      }
      {
        size_t nn = 0;
        cudaGraphGetNodes(g, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        if (nn) cudaGraphGetNodes(g, nodes.data(), &nn);
        int kn = 0;
        for (auto nd : nodes) {
          cudaGraphNodeType ty;
          if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++kn;
        }
        ctx->graph_kernels[key] = kn;
      }
      if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
        cudaGetLastError();
        cudaGraphDestroy(g);
        set_err(ctx, "cudaGraphInstantiate failed");
        return RSVD_E_CUDA;
      }
      cudaGraphDestroy(g);
      ctx->graphs[key] = ge;
    }
    rc = do_h2d(E.h2d);
    if (rc == RSVD_OK && cudaGraphLaunch(ge, st) != cudaSuccess) rc = RSVD_E_CUDA;
  } else {
    // direct enqueue: collect transfers first (launch-free pass), then launch
    Exec pre(ctx, call, false, ctx->arena);
    pre.launch_off = true;
    bind_A(pre, call);
    run_alg(pre);
    rc = do_h2d(pre.h2d);
    if (rc == RSVD_OK) {
      cudaMemsetAsync(ctx->dstat, 0, sizeof(DevStatus), st);
      int ev0 = -1, ev1 = -1;
      E.ev_record(&ev0);
      run_alg(E);
      E.ev_record(&ev1);
      rc = E.rc;
      if (profile && ev0 >= 0) E.ev_pairs.insert(E.ev_pairs.begin(), {ev0, ev1});
    }
  }
  if (rc == RSVD_OK) {
    for (auto& t : E.d2h)
      if (cudaMemcpy2DAsync(t.dst, t.ldd * t.esz, t.src, t.lds * t.esz, t.rows * t.esz, t.cols, cudaMemcpyDefault,
                            st) != cudaSuccess) {
        rc = RSVD_E_CUDA;
        break;
      }
  }
  if (rc == RSVD_OK) cudaMemcpyAsync(ctx->hstat, ctx->dstat, sizeof(DevStatus), cudaMemcpyDefault, st);
  rsvd_info base_info;
  memset(&base_info, 0, sizeof(base_info));
  base_info.graph_replayed = replay ? 1 : 0;
  base_info.host_staged = (call.kA == PTR_HOST || call.kOm == PTR_HOST || call.kPhi == PTR_HOST ||
                           call.kXr == PTR_HOST || call.kXc == PTR_HOST ||
                           call.kU == PTR_HOST || call.kV == PTR_HOST || call.kS == PTR_HOST)
                              ? 1
                              : 0;
  if (sz.a_restaged && call.kA == PTR_DEVICE) base_info.host_staged = 2;
  base_info.view_launches = sz.view_launches;
  if (use_graph) base_info.kernel_launches = ctx->graph_kernels[key];
  base_info.view_bytes = sz.view_bytes;
  base_info.view_flops = sz.view_flops;
  base_info.nondeterministic = sz.nondet;
  base_info.views = call.info_views;
  base_info.vectors = call.info_vectors;
  base_info.lc_used = call.info_lc;
  if ((call.flags & RSVD_ASYNC) && rc == RSVD_OK) {
    // enqueued only: rsvd_wait synchronises the stream and completes the info
    ctx->pending = true;
    ctx->pending_info = base_info;
    if (info) *info = base_info;
    return RSVD_OK;
  }
  {
    const int wr = wait_stream(ctx);
    if (wr != RSVD_OK) return wr;
  }
  if (rc != RSVD_OK) {
    cudaError_t le = cudaGetLastError();
    set_err(ctx, "launch failed (rc %d): %s", rc, cudaGetErrorString(le));
    return rc;
  }
  const DevStatus hs = *ctx->hstat;
  if (info) {
    const int32_t st0 = info->status;
    *info = base_info;
    info->status = st0;
    info->rank_deficient_cols = hs.deficient;
    info->jacobi_sweeps = hs.jacobi_sweeps;
    if (call.info_lc == RSVD_LC_MINVAR) info->lc_used = hs.minvar_lc;
    if (profile && !E.ev_pairs.empty()) {
      double vm = 0;
      for (size_t i = 1; i < E.ev_pairs.size(); ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ctx->events[E.ev_pairs[i].first], ctx->events[E.ev_pairs[i].second]);
        vm += ms;
      }
      float tot = 0;
      cudaEventElapsedTime(&tot, ctx->events[E.ev_pairs[0].first], ctx->events[E.ev_pairs[0].second]);
      info->view_ms = vm;
      info->total_ms = tot;
    }
  }
  if (hs.jacobi_fail) {
    set_err(ctx, "Jacobi SVD of the core did not converge");
    if (info) info->status = RSVD_E_NUMERIC;
    return RSVD_E_NUMERIC;
  }
  return RSVD_OK;
}

int check_mat(rsvd_ctx* ctx, const rsvd_mat* A) {
  if (!A || !A->data) { set_err(ctx, "A is NULL"); return RSVD_E_ARG; }
  if (A->dtype != RSVD_F64 && A->dtype != RSVD_F32) { set_err(ctx, "unknown dtype %d", A->dtype); return RSVD_E_DTYPE; }
  if (A->m < 1 || A->n < 1 || A->m_local < 0 || A->row0 < 0 || A->row0 + A->m_local > A->m) {
    set_err(ctx, "bad shape m=%lld n=%lld m_local=%lld row0=%lld", (long long)A->m, (long long)A->n,
            (long long)A->m_local, (long long)A->row0);
    return RSVD_E_ARG;
  }
  if (A->lda < A->n) { set_err(ctx, "lda < n"); return RSVD_E_ARG; }
  if (ctx->nranks == 1 && (A->m_local != A->m || A->row0 != 0)) {
    set_err(ctx, "single-GPU call needs m_local == m and row0 == 0");
    return RSVD_E_ARG;
  }
  if (A->m_local < 1) { set_err(ctx, "empty shard"); return RSVD_E_ARG; }
  return RSVD_OK;
}

int common_checks(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p) {
  if (!ctx) return RSVD_E_ARG;
  int r = check_mat(ctx, A);
  if (r) return r;
  if (k < 1 || p < 0) { set_err(ctx, "need k >= 1 and p >= 0"); return RSVD_E_ARG; }
  const int64_t l = (int64_t)k + p;
  if (l > std::min(A->m, A->n)) { set_err(ctx, "k + p = %lld exceeds min(m, n)", (long long)l); return RSVD_E_ARG; }
  if (l > 512) { set_err(ctx, "k + p > 512 is not supported"); return RSVD_E_ARG; }
  return RSVD_OK;
}

}  // namespace

// ================================================================ exported C ABI
extern "C" {

int rsvd_version(void) { return 100; }

const char* rsvd_strerror(int code) {
  switch (code) {
    case RSVD_OK: return "ok";
    case RSVD_E_ARG: return "invalid argument";
    case RSVD_E_DTYPE: return "unsupported dtype";
    case RSVD_E_CUDA: return "CUDA error";
    case RSVD_E_NCCL: return "NCCL error";
    case RSVD_E_NOMEM: return "out of device memory";
    case RSVD_E_NUMERIC: return "numerical failure";
    case RSVD_E_STATE: return "invalid state";
    default: return "unknown error";
  }
}

const char* rsvd_last_error(const rsvd_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

int rsvd_recommend_input(int goal, int v) {
  if (goal == RSVD_GOAL_RIGHT || goal == RSVD_GOAL_NORMAL) return (v % 2 == 0) ? RSVD_INPUT_A : RSVD_INPUT_AT;
  if (goal == RSVD_GOAL_LEFT) return (v % 2 == 0) ? RSVD_INPUT_AT : RSVD_INPUT_A;
  return RSVD_INPUT_A;
}

int rsvd_create(rsvd_ctx** out, int device, void* stream) {
  if (!out) return RSVD_E_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return RSVD_E_CUDA;
  }
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10) return RSVD_E_CUDA;  // sm_100a kernels only
  rsvd_ctx* c = new rsvd_ctx();
  c->device = device;
  c->sms = prop.multiProcessorCount;
  cudaSetDevice(device);
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
  } else {
    // a BLOCKING stream: it is ordered with the legacy default stream (handle 0, torch's default)
    // in both directions, so the work a caller queued there before the call (inputs produced,
    // buffers reused by a caching allocator) completes first, and later default-stream work waits
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamDefault) != cudaSuccess) {
      delete c;
      return RSVD_E_CUDA;
    }
    c->own_stream = true;
  }
  if (cudaMalloc(&c->counter, 256) != cudaSuccess || cudaMemset(c->counter, 0, 256) != cudaSuccess ||
      cudaMalloc(&c->dstat, sizeof(DevStatus)) != cudaSuccess ||
      cudaMallocHost(&c->hstat, sizeof(DevStatus)) != cudaSuccess) {
    delete c;
    return RSVD_E_NOMEM;
  }
  *out = c;
  return RSVD_OK;
}

int rsvd_destroy(rsvd_ctx* c) {
  if (!c) return RSVD_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  for (auto e : c->events) cudaEventDestroy(e);
  if (c->arena) cudaFree(c->arena);
  if (c->dstat) cudaFree(c->dstat);
  if (c->counter) cudaFree(c->counter);
  if (c->hstat) cudaFreeHost(c->hstat);
  delete c->comm;
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return RSVD_OK;
}

int rsvd_sm_count(const rsvd_ctx* c) { return c ? c->sms : 0; }

int rsvd_set_sm_limit(rsvd_ctx* c, int n) {
  if (!c || n < 1) return RSVD_E_ARG;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, c->device) != cudaSuccess) return RSVD_E_CUDA;
  c->sms = std::min(n, prop.multiProcessorCount);
  return RSVD_OK;
}

int rsvd_wait(rsvd_ctx* c, rsvd_info* info) {
  if (!c) return RSVD_E_ARG;
  if (!c->pending) return RSVD_OK;
  cudaSetDevice(c->device);
  c->pending = false;
  const int wr = wait_stream(c);
  if (wr != RSVD_OK) {
    if (info) info->status = wr;
    return wr;
  }
  const DevStatus hs = *c->hstat;
  if (info) {
    // everything known at enqueue time comes from the ctx (the caller's struct may be fresh)
    *info = c->pending_info;
    if (info->lc_used == RSVD_LC_MINVAR) info->lc_used = hs.minvar_lc;
    info->rank_deficient_cols = hs.deficient;
    info->jacobi_sweeps = hs.jacobi_sweeps;
    info->status = RSVD_OK;
  }
  if (hs.jacobi_fail) {
    set_err(c, "Jacobi SVD of the core did not converge");
    if (info) info->status = RSVD_E_NUMERIC;
    return RSVD_E_NUMERIC;
  }
  return RSVD_OK;
}

int rsvd_probe_peaks(rsvd_ctx* c, double* dmma_tflops, double* read_gbs) {
  if (!c || !dmma_tflops || !read_gbs) return RSVD_E_ARG;
  cudaSetDevice(c->device);
  return probe_peaks(c->sms, c->stream, dmma_tflops, read_gbs);
}

int rsvd_get_unique_id(void* id128) {
  if (!id128) return RSVD_E_ARG;
  return nccl_unique_id(id128);
}

static void install_comm(rsvd_ctx* c, Comm* comm) {
  c->comm = comm;
  c->nranks = comm->nranks;
  c->rank = comm->rank;
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  c->graphs.clear();
  c->graph_kernels.clear();
}

int rsvd_comm_init(rsvd_ctx* c, int nranks, int rank, const void* id128) {
  if (!c || nranks < 1 || rank < 0 || rank >= nranks || !id128) return RSVD_E_ARG;
  if (c->comm) return RSVD_E_STATE;
  // nranks == 1 also creates a (1-rank) communicator: the sharded code path then runs on one GPU
  cudaSetDevice(c->device);
  std::string e;
  Comm* comm = nccl_comm_create(nranks, rank, id128, &e);
  if (!comm) {
    set_err(c, "%s", e.c_str());
    return RSVD_E_NCCL;
  }
  install_comm(c, comm);
  return RSVD_OK;
}

struct rsvd_loop {
  LoopGroup* g;
};

int rsvd_loop_create(int nranks, double timeout_s, rsvd_loop** out) {
  if (!out) return RSVD_E_ARG;
  *out = nullptr;
  LoopGroup* g = loop_group_create(nranks, timeout_s);
  if (!g) return RSVD_E_ARG;
  *out = new rsvd_loop{g};
  return RSVD_OK;
}

int rsvd_loop_destroy(rsvd_loop* lp) {
  if (!lp) return RSVD_OK;
  loop_group_release(lp->g);
  delete lp;
  return RSVD_OK;
}

int rsvd_comm_init_loopback(rsvd_ctx* c, rsvd_loop* lp, int rank) {
  if (!c || !lp) return RSVD_E_ARG;
  if (c->comm) return RSVD_E_STATE;
  std::string e;
  Comm* comm = loop_comm_create(lp->g, rank, c->device, &e);
  if (!comm) {
    set_err(c, "%s", e.c_str());
    return RSVD_E_ARG;
  }
  install_comm(c, comm);
  return RSVD_OK;
}

int rsvd_comm_nranks(const rsvd_ctx* c) { return c ? c->nranks : 0; }

static int algo_entry(int alg, rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int v, int input, const void* Omega,
                      int64_t ld_omega, void* U, int64_t ldu, void* S, void* V, int64_t ldv, unsigned flags,
                      rsvd_info* info) {
  int r = common_checks(ctx, A, k, p);
  if (r == RSVD_OK) {
    const int l = k + p;
    if (v < 2) { set_err(ctx, "v >= 2 required (P:142, P:903); use rsvd_single_pass for v = 1"); r = RSVD_E_ARG; }
    else if (input != RSVD_INPUT_A && input != RSVD_INPUT_AT) { set_err(ctx, "bad input"); r = RSVD_E_ARG; }
    else if (!Omega) { set_err(ctx, "Omega is NULL"); r = RSVD_E_ARG; }
    else {
      const int64_t om_rows = (input == RSVD_INPUT_A) ? A->n : A->m_local;
      if (ld_omega < om_rows) { set_err(ctx, "ld_omega < rows of Omega"); r = RSVD_E_ARG; }
      if (U && ldu < A->m_local) { set_err(ctx, "ldu < m_local"); r = RSVD_E_ARG; }
      if (V && ldv < A->n) { set_err(ctx, "ldv < n"); r = RSVD_E_ARG; }
      if (alg == 1 && r == RSVD_OK) {
        const int nb = (v % 2 == 0) ? v / 2 : (v - 1) / 2;
        const int64_t W = (int64_t)nb * l;
        const int64_t side_rows_c = (input == RSVD_INPUT_A) ? A->m : A->n;
        const int64_t side_rows_r = (input == RSVD_INPUT_A) ? A->n : A->m;
        const int64_t krows = (v % 2 == 0) ? side_rows_c : side_rows_r;
        if (W > krows || W > 512) {
          set_err(ctx, "Krylov basis width %lld exceeds its side (%lld rows) or 512", (long long)W,
                  (long long)krows);
          r = RSVD_E_ARG;
        }
      }
    }
  }
  if (r != RSVD_OK) {
    if (info) { memset(info, 0, sizeof(*info)); info->status = r; }
    return r;
  }
  Call c;
  c.alg = alg;
  c.A = A;
  c.k = k;
  c.p = p;
  c.v = v;
  c.input = input;
  c.Om = Omega;
  c.ldom = ld_omega;
  c.U = U;
  c.ldu = ldu;
  c.S = S;
  c.V = V;
  c.ldv = ldv;
  c.flags = flags;
  c.info_views = v;
  c.info_vectors = (alg == 0) ? (int64_t)v * (k + p) : (int64_t)(v + v / 2 - 1) * (k + p);
  r = execute(ctx, c, info);
  if (info) info->status = r;
  return r;
}

int rsvd_subspace(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int v, int input, const void* Omega,
                  int64_t ld_omega, void* U, int64_t ldu, void* S, void* V, int64_t ldv, unsigned flags,
                  rsvd_info* info) {
  return algo_entry(0, ctx, A, k, p, v, input, Omega, ld_omega, U, ldu, S, V, ldv, flags, info);
}

int rsvd_block_krylov(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int v, int input, const void* Omega,
                      int64_t ld_omega, void* U, int64_t ldu, void* S, void* V, int64_t ldv, unsigned flags,
                      rsvd_info* info) {
  return algo_entry(1, ctx, A, k, p, v, input, Omega, ld_omega, U, ldu, S, V, ldv, flags, info);
}

int rsvd_single_pass(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int l2, int lc, const void* Omega,
                     int64_t ld_omega, const void* Phi, int64_t ld_phi, void* U, int64_t ldu, void* S, void* V,
                     int64_t ldv, unsigned flags, rsvd_info* info) {
  int r = common_checks(ctx, A, k, p);
  if (lc == -1) lc = p;
  if (r == RSVD_OK) {
    if (l2 < k + p) { set_err(ctx, "l2 >= k + p required (P:663)"); r = RSVD_E_ARG; }
    else if (l2 > std::min<int64_t>(A->m, 512)) { set_err(ctx, "l2 exceeds min(m, 512)"); r = RSVD_E_ARG; }
    else if ((lc < 0 || lc > p) && lc != RSVD_LC_MINVAR) { set_err(ctx, "lc must be in [0, p] (P:663)"); r = RSVD_E_ARG; }
    else if (lc == RSVD_LC_MINVAR && (flags & RSVD_WOOLFE)) { set_err(ctx, "MinVar l_c is defined for Alg. 7 only"); r = RSVD_E_ARG; }
    else if (!Omega || !Phi) { set_err(ctx, "Omega/Phi NULL"); r = RSVD_E_ARG; }
    else if (ld_omega < A->n || ld_phi < A->m_local) { set_err(ctx, "ld_omega/ld_phi too small"); r = RSVD_E_ARG; }
    else if ((U && ldu < A->m_local) || (V && ldv < A->n)) { set_err(ctx, "ldu/ldv too small"); r = RSVD_E_ARG; }
  }
  if (r != RSVD_OK) {
    if (info) { memset(info, 0, sizeof(*info)); info->status = r; }
    return r;
  }
  Call c;
  c.alg = 2;
  c.A = A;
  c.k = k;
  c.p = p;
  c.l2 = l2;
  c.lc = lc;
  c.Om = Omega;
  c.ldom = ld_omega;
  c.Phi = Phi;
  c.ldphi = ld_phi;
  c.U = U;
  c.ldu = ldu;
  c.S = S;
  c.V = V;
  c.ldv = ldv;
  c.flags = flags;
  c.info_views = 1;
  c.info_vectors = (int64_t)(k + p) + l2;
  c.info_lc = lc;   // MinVar: replaced by the device's choice when the call completes
  r = execute(ctx, c, info);
  if (info) info->status = r;
  return r;
}

int rsvd_single_pass_extended(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int l2, int s, const void* Omega,
                              int64_t ld_omega, const void* Phi, int64_t ld_phi, const void* Xi_r, int64_t ld_xi_r,
                              const void* Xi_c, int64_t ld_xi_c, int variant, void* U, int64_t ldu, void* S,
                              void* V, int64_t ldv, unsigned flags, rsvd_info* info) {
  int r = common_checks(ctx, A, k, p);
  if (r == RSVD_OK) {
    if (l2 < k + p) { set_err(ctx, "l2 >= k + p required (P:663)"); r = RSVD_E_ARG; }
    else if (l2 > std::min<int64_t>(A->m, 512)) { set_err(ctx, "l2 exceeds min(m, 512)"); r = RSVD_E_ARG; }
    else if (s < k + p || s > std::min<int64_t>(std::min(A->m, A->n), 512)) {
      set_err(ctx, "k + p <= s <= min(m, n, 512) required (P:805)");
      r = RSVD_E_ARG;
    } else if (variant != RSVD_EXT_BWZ && variant != RSVD_EXT_BWZ2) { set_err(ctx, "unknown variant"); r = RSVD_E_ARG; }
    else if (!Omega || !Phi || !Xi_r || !Xi_c) { set_err(ctx, "Omega/Phi/Xi_r/Xi_c NULL"); r = RSVD_E_ARG; }
    else if (ld_omega < A->n || ld_phi < A->m_local || ld_xi_r < A->m_local || ld_xi_c < A->n) {
      set_err(ctx, "ld_omega/ld_phi/ld_xi_r/ld_xi_c too small");
      r = RSVD_E_ARG;
    } else if ((U && ldu < A->m_local) || (V && ldv < A->n)) { set_err(ctx, "ldu/ldv too small"); r = RSVD_E_ARG; }
  }
  if (r != RSVD_OK) {
    if (info) { memset(info, 0, sizeof(*info)); info->status = r; }
    return r;
  }
  Call c;
  c.alg = 5;
  c.A = A;
  c.k = k;
  c.p = p;
  c.l2 = l2;
  c.s = s;
  c.variant = variant;
  c.Om = Omega;
  c.ldom = ld_omega;
  c.Phi = Phi;
  c.ldphi = ld_phi;
  c.Xr = Xi_r;
  c.ldxr = ld_xi_r;
  c.Xc = Xi_c;
  c.ldxc = ld_xi_c;
  c.U = U;
  c.ldu = ldu;
  c.S = S;
  c.V = V;
  c.ldv = ldv;
  c.flags = flags;
  c.info_views = 1;
  c.info_vectors = (int64_t)(k + p) + s + l2;   // A [Omega | Xi_c] and A^T Phi
  r = execute(ctx, c, info);
  if (info) info->status = r;
  return r;
}

int rsvd_row_stream(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, const void* Omega, int64_t ld_omega, void* U,
                    int64_t ldu, void* S, void* V, int64_t ldv, unsigned flags, rsvd_info* info) {
  int r = common_checks(ctx, A, k, p);
  if (r == RSVD_OK) {
    if (!Omega) { set_err(ctx, "Omega NULL"); r = RSVD_E_ARG; }
    else if (ld_omega < A->n) { set_err(ctx, "ld_omega too small"); r = RSVD_E_ARG; }
    else if ((U && ldu < A->m_local) || (V && ldv < A->n)) { set_err(ctx, "ldu/ldv too small"); r = RSVD_E_ARG; }
  }
  if (r != RSVD_OK) {
    if (info) { memset(info, 0, sizeof(*info)); info->status = r; }
    return r;
  }
  Call c;
  c.alg = 6;
  c.A = A;
  c.k = k;
  c.p = p;
  c.Om = Omega;
  c.ldom = ld_omega;
  c.U = U;
  c.ldu = ldu;
  c.S = S;
  c.V = V;
  c.ldv = ldv;
  c.flags = flags;
  c.info_views = 1;                                 // one pass over the rows
  c.info_vectors = 2 * (int64_t)(k + p);
  r = execute(ctx, c, info);
  if (info) info->status = r;
  return r;
}

int rsvd_block_krylov_rows(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int v, const void* Omega,
                           int64_t ld_omega, void* U, int64_t ldu, void* S, void* V, int64_t ldv, unsigned flags,
                           rsvd_info* info) {
  int r = common_checks(ctx, A, k, p);
  const int l = k + p;
  const bool even = (v % 2 == 0);
  const int nb = even ? v / 2 : (v - 1) / 2;
  if (r == RSVD_OK) {
    if (v < 2) { set_err(ctx, "v >= 2 required (P:903)"); r = RSVD_E_ARG; }
    else if (!Omega || ld_omega < A->n) { set_err(ctx, "Omega NULL or ld_omega < n"); r = RSVD_E_ARG; }
    else if ((U && ldu < A->m_local) || (V && ldv < A->n)) { set_err(ctx, "ldu/ldv too small"); r = RSVD_E_ARG; }
    else if ((int64_t)nb * l > (even ? A->m : A->n) || (int64_t)nb * l > 512) {
      set_err(ctx, "Krylov basis width %lld exceeds its side or 512", (long long)nb * l);
      r = RSVD_E_ARG;
    }
  }
  if (r != RSVD_OK) {
    if (info) { memset(info, 0, sizeof(*info)); info->status = r; }
    return r;
  }
  Call c;
  c.alg = 7;
  c.A = A;
  c.k = k;
  c.p = p;
  c.v = v;
  c.Om = Omega;
  c.ldom = ld_omega;
  c.U = U;
  c.ldu = ldu;
  c.S = S;
  c.V = V;
  c.ldv = ldv;
  c.flags = flags;
  // reads of A: (v-1)/2 row passes + 1 (odd v), v/2 + 1 (even v); vectors: 2l per row pass
  c.info_views = even ? nb + 1 : nb + 1;
  c.info_vectors = even ? (int64_t)(nb - 1) * 2 * l + l + (int64_t)nb * l : (int64_t)nb * 2 * l + (int64_t)nb * l;
  r = execute(ctx, c, info);
  if (info) info->status = r;
  return r;
}

int rsvd_plan(int scheme, int k, int T, double alpha, int* p, int* l2, int* lc) {
  if (!p || !l2 || !lc || k < 1 || T < 2 * k + 6 || !(alpha >= 0.0 && alpha <= 1.0)) return RSVD_E_ARG;
  int l1;
  int cut = -1;
  switch (scheme) {
    case RSVD_PLAN_FLAT: {
      const double num = std::sqrt((double)k * (T - k - 2) * (1.0 - 2.0 / (T - 1))) - (k - 1);
      l1 = std::max(2, (int)std::floor((T - 1) * num / (T - 2 * k - 1)) - k);
      break;
    }
    case RSVD_PLAN_DECAY: l1 = std::max(2, (T - 1) / 3 - k); break;
    case RSVD_PLAN_RAPID: l1 = (T - 2) / 2 - k; break;
    case RSVD_PLAN_BALANCED:
      l1 = T / 2 - k;
      cut = (int)std::floor(alpha * l1);
      break;
    default: return RSVD_E_ARG;
  }
  *p = l1;
  *l2 = k + (T - 2 * k - l1);
  *lc = cut >= 0 ? cut : l1;
  return RSVD_OK;
}

static int normal_entry(int alg, rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int v, const void* Omega,
                        int64_t ld_omega, void* S, void* V, int64_t ldv, unsigned flags, rsvd_info* info) {
  int r = common_checks(ctx, A, k, p);
  if (r == RSVD_OK) {
    // Omega lives on the side the first basis is built from: Alg. 4 starts from A for even v
    // and from A^T for odd v; Alg. 5 the other way round
    const bool om_m = (alg == 3) ? (v % 2 == 1) : (v % 2 == 0);
    const int64_t om_rows = om_m ? A->m_local : A->n;
    if (v < 2) { set_err(ctx, "v >= 2 required (Alg. 4 / Alg. 5)"); r = RSVD_E_ARG; }
    else if (!Omega || ld_omega < om_rows) { set_err(ctx, "Omega NULL or ld_omega < %lld", (long long)om_rows); r = RSVD_E_ARG; }
    else if (V && ldv < A->n) { set_err(ctx, "ldv < n"); r = RSVD_E_ARG; }
  }
  if (r != RSVD_OK) {
    if (info) { memset(info, 0, sizeof(*info)); info->status = r; }
    return r;
  }
  Call c;
  c.alg = alg;
  c.A = A;
  c.k = k;
  c.p = p;
  c.v = v;
  c.Om = Omega;
  c.ldom = ld_omega;
  c.S = S;
  c.V = V;
  c.ldv = ldv;
  c.flags = flags;
  c.info_views = v;
  c.info_vectors = (int64_t)v * (k + p);
  r = execute(ctx, c, info);
  if (info) info->status = r;
  return r;
}

int rsvd_nystrom(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int v, const void* Omega, int64_t ld_omega, void* S,
                 void* V, int64_t ldv, unsigned flags, rsvd_info* info) {
  return normal_entry(3, ctx, A, k, p, v, Omega, ld_omega, S, V, ldv, flags, info);
}

int rsvd_pinched(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int v, const void* Omega, int64_t ld_omega, void* S,
                 void* V, int64_t ldv, unsigned flags, rsvd_info* info) {
  return normal_entry(4, ctx, A, k, p, v, Omega, ld_omega, S, V, ldv, flags, info);
}

int rsvd_view(rsvd_ctx* ctx, const rsvd_mat* A, int trans, const void* X, int64_t ldx, int w, void* Y, int64_t ldy,
              unsigned flags, rsvd_info* info) {
  if (!ctx) return RSVD_E_ARG;
  int r = check_mat(ctx, A);
  if (r == RSVD_OK) {
    const int64_t xr = trans ? A->m_local : A->n, yr = trans ? A->n : A->m_local;
    if (w < 1 || w > 1024 || !X || !Y || ldx < xr || ldy < yr) { set_err(ctx, "bad view arguments"); r = RSVD_E_ARG; }
  }
  if (r) return r;
  Call c;
  c.alg = 10;
  c.A = A;
  c.trans = trans ? 1 : 0;
  c.w = w;
  c.Om = X;
  c.ldom = ldx;
  c.U = Y;
  c.ldu = ldy;
  c.flags = flags;
  return execute(ctx, c, info);
}

int rsvd_view_fused(rsvd_ctx* ctx, const rsvd_mat* A, const void* Omega, int64_t ld_omega, int l, const void* Phi,
                    int64_t ld_phi, int l2, void* Yc, int64_t ld_yc, void* Yr, int64_t ld_yr, unsigned flags,
                    rsvd_info* info) {
  if (!ctx) return RSVD_E_ARG;
  int r = check_mat(ctx, A);
  if (r == RSVD_OK) {
    const bool narrow = l >= 1 && l <= kFusedMaxL && l2 >= 1 && (l2 + 7) / 8 <= kFusedMaxL2T;
    const bool wide = A->dtype == RSVD_F64 && fused_cl_supported(l, l2);
    if (!(narrow || wide) || !Omega || !Phi || !Yc || !Yr ||
        ld_omega < A->n || ld_phi < A->m_local || ld_yc < A->m_local || ld_yr < A->n) {
      set_err(ctx, "bad fused-view arguments (fp64: l <= 128, l2 <= 256)");
      r = RSVD_E_ARG;
    }
  }
  if (r) return r;
  Call c;
  c.alg = 11;
  c.A = A;
  c.w = l;
  c.l2 = l2;
  c.Om = Omega;
  c.ldom = ld_omega;
  c.Phi = Phi;
  c.ldphi = ld_phi;
  c.U = Yc;
  c.ldu = ld_yc;
  c.V = Yr;
  c.ldv = ld_yr;
  c.flags = flags;
  return execute(ctx, c, info);
}

int rsvd_orth(rsvd_ctx* ctx, int64_t rows, int w, void* Y, int64_t ldy, void* R, unsigned flags, rsvd_info* info) {
  if (!ctx) return RSVD_E_ARG;
  if (rows < 1 || w < 1 || w > 512 || w > rows || !Y || ldy < rows) {
    set_err(ctx, "bad orth arguments (1 <= w <= min(rows, 512))");
    return RSVD_E_ARG;
  }
  Call c;
  c.alg = 12;
  c.rows = rows;
  c.w = w;
  c.U = Y;
  c.ldu = ldy;
  c.R = R;
  c.flags = flags;
  return execute(ctx, c, info);
}

int rsvd_core_svd(rsvd_ctx* ctx, int r, int cc, const void* M, int64_t ldm, void* U, void* S, void* V,
                  unsigned flags, rsvd_info* info) {
  if (!ctx) return RSVD_E_ARG;
  if (cc < 1 || r < cc || r > 512 || !M || ldm < r) {
    set_err(ctx, "bad core-svd arguments (1 <= c <= r <= 512)");
    return RSVD_E_ARG;
  }
  Call c;
  c.alg = 13;
  c.rows = r;
  c.cols = cc;
  c.Om = M;
  c.ldom = ldm;
  c.U = U;
  c.S = S;
  c.V = V;
  c.flags = flags;
  return execute(ctx, c, info);
}

}  // extern "C"
