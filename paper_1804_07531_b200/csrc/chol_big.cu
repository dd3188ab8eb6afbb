// Guarded Cholesky G = R^T R and the triangular inverse R^-1 for Gram matrices too wide for
// shared memory (160 < w <= 512; C5's l = 250 sketches and w = 500 Krylov bases).  This is
// the "chol" step of CholeskyQR2, the qr of PAPER.md P:69 used at P:149/151 (Alg. 2) and
// P:917/922 (Alg. 9).  Semantics match k_chol (small_kernels.cu) exactly: a pivot d_j <=
// tol * ref_j marks column j rank deficient -> row j of R and column j of R^-1 are zero.
//
// One CTA, right-looking blocked factorisation with 32-wide panels, working in place in the
// caller's R buffer (L2 resident: 2 MB at w = 512):
//   diag block: unblocked guarded factorisation by one warp in shared memory
//   panel:      R12 = R11^-T G12 (one thread per trailing column)
//   update:     G22 -= R12^T R12 on the upper triangle (4x4 register tiles)
// then R^-1 by blocked back substitution, bottom block row first.
#include <atomic>
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

namespace rsvd {
namespace cg = cooperative_groups;
namespace {

constexpr int kNB = 32;
constexpr int kMaxW = 512;
constexpr int kThr = 256;      // up to 255 registers per thread (32-entry column solves in registers)

// unblocked guarded factorisation of the jb x jb diagonal block D (smem, col-major ld 33),
// executed by warp 0; writes defi[] for the block's columns and dinv[] = 1 / R_pp (0 for a
// deficient pivot).  Per pivot one reciprocal (shared by every lane); the trailing update of
// column `lane` reads row p of R once (broadcast loads, issued together) before it writes.
__device__ void factor_diag(double* D, int jb, const double* gdiag, bool has_ref, int j0, double tol,
                            double shift, int* defi, double* dinv) {
  const int lane = threadIdx.x & 31;
  for (int p = 0; p < jb; ++p) {
    const double d = D[p * 33 + p];
    const double rf = has_ref ? gdiag[j0 + p] : (gdiag[j0 + p] + shift);
    const bool def = !(d > tol * rf) || !(rf > 0.0);
    const double rjj = def ? 0.0 : sqrt(d);
    const double inv = def ? 0.0 : 1.0 / rjj;
    __syncwarp();
    double rpc = 0.0;
    if (lane > p && lane < jb) {
      rpc = D[lane * 33 + p] * inv;
      D[lane * 33 + p] = rpc;
    }
    if (lane == 0) {
      D[p * 33 + p] = rjj;
      defi[j0 + p] = def ? 1 : 0;
      dinv[p] = inv;
    }
    __syncwarp();
    // trailing in-block update of column `lane`: D(i, lane) -= R(p, i) R(p, lane), p < i <= lane
    if (!def && lane > p && lane < jb) {
      double v[kNB];
#pragma unroll
      for (int i = 0; i < kNB; ++i) v[i] = (i > p && i <= lane) ? D[i * 33 + p] : 0.0;
#pragma unroll
      for (int i = 0; i < kNB; ++i)
        if (i > p && i <= lane) D[lane * 33 + i] = fma(-v[i], rpc, D[lane * 33 + i]);
    }
    __syncwarp();
  }
}

// upper-triangular inverse of the jb x jb block D (rows of deficient pivots -> 0), warp 0,
// result in X (smem col-major ld 33).  Column `lane` of X is held in registers (compile-time
// indices) and solved from the bottom; 1 / D_ii comes from dinv (0 for a deficient pivot).
__device__ void invert_diag(const double* D, int jb, const int* defi, int j0, const double* dinv, double* X) {
  const int lane = threadIdx.x & 31;
  double x[kNB];
#pragma unroll
  for (int i = kNB - 1; i >= 0; --i) {
    double v = 0.0;
    if (i < jb && lane < jb && lane >= i && !defi[j0 + i]) {
      if (lane == i) {
        v = dinv[i];
      } else {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int k = i + 1; k < kNB; k += 2) {
          if (k <= lane) s0 = fma(D[k * 33 + i], x[k], s0);
          if (k + 1 < kNB && k + 1 <= lane) s1 = fma(D[(k + 1) * 33 + i], x[k + 1], s1);
        }
        v = -(s0 + s1) * dinv[i];
      }
    }
    x[i] = (i < jb && lane >= i) ? v : 0.0;
  }
  if (lane < jb)
#pragma unroll
    for (int i = 0; i < kNB; ++i)
      if (i < jb) X[lane * 33 + i] = x[i];
  __syncwarp();
}

__global__ void __launch_bounds__(kThr, 1) k_chol_big(const double* __restrict__ G, const double* __restrict__ ref,
                                                      int w, double tol, double shift_coef, double* __restrict__ R,
                                                      double* __restrict__ Rinv, DevStatus* status) {
  extern __shared__ double sm[];
  double* P = sm;                       // kNB x kMaxW panel (row k of the panel at P[k * kMaxW])
  double* D = P + kNB * kMaxW;          // 32 x 33
  double* Xd = D + kNB * 33;            // 32 x 33
  double* gdiag = Xd + kNB * 33;        // w (diagonal of G, the default rank-guard reference)
  int* defi = reinterpret_cast<int*>(gdiag + kMaxW);
  __shared__ double s_dinv[kMaxW];      // 1 / R_jj (0 for a deficient pivot)
  __shared__ double s_shift;
  __shared__ int s_fast;
  const int tid = threadIdx.x;
  if (ref == nullptr && shift_coef == 0.0 && chol_near_identity(G, w, R, Rinv, status, &s_fast)) return;
  // working copy: upper triangle of G (+ shift on the diagonal), zero below
  if (tid == 0) {
    double tr = 0.0;
    for (int j = 0; j < w; ++j) tr += G[(int64_t)j * w + j];
    s_shift = shift_coef > 0.0 ? shift_coef * tr : 0.0;
  }
  __syncthreads();
  const double shift = s_shift;
  for (int e = tid; e < w * w; e += kThr) {
    const int i = e % w, c = e / w;
    double v = (i <= c) ? G[e] : 0.0;
    if (i == c) v += shift;
    R[e] = v;
  }
  // guard references in shared memory (ref, else diag(G)): no global load on the pivot chain
  for (int j = tid; j < w; j += kThr) gdiag[j] = ref ? ref[j] : G[(int64_t)j * w + j];
  __syncthreads();

  for (int j0 = 0; j0 < w; j0 += kNB) {
    const int jb = min(kNB, w - j0);
    const int t0 = j0 + jb, T = w - t0;
    for (int e = tid; e < jb * jb; e += kThr) {
      const int i = e % jb, c = e / jb;
      D[c * 33 + i] = (i <= c) ? R[(int64_t)(j0 + c) * w + j0 + i] : 0.0;
    }
    __syncthreads();
    if (tid < 32) factor_diag(D, jb, gdiag, ref != nullptr, j0, tol, shift, defi, s_dinv + j0);
    __syncthreads();
    for (int e = tid; e < jb * jb; e += kThr) {
      const int i = e % jb, c = e / jb;
      R[(int64_t)(j0 + c) * w + j0 + i] = (i <= c) ? D[c * 33 + i] : 0.0;
    }
    // panel: for trailing column c solve R11^T y = x (forward substitution, column oriented:
    // y_p = y_p / R_pp, then y_k -= R(p, k) y_p for every k > p — independent updates, so the
    // dependent chain is one multiply and one FMA per pivot), y -> P and R
    for (int cc0 = tid; cc0 < T; cc0 += kThr) {
      const int c = t0 + cc0;
      double y[kNB];
#pragma unroll
      for (int k = 0; k < kNB; ++k) y[k] = (k < jb) ? R[(int64_t)c * w + j0 + k] : 0.0;
#pragma unroll
      for (int p = 0; p < kNB; ++p) {
        if (p < jb) {
          const double yp = y[p] * s_dinv[j0 + p];   // 0 for a deficient pivot
          y[p] = yp;
#pragma unroll
          for (int k = p + 1; k < kNB; ++k)
            if (k < jb) y[k] = fma(-D[k * 33 + p], yp, y[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < kNB; ++k)
        if (k < jb) {
          R[(int64_t)c * w + j0 + k] = y[k];
          P[k * kMaxW + cc0] = y[k];
        }
    }
    __syncthreads();
    // trailing update of the upper triangle: R(i, c) -= sum_k P(k, i) P(k, c), t0 <= i <= c
    if (T > 0) {
      const int nt4 = (T + 3) / 4;
      const int ntiles = nt4 * (nt4 + 1) / 2;
      for (int tt = tid; tt < ntiles; tt += kThr) {
        // tile (ti, tc) with ti <= tc, enumerated column by column
        int tc = (int)((sqrt(8.0 * tt + 1.0) - 1.0) * 0.5);
        while ((tc + 1) * (tc + 2) / 2 <= tt) ++tc;
        while (tc * (tc + 1) / 2 > tt) --tc;
        const int ti = tt - tc * (tc + 1) / 2;
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
        for (int k = 0; k < jb; ++k) {
          double pi[4], pc[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            pi[a] = P[k * kMaxW + ti * 4 + a];
            pc[a] = P[k * kMaxW + tc * 4 + a];
          }
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(pi[a], pc[b], acc[a][b]);
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int c = tc * 4 + b;
          if (c >= T) continue;
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int i = ti * 4 + a;
            if (i <= c) R[(int64_t)(t0 + c) * w + t0 + i] -= acc[a][b];
          }
        }
      }
    }
    __syncthreads();
  }

  // ---- R^-1 by blocked back substitution (X = Rinv, col-major w x w)
  for (int e = tid; e < w * w; e += kThr) Rinv[e] = 0.0;
  __syncthreads();
  const int nblk = (w + kNB - 1) / kNB;
  for (int bi = nblk - 1; bi >= 0; --bi) {
    const int i0 = bi * kNB, ib = min(kNB, w - i0), t0 = i0 + ib, T = w - t0;
    for (int e = tid; e < ib * ib; e += kThr) {
      const int i = e % ib, c = e / ib;
      D[c * 33 + i] = R[(int64_t)(i0 + c) * w + i0 + i];
    }
    // rows i0..i0+ib of R to the right of the block -> P
    for (int e = tid; e < ib * T; e += kThr) {
      const int k = e % ib, cc = e / ib;
      P[k * kMaxW + cc] = R[(int64_t)(t0 + cc) * w + i0 + k];
    }
    __syncthreads();
    if (tid < 32) invert_diag(D, ib, defi, i0, s_dinv + i0, Xd);
    __syncthreads();
    // X(i0.., j) = -Dinv * sum_{k = t0..j} R(i0.., k) X(k, j)   for j >= t0
    for (int jj = tid; jj < T; jj += kThr) {
      const int j = t0 + jj;
      double acc[kNB];
#pragma unroll
      for (int r = 0; r < kNB; ++r) acc[r] = 0.0;
      // the already-computed rows of column j of R^-1 (L2): 4 loads in flight per batch
      const double* xj = Rinv + (int64_t)j * w;
      int k = t0;
      for (; k + 4 <= j + 1; k += 4) {
        double xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = xj[k + u];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int r = 0; r < kNB; ++r) acc[r] = fma(P[r * kMaxW + (k + u - t0)], xv[u], acc[r]);
      }
      for (; k <= j; ++k) {
        const double x = xj[k];
#pragma unroll
        for (int r = 0; r < kNB; ++r) acc[r] = fma(P[r * kMaxW + (k - t0)], x, acc[r]);
      }
#pragma unroll
      for (int r = 0; r < kNB; ++r) {
        if (r < ib) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < kNB; ++q)
            if (q < ib) s = fma(Xd[q * 33 + r], acc[q], s);
          Rinv[(int64_t)j * w + i0 + r] = -s;
        }
      }
    }
    for (int e = tid; e < ib * ib; e += kThr) {
      const int i = e % ib, c = e / ib;
      Rinv[(int64_t)(i0 + c) * w + i0 + i] = Xd[c * 33 + i];
    }
    __syncthreads();
  }
  if (tid == 0 && status) {
    int cnt = 0;
    for (int j = 0; j < w; ++j) cnt += defi[j];
    if (cnt) atomicAdd(&status->deficient, cnt);
  }
}


// ================================================================ cluster version (64 < w <= 512)
// The same factorisation and inverse on a thread-block cluster of nb = ceil(w / 32) CTAs: CTA j
// owns the 32-column panel j (rows 0 .. 32 j + 31 of the upper triangle) in shared memory and all
// block products run on the FP64 tensor cores (DMMA m8n8k4).  Right-looking, per block step k:
//   CTA k:      guarded factorisation + inverse of its (fully updated) diagonal block, one warp,
//               register resident (R_kk, X_k = R_kk^-1 -> R and Rinv in global memory)
//   barrier;    CTA j > k:  R_kj = X_k^T G_kj   (-> R in global memory)
//   barrier;    CTA j > k:  G_ij -= R_ki^T R_kj for k < i <= j   (the next diagonal block first)
// Operands of other panels are read from the final R / Rinv in global memory (L2: ~5x the
// per-SM bandwidth of distributed shared memory); the cluster barriers order them.  Then every
// CTA forms its column panel of X = R^-1 on its own, right-looking from the diagonal block up,
// in place over its panel: S_ij = R_ij X_jj, then for k = j-1 .. 0: X_kj = -X_k S_kj and
// S_ij += R_ik X_kj (i < k).  Guard, deficient columns and the near-identity closed form as
// k_chol_big / k_chol: a pivot <= tol * ref zeroes row j of R and row and column j of R^-1.
constexpr int kClThr = 256;
#ifndef CHOL_PAIRS
#define CHOL_PAIRS 1
#endif
constexpr unsigned kFull = 0xffffffffu;

#ifdef RSVD_CHOL_TIMING
__device__ unsigned long long chol_ph[16 * 8];   // cycles per (cluster rank, phase), thread 0
#define CH_T0() long long ch_t0 = clock64()
#define CH_T(i)                                          \
  if (tid == 0) {                                        \
    const long long ch_t = clock64();                    \
    chol_ph[j * 8 + (i)] += ch_t - ch_t0;                \
    ch_t0 = ch_t;                                        \
  }
#else
#define CH_T0()
#define CH_T(i)
#endif

__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Guarded Cholesky and inverse of the jb x jb diagonal block by one warp, in registers: lane c
// holds column c.  In: D (col-major ld 33, upper triangle).  Out: D = R (upper, zero below),
// X = R^-1 (ld 33), defi[p].  Pivot p: d = D(p,p) after the previous updates; deficient when
// d <= tol * ref_p (ref_p = gd[p], + shift without a caller reference): R's row p and R^-1's row
// and column p are zero.  Row p of R = D(p, :) / sqrt(d) (rsqrt, as k_chol).

__device__ void factor_inv_warp(double* D, int jb, const double* gd, bool has_ref, double tol, double shift,
                                int* defi, double* X, double* sb, double* dinv) {
  // lane c keeps column c in registers; the pivot and row p of R are broadcast through shared
  // memory (sb: two 33-entry rows, alternating), not shuffles: shuffles in this (potentially
  // divergent) code get a WARPSYNC / BRA.DIV guard each and serialise at full latency
  const int lane = threadIdx.x & 31;
  double a[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = (i <= lane && lane < jb) ? D[lane * 33 + i] : 0.0;
  unsigned defm = 0;
#pragma unroll
  for (int p = 0; p < 32; ++p) {
    double* row = sb + (p & 1) * 33;
    if (lane == p) row[32] = a[p];
    __syncwarp();
    const double d = row[32];
    const double rf = has_ref ? gd[p] : gd[p] + shift;
    const bool def = !(d > tol * rf) || !(rf > 0.0) || p >= jb;
    const double inv = def ? 0.0 : rsqrt_nr(d);
    // row p of R (0 when deficient).  Lanes < p compute (and later discard) values from their
    // below-diagonal entries: every entry stays finite, the lower triangle is zeroed on output
    const double r = (lane == p) ? d * inv : a[p] * inv;
    a[p] = r;
    if (lane == p) dinv[p] = inv;
    defm |= (def ? 1u : 0u) << p;
    row[lane] = r;
    __syncwarp();
    // trailing update of column lane: a[i] -= R(p, i) R(p, lane), i > p (rows below the diagonal
    // of column lane are updated too, unmasked, and never used)
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i > p) a[i] = fma(-row[i], r, a[i]);
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) D[lane * 33 + i] = (i <= lane) ? a[i] : 0.0;
  __syncwarp();
  // X = R^-1, column lane, back substitution: x_i = (delta_i,lane - sum_{k>i} R(i,k) x_k) / R_ii,
  // R(i, k) = D[k * 33 + i] (a broadcast load)
  double x[32];
#pragma unroll
  for (int i = 31; i >= 0; --i) {
    double s0 = (i == lane) ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
      if (k > i) s0 = fma(-D[k * 33 + i], x[k], s0);
      if (k + 1 > i) s1 = fma(-D[(k + 1) * 33 + i], x[k + 1], s1);
      if (k + 2 > i) s2 = fma(-D[(k + 2) * 33 + i], x[k + 2], s2);
      if (k + 3 > i) s3 = fma(-D[(k + 3) * 33 + i], x[k + 3], s3);
    }
    x[i] = ((s0 + s1) + (s2 + s3)) * dinv[i];   // = 0 for i > lane (delta and x_k, k > i, are 0)
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) X[lane * 33 + i] = x[i];
  defi[lane] = (lane < jb) ? (int)((defm >> lane) & 1u) : 0;
  __syncwarp();
}

// acc[b][n] += A_b (rows ti*8 .. +8, depth 32) * B (depth 32, cols (tn0 + n) * 8 .. +8) for NB
// blocks b sharing B; fa(b, q) = A_b(ti*8 + g, q), fb(n, q) = B(q, (tn0 + n)*8 + g).  Every load
// of the group is issued before the first DMMA.
template <int NB, class FA, class FB>
__device__ __forceinline__ void blk_mma(double (&acc)[NB][2][2], int t, FA fa, FB fb) {
  double a[NB][8], b0[8], b1[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
#pragma unroll
    for (int b = 0; b < NB; ++b) a[b][s] = fa(b, s * 4 + t);
    b0[s] = fb(0, s * 4 + t);
    b1[s] = fb(1, s * 4 + t);
  }
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      dmma(acc[b][0][0], acc[b][0][1], a[b][s], b0[s]);
      dmma(acc[b][1][0], acc[b][1][1], a[b][s], b1[s]);
    }
}

__global__ void __launch_bounds__(kClThr, 1) k_chol_cl(const double* __restrict__ G, const double* __restrict__ ref,
                                                        int w, double tol, double shift_coef, double* R, double* Rinv,
                                                        DevStatus* status) {
  cg::cluster_group cluster = cg::this_cluster();
  const int nb = (int)cluster.num_blocks();
  const int j = (int)cluster.block_rank();      // this CTA's column panel
  const int LP = 32 * nb + 4;                   // panel column stride (fragment loads conflict free)
  extern __shared__ __align__(16) double sm[];
  double* Pn = sm;                              // panel: column c (local) at Pn[c * LP], rows 0 .. c0 + 31
  double* D = Pn + 32 * LP;                     // 32 x 33 diagonal block
  double* Xd = D + 32 * 33;                     // 32 x 33: X_j = R_jj^-1
  double* gall = Xd + 32 * 33;                  // diag(G) (the near-identity test), kMaxW
  __shared__ double s_gd[32], s_shift, s_sb[66], s_dinv[32];
  __shared__ int s_defi[32], s_fast;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3, ti = warp >> 1, tn0 = 2 * (warp & 1);
  const int c0 = 32 * j, jb = min(32, w - c0), rows = c0 + 32;
  CH_T0();

  // ---- panel load: rows 0 .. min(rows, w) of the own columns, asynchronously (all in flight)
  {
    const int rv = min(rows, w);
    for (int e = tid; e < 32 * rv; e += kClThr) {
      const int c = e / rv, i = e - c * rv;
      if (c < jb) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(Pn + c * LP + i)),
                     "l"(G + (int64_t)(c0 + c) * w + i) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const bool try_fast = (ref == nullptr && shift_coef == 0.0);
  if (try_fast)
    for (int i = tid; i < w; i += kClThr) gall[i] = G[(int64_t)i * w + i];
  if (tid < 32) {
    s_gd[tid] = tid < jb ? (ref ? ref[c0 + tid] : G[(int64_t)(c0 + tid) * w + c0 + tid]) : 0.0;
    s_defi[tid] = 0;
  }
  if (warp == 0) {
    double tr = 0.0;
    if (shift_coef > 0.0)
      for (int i = lane; i < w; i += 32) tr += G[(int64_t)i * w + i];
    tr = warp_sum(tr);
    if (lane == 0) {
      s_shift = shift_coef > 0.0 ? shift_coef * tr : 0.0;
      s_fast = 1;
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const double shift = s_shift;
  // zero below the diagonal and beyond w, add the shift; the near-identity test on the own columns
  // (upper triangle: G is symmetric to rounding and only its upper triangle is used)
  for (int c = warp; c < 32; c += kClThr / 32) {
    const int gc = c0 + c;
    for (int i = lane; i < rows; i += 32) {
      double v = Pn[c * LP + i];
      if (c >= jb || i >= w || i > gc) v = 0.0;
      else if (i == gc) v += shift;
      Pn[c * LP + i] = v;
      if (try_fast && c < jb && i <= gc && gall[i] != 0.0 && gall[gc] != 0.0) {
        const double E = v - (i == gc ? 1.0 : 0.0);
        if (!(fabs(E) <= 1e-8)) s_fast = 0;
      }
    }
  }
  if (try_fast) {
    cluster.sync();
    int all = 1;
    for (int q = 0; q < nb; ++q) all &= *cluster.map_shared_rank(&s_fast, q);
    cluster.sync();
    if (all) {   // CholeskyQR's second pass: R = I + triu(E, 1) + diag(E) / 2, R^-1 = I - triu(E, 1) - diag(E) / 2
      int ndef = 0;
      for (int e = tid; e < w * jb; e += kClThr) {
        const int c = e / w, i = e - c * w, gc = c0 + c;
        const bool dz = i >= w || gall[i] == 0.0 || gall[gc] == 0.0;
        double r = 0.0, ri = 0.0;
        if (!dz && i <= gc) {
          const double E = Pn[c * LP + i] - (i == gc ? 1.0 : 0.0);
          r = (i == gc) ? 1.0 + 0.5 * E : E;
          ri = (i == gc) ? 1.0 - 0.5 * E : -E;
        }
        R[(int64_t)gc * w + i] = r;
        Rinv[(int64_t)gc * w + i] = ri;
        if (i == gc && gall[gc] == 0.0) ++ndef;
      }
      if (status && ndef) atomicAdd(&status->deficient, ndef);
      return;
    }
  }
  __syncthreads();
  CH_T(0);

  // ---- right-looking blocked factorisation
  for (int k = 0; k < nb; ++k) {
    if (j == k) {
      __syncthreads();   // the previous step's update of this block (all warps) is complete
      for (int e = tid; e < 32 * 32; e += kClThr) {
        const int c = e >> 5, r = e & 31;
        D[c * 33 + r] = Pn[c * LP + c0 + r];
      }
      __syncthreads();
      if (warp == 0) factor_inv_warp(D, jb, s_gd, ref != nullptr, tol, shift, s_defi, Xd, s_sb, s_dinv);
      __syncthreads();
      for (int e = tid; e < 32 * 32; e += kClThr) {
        const int c = e >> 5, r = e & 31;
        const double v = D[c * 33 + r];
        Pn[c * LP + c0 + r] = v;
        if (c < jb && c0 + r < w) {
          R[(int64_t)(c0 + c) * w + c0 + r] = v;
          Rinv[(int64_t)(c0 + c) * w + c0 + r] = Xd[c * 33 + r];
        }
      }
      CH_T(1);
    }
    cl_sync();   // R_kk, X_k in global memory
    CH_T(2);
    if (j > k) {
      // R_kj = X_k^T G_kj (rows 32 k of this panel, in place); X_k(q, r) = Rinv(32k + q, 32k + r)
      const double* Xk = Rinv + (int64_t)(32 * k) * w + 32 * k;
      const double* Bk = Pn + 32 * k;
      double acc[1][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}};
      blk_mma<1>(acc, t, [&](int, int q) { return __ldcg(Xk + (int64_t)(ti * 8 + g) * w + q); },
                 [&](int n, int q) { return Bk[((tn0 + n) * 8 + g) * LP + q]; });
      __syncthreads();
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = (tn0 + n) * 8 + 2 * t + h, r = 32 * k + ti * 8 + g;
          Pn[c * LP + r] = acc[0][n][h];
          if (c < jb) R[(int64_t)(c0 + c) * w + r] = acc[0][n][h];
        }
      CH_T(3);
    }
    cl_sync();   // row panel k of R complete (global memory)
    CH_T(4);
    if (j > k) {
      // G_ij -= R_ki^T R_kj, k < i <= j: R_ki^T(r, q) = R(32k + q, 32i + r); two blocks per group
      const double* Bk = Pn + 32 * k;
      auto fb = [&](int n, int q) { return Bk[((tn0 + n) * 8 + g) * LP + q]; };
      int i = k + 1;
      for (; CHOL_PAIRS && i + 1 < j; i += 2) {
        double acc[2][2][2] = {};
        blk_mma<2>(acc, t, [&](int b, int q) {
          return __ldcg(R + (int64_t)(32 * (i + b) + ti * 8 + g) * w + 32 * k + q); }, fb);
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int n = 0; n < 2; ++n) {
            const int c = (tn0 + n) * 8 + 2 * t;
            Pn[c * LP + 32 * (i + b) + ti * 8 + g] -= acc[b][n][0];
            Pn[(c + 1) * LP + 32 * (i + b) + ti * 8 + g] -= acc[b][n][1];
          }
      }
      for (; i <= j; ++i) {
        double acc[1][2][2] = {};
        if (i == j)
          blk_mma<1>(acc, t, [&](int, int q) { return Pn[(ti * 8 + g) * LP + 32 * k + q]; }, fb);
        else
          blk_mma<1>(acc, t, [&](int, int q) {
            return __ldcg(R + (int64_t)(32 * i + ti * 8 + g) * w + 32 * k + q); }, fb);
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          const int c = (tn0 + n) * 8 + 2 * t;
          Pn[c * LP + 32 * i + ti * 8 + g] -= acc[0][n][0];
          Pn[(c + 1) * LP + 32 * i + ti * 8 + g] -= acc[0][n][1];
        }
      }
      CH_T(5);
    }
  }
  // ---- R below the panel's diagonal block, and Rinv there, are zero
  for (int c = warp; c < jb; c += kClThr / 32) {
    const int gc = c0 + c;
    for (int i = rows + lane; i < w; i += 32) {
      R[(int64_t)gc * w + i] = 0.0;
      Rinv[(int64_t)gc * w + i] = 0.0;
    }
  }
  // ---- X = R^-1, column panel j, in place over the panel (own work only; other panels' R and
  // X_k come from global memory, final since the last barrier)
  __syncthreads();
  for (int e = tid; e < 32 * 32; e += kClThr) {
    const int c = e >> 5, r = e & 31;
    Pn[c * LP + c0 + r] = Xd[c * 33 + r];         // X_jj
  }
  __syncthreads();
  {
    // S_ij = R_ij X_jj, i < j (R_ij: the panel's own rows 32 i)
    auto fx = [&](int n, int q) { return Pn[((tn0 + n) * 8 + g) * LP + c0 + q]; };
    for (int i = 0; i < j; ++i) {
      double acc[1][2][2] = {};
      blk_mma<1>(acc, t, [&](int, int q) { return __ldcg(R + (int64_t)(c0 + q) * w + 32 * i + ti * 8 + g); }, fx);
      __syncthreads();   // (reads of block i's R rows by other warps are only through global memory)
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        const int c = (tn0 + n) * 8 + 2 * t;
        Pn[c * LP + 32 * i + ti * 8 + g] = acc[0][n][0];
        Pn[(c + 1) * LP + 32 * i + ti * 8 + g] = acc[0][n][1];
      }
    }
    __syncthreads();
    for (int k = j - 1; k >= 0; --k) {
      // X_kj = -X_k S_kj; X_k(r, q) = Rinv(32k + r, 32k + q)
      const double* Xk = Rinv + (int64_t)(32 * k) * w + 32 * k;
      auto fs = [&](int n, int q) { return Pn[((tn0 + n) * 8 + g) * LP + 32 * k + q]; };
      double acc[1][2][2] = {};
      blk_mma<1>(acc, t, [&](int, int q) { return __ldcg(Xk + (int64_t)q * w + ti * 8 + g); }, fs);
      __syncthreads();
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        const int c = (tn0 + n) * 8 + 2 * t;
        Pn[c * LP + 32 * k + ti * 8 + g] = -acc[0][n][0];
        Pn[(c + 1) * LP + 32 * k + ti * 8 + g] = -acc[0][n][1];
      }
      __syncthreads();
      // S_ij += R_ik X_kj, i < k; R_ik(r, q) = R(32i + r, 32k + q)
      auto fxk = [&](int n, int q) { return Pn[((tn0 + n) * 8 + g) * LP + 32 * k + q]; };
      int i = 0;
      for (; CHOL_PAIRS && i + 1 < k; i += 2) {
        double a2[2][2][2] = {};
        blk_mma<2>(a2, t, [&](int b, int q) {
          return __ldcg(R + (int64_t)(32 * k + q) * w + 32 * (i + b) + ti * 8 + g); }, fxk);
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int n = 0; n < 2; ++n) {
            const int c = (tn0 + n) * 8 + 2 * t;
            Pn[c * LP + 32 * (i + b) + ti * 8 + g] += a2[b][n][0];
            Pn[(c + 1) * LP + 32 * (i + b) + ti * 8 + g] += a2[b][n][1];
          }
      }
      for (; i < k; ++i) {
        double a1[1][2][2] = {};
        blk_mma<1>(a1, t, [&](int, int q) { return __ldcg(R + (int64_t)(32 * k + q) * w + 32 * i + ti * 8 + g); },
                   fxk);
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          const int c = (tn0 + n) * 8 + 2 * t;
          Pn[c * LP + 32 * i + ti * 8 + g] += a1[0][n][0];
          Pn[(c + 1) * LP + 32 * i + ti * 8 + g] += a1[0][n][1];
        }
      }
      __syncthreads();
    }
  }
  // the panel of R^-1 (rows 0 .. c0 - 1; the diagonal block was written with R_jj)
  for (int c = warp; c < jb; c += kClThr / 32)
    for (int i = lane; i < c0; i += 32) Rinv[(int64_t)(c0 + c) * w + i] = Pn[c * LP + i];
  if (tid == 0 && status) {
    int cnt = 0;
    for (int p = 0; p < jb; ++p) cnt += s_defi[p];
    if (cnt) atomicAdd(&status->deficient, cnt);
  }
  CH_T(6);
  cluster.sync();   // the near-identity flags (read through DSMEM) stay valid until everyone is done
}

}  // namespace

int launch_chol_big(const double* G, const double* ref, int w, double tol, double* R, double* Rinv,
                    DevStatus* status, cudaStream_t st, double shift_coef) {
  if (w < 1 || w > kMaxW) return RSVD_E_ARG;
  const size_t smem = (size_t)(kNB * kMaxW + 2 * kNB * 33 + kMaxW) * 8 + kMaxW * 4;
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_chol_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_chol_big<<<1, kThr, smem, st>>>(G, ref, w, tol, shift_coef, R, Rinv, status);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

int launch_chol_cl(const double* G, const double* ref, int w, double tol, double* R, double* Rinv, DevStatus* status,
                   cudaStream_t st, double shift_coef) {
  if (w < 1 || w > kMaxW) return RSVD_E_ARG;
  const int nb = (w + 31) / 32;
  const size_t smem = ((size_t)32 * (32 * nb + 4) + 2 * 32 * 33 + kMaxW) * 8;
  static std::atomic<bool> attr{false};
  if (!attr) {
    cudaFuncSetAttribute(k_chol_cl, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(((size_t)32 * (32 * 16 + 4) + 2 * 32 * 33 + kMaxW) * 8));
    cudaFuncSetAttribute(k_chol_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb);
  cfg.blockDim = dim3(kClThr);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nb;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_chol_cl, G, ref, w, tol, shift_coef, R, Rinv, status);
  return e == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

}  // namespace rsvd
