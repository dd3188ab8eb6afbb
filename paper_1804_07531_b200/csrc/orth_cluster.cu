// CholeskyQR2 (and shifted CholeskyQR3) of a tall-skinny block in ONE launch on a thread-block
// cluster: the qr of PAPER.md P:69, applied to the m x l and n x l blocks at P:149/151 (Alg. 2),
// P:671 (Alg. 7) and P:910-922 (Alg. 9 Krylov blocks).  For blocks that fit in the cluster's
// shared memory (w <= 64, rows x w x 8 <= ~3.4 MB: every C1/C2 block), it replaces the chain
// pass / pass / apply kernels whose serial finishers dominated the small configurations.
//
//   each CTA: its row chunk of Y resident in shared memory for the whole call
//   per pass:  [apply R_prev^-1 in place]  Gram partial (FP64 DMMA)  -> cluster barrier
//              CTA 0: fixed-order DSMEM sum of the partials, guarded Cholesky G = R^T R and
//              R^-1 (thread j owns column j, in registers)          -> cluster barrier
//              every CTA copies R^-1 from CTA 0's shared memory (DSMEM)
//   end:       apply the last R^-1, write Q over Y; R_out = R_2 R_1 (R_2 R_1 R_0 when shifted)
// Same numerics as the pass kernels (small_kernels.cu): rank guard d_j <= tol * ref_j zeroes
// row j of R and column j of R^-1; the second pass takes the first-order closed form when
// |G - I| <= 1e-8.  The kernel is compiled per padded width W (multiple of 8): the padding
// columns of Y are zero and the padding block of G is set to the identity, so they factor
// trivially, never count as deficient and never mix with the real columns.
// Deterministic (fixed summation orders).
#include <atomic>
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace rsvd {
namespace {

constexpr int kThreads = 256;
constexpr int kCluster = 16;
constexpr int kSmemMax = 220 * 1024;

// smem row stride for a W-wide tile: == 4 (mod 16) -> conflict-free m8n8k4 fragment loads
__host__ __device__ constexpr int oc_ld(int W) { return W + ((4 - W % 16) + 16) % 16; }
// fixed smem (doubles): Ri (W x ld), G (W x W), broadcast / pivot scratch
__host__ __device__ constexpr int oc_fixed(int W) { return W * oc_ld(W) + W * W + 4 * 64; }
__host__ __device__ constexpr int oc_rows_max(int W) {
  return ((kSmemMax / 8 - oc_fixed(W)) / oc_ld(W)) / 16 * 16;
}

enum { PASS_SHIFT = 0, PASS_GUARD = 1, PASS_SECOND = 2 };

#ifdef RSVD_ORTH_TIMING
__device__ long long g_orth_t[32];
#define OT(i) do { if (threadIdx.x == 0 && cg::this_cluster().block_rank() == 0) g_orth_t[i] = clock64(); } while (0)
#else
#define OT(i) do {} while (0)
#endif

// The factorisation runs with every thread of the CTA in uniform control flow (threads
// j >= W only take part in the synchronisation): a warp that enters warp-synchronous code in a
// diverged state executes every shuffle on the slow divergent path (measured ~100x slower).
template <int W>
__device__ __forceinline__ void csync() {
  if (W <= 32) __syncwarp(); else asm volatile("bar.sync 1, 64;" ::: "memory");
}
// warps that run the factorisation (they do nothing else on CTA 0, so they enter it converged)
template <int W>
__host__ __device__ constexpr int chol_warps() { return W <= 32 ? 1 : 2; }

// Guarded Cholesky of the W x W matrix G (smem, col-major, padding block = I), thread j owning
// column j.  The column lives in registers as a shift register: before pivot p, c[i] holds the
// updated entry G~(p + i, j), so every register index is a compile-time constant while the
// pivot loop itself stays a compact runtime loop (straight-line code executed once is dominated
// by instruction-cache misses).  R(p, j) goes to shared memory (G is overwritten: its upper
// triangle becomes R), then thread j back-substitutes column j of R^-1 into Ri.
// Writes R (global, col-major w x w, the real block).  Returns the deficient real columns.
template <int W>
__device__ int chol_inv_cols(double* G, int w, double shift, double tol, double* R, double* Ri, int ld, double* bc) {
  const int j = threadIdx.x;  // column; threads j >= W only take part in the barriers
  const bool act = j < W;
  double* rrow = bc;          // R(p, .) broadcast, 2W slots (the upper W stay 0)
  double* invd = bc + 128;    // 1 / R(p, p), 0 for a deficient pivot
  double c[W];
#pragma unroll
  for (int i = 0; i < W; ++i) c[i] = act ? G[j * W + i] : 0.0;
  const double sj = (j < w) ? shift : 0.0;
  // W <= 32: the pivot and the broadcast row are double-buffered by pivot parity (rows at bc and
  // bc + 64, pivots at bc[192..195]), so a pivot needs two barriers instead of three
  constexpr bool DB = (W <= 32);
  if (j < 2 * W && j >= W) {
    rrow[j] = 0.0;
    if (DB) rrow[64 + j] = 0.0;
  }
  double refj = 0.0;
#pragma unroll
  for (int i = 0; i < W; ++i)
    if (i == j) refj = c[i] + sj;  // G_jj + shift: the rank-guard reference
  csync<W>();                      // everyone has read G before it is overwritten with R
  int ndef = 0;
  OT(25);
  // rrow has 2W slots so that rrow[p + i] (i < W) never needs clamping; pivot values are
  // broadcast through shared memory (immediate-offset loads, no shuffles).  8 pivots per iteration
  // with c indexed from the window base p0 and updated in place at compile-time offsets (k, i);
  // the window shifts once per 8 pivots.  (A one-pivot runtime loop over a shift register made
  // the compiler copy the whole column every pivot: W = 64 74k -> 46k cycles, W = 32 24k -> 18k.)
  {
    for (int p0 = 0; p0 < W; p0 += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int p = p0 + k;
        double* rr = rrow + (DB ? 64 * (k & 1) : 0);
        double* pv = bc + 192 + (DB ? 2 * (k & 1) : 0);
        if (j == p) {
          c[k] += sj;
          pv[0] = c[k];
          pv[1] = refj;
        }
        csync<W>();
        const double d = pv[0], rf = pv[1];
        const bool def = !(d > tol * rf) || !(rf > 0.0);
        ndef += (def && p < w) ? 1 : 0;
        const double inv = def ? 0.0 : rsqrt_nr(d);
        const double rpj = (j > p) ? c[k] * inv : ((j == p) ? d * inv : 0.0);
        if (act && j >= p) G[j * W + p] = def ? 0.0 : rpj;  // R(p, j)
        if (j == p) invd[p] = inv;
        if (act) rr[j] = rpj;
        csync<W>();
        const double* rp = rr + p0;  // rp[i] = R(p, p0 + i)
        // a deficient pivot has rpj = 0: the update leaves c unchanged (no select needed)
#pragma unroll
        for (int i = k + 1; i < W; ++i) c[i] = fma(-rp[i], rpj, c[i]);
        if (!DB) csync<W>();
      }
#pragma unroll
      for (int i = 0; i < W - 8; ++i) c[i] = c[i + 8];
#pragma unroll
      for (int i = W - 8; i < W; ++i) c[i] = 0.0;
    }
  }
  csync<W>();
  OT(26);
  // R (global, real block; lower part zero) and, for the row solves, R row-major with
  // 1 / R_jj on the diagonal (0 for a deficient pivot) in Ri
  if (act) {
    for (int i = 0; i < W; ++i) {
      const double r = (i <= j) ? G[j * W + i] : 0.0;
      if (R && i < w && j < w) R[j * w + i] = r;
      Ri[i * ld + j] = (i == j) ? invd[j] : r;
    }
  }
  OT(27);
  return ndef;
}

// O = Yc Ri for this warp's 8-row tiles (mt = warp, warp + 8, ...), up to 4 tiles at once
// (4 * W/8 independent DMMA chains).  In place (out == nullptr) or to global column-major out.
template <int W>
__device__ __forceinline__ void apply_rinv(double* Yc, const double* Ri, int rpc, int warp_in, int g, int t4,
                                           double* out, int64_t ldo, int nr, int w) {
  constexpr int NT = W / 8, ld = oc_ld(W);
  const int warp = __shfl_sync(0xffffffffu, warp_in, 0);  // uniform: the tile predicates need no WARPSYNC
  const int nmt = rpc / 8;
  for (int mt0 = warp; mt0 < nmt; mt0 += 32) {
    double oc[4][NT][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n) oc[m][n][0] = oc[m][n][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < W; k0 += 4) {
      double b[NT];
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = Ri[(n * 8 + g) * ld + k0 + t4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int mt = mt0 + 8 * m;
        if (mt < nmt) {
          const double a = Yc[(mt * 8 + g) * ld + k0 + t4];
#pragma unroll
          for (int n = 0; n < NT; ++n) dmma(oc[m][n][0], oc[m][n][1], a, b[n]);
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int mt = mt0 + 8 * m;
      if (mt >= nmt) continue;
      const int row = mt * 8 + g;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int c0 = n * 8 + 2 * t4;
        if (out == nullptr) {
          *reinterpret_cast<double2*>(Yc + row * ld + c0) = make_double2(oc[m][n][0], oc[m][n][1]);
        } else if (row < nr) {
          if (c0 < w) out[(int64_t)c0 * ldo + row] = oc[m][n][0];
          if (c0 + 1 < w) out[(int64_t)(c0 + 1) * ldo + row] = oc[m][n][1];
        }
      }
    }
  }
}

// Gram partial G (upper triangle, col-major W x W) = Yc^T Yc over this CTA's rpc rows: warp q
// owns upper 8x8 tiles q, q+8, ... over all rows, with 4 DMMA chains per tile (k-steps
// interleaved) summed in a fixed order: no cross-warp reduction.
// Yc <- Yc R^-1 by forward substitution, one thread per row (q R = y): Rm is R row-major
// (Rm[i*ld + k] = R(i, k)) with 1/R_jj on the diagonal.  The row lives in registers, indexed
// from an 8-column window that shifts once per 8 columns, so the column loop stays compact.
// Reads past column W-1 of a row of Rm (its padding, the next row, or G after the last row)
// only ever multiply into entries beyond the row, which are never solved or stored.
template <int W>
__device__ __forceinline__ void solve_rows(double* Yc, const double* Rm, int rpc, int tid) {
  constexpr int ld = oc_ld(W);
  for (int r = tid; r < rpc; r += kThreads) {
    double* yr = Yc + r * ld;
    double y[W];
    // 16-byte accesses (ld is even and Yc 16-byte aligned): a row per thread at stride ld hits
    // only a few banks, so half as many accesses means half the conflicted wavefronts
#pragma unroll
    for (int i = 0; i < W; i += 2) {
      const double2 v = *reinterpret_cast<const double2*>(yr + i);
      y[i] = v.x;
      y[i + 1] = v.y;
    }
    // 8 columns per iteration, y indexed from the window base j0 and solved in place at
    // compile-time offsets, the window shifted once per 8 columns (as in the Cholesky)
    {
      for (int j0 = 0; j0 < W; j0 += 8) {
        double qe = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double* rj = Rm + (j0 + k) * ld + j0;  // R(j0 + k, j0 + i) at rj[i]
          const double q = y[k] * rj[k];
          if (k & 1) *reinterpret_cast<double2*>(yr + j0 + k - 1) = make_double2(qe, q);
          else qe = q;
#pragma unroll
          for (int i = k + 1; i < W; ++i) y[i] = fma(-q, rj[i], y[i]);
        }
#pragma unroll
        for (int i = 0; i < W - 8; ++i) y[i] = y[i + 8];
#pragma unroll
        for (int i = W - 8; i < W; ++i) y[i] = 0.0;
      }
    }
  }
}

template <int W>
__device__ __forceinline__ void gram_tiles(const double* Yc, int rpc, double* G, int warp_in, int g, int t4) {
  constexpr int NT = W / 8, NTILES = NT * (NT + 1) / 2, ld = oc_ld(W);
  // a provably warp-uniform warp index: a tile predicate on it needs no WARPSYNC before the
  // predicated mma.sync (rpc is a multiple of 16, so the k-steps need no predicate at all)
  const int warp = __shfl_sync(0xffffffffu, warp_in, 0);
  constexpr int TPW = (NTILES + 7) / 8;  // tiles per warp (max)
  int tbi[TPW], tbj[TPW];
#pragma unroll
  for (int q = 0; q < TPW; ++q) {
    int u = warp + 8 * q, bi = 0;
    if (u >= NTILES) u = NTILES - 1;
    while (u >= NT - bi) { u -= NT - bi; ++bi; }
    tbi[q] = bi;
    tbj[q] = bi + u;
  }
  double ga[TPW][4][2];
#pragma unroll
  for (int q = 0; q < TPW; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) ga[q][r][0] = ga[q][r][1] = 0.0;
  for (int k0 = 0; k0 < rpc; k0 += 16) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int kr = k0 + 4 * r + t4;
#pragma unroll
      for (int q = 0; q < TPW; ++q)
        if (warp + 8 * q < NTILES)
          dmma(ga[q][r][0], ga[q][r][1], Yc[kr * ld + tbi[q] * 8 + g], Yc[kr * ld + tbj[q] * 8 + g]);
    }
  }
#pragma unroll
  for (int q = 0; q < TPW; ++q)
    if (warp + 8 * q < NTILES) {
      const int i = tbi[q] * 8 + g;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int jj = tbj[q] * 8 + 2 * t4 + h;
        if (tbi[q] < tbj[q] || i <= jj)
          G[jj * W + i] = (ga[q][0][h] + ga[q][1][h]) + (ga[q][2][h] + ga[q][3][h]);
      }
    }
  __syncthreads();
}

// out = A B for upper-triangular A, B (col-major W x W in shared memory, zero outside w x w) on
// FP64 DMMA: warp q owns the upper 8x8 output tiles q, q+8, ...; tile (bi, bj) sums the k-blocks
// bi..bj (the only non-zero contributions) in k order.  out is col-major w x w (global), lower
// triangle zero.  The warp index is shuffled to make the loop bounds provably warp-uniform.
template <int W>
__device__ __forceinline__ void triu_product_dmma(const double* As, const double* Bs, int w, double* out, int warp_in,
                                                  int g, int t4) {
  constexpr int NT = W / 8, NTILES = NT * (NT + 1) / 2;
  const int warp = __shfl_sync(0xffffffffu, warp_in, 0);
  // the strictly lower triangle (the tiles below the diagonal are not computed); the lower
  // entries of the diagonal tiles are also written as 0 below, the same value
  for (int e = threadIdx.x; e < w * w; e += kThreads)
    if (e % w > e / w) out[e] = 0.0;
  for (int u0 = warp; u0 < NTILES; u0 += 8) {
    int u = u0, bi = 0;
    while (u >= NT - bi) { u -= NT - bi; ++bi; }
    const int bj = bi + u;
    double d0 = 0.0, d1 = 0.0;
    for (int k0 = bi * 8; k0 < bj * 8 + 8; k0 += 4)
      dmma(d0, d1, As[(k0 + t4) * W + bi * 8 + g], Bs[(bj * 8 + g) * W + k0 + t4]);
    const int i = bi * 8 + g;
    const int k = bj * 8 + 2 * t4;
    if (i < w && k < w) out[k * w + i] = (i <= k) ? d0 : 0.0;
    if (i < w && k + 1 < w) out[(k + 1) * w + i] = (i <= k + 1) ? d1 : 0.0;
  }
}

// (upper-triangular A B)(i, k) = sum_{q=i..k} A(i, q) B(q, k), col-major w x w, four named
// accumulators (an accumulator array indexed by q & 3 lives in local memory)
__device__ __forceinline__ double triu_dot(const double* A, const double* B, int w, int i, int k) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int q = i;
  for (; q + 3 <= k; q += 4) {
    s0 = fma(A[q * w + i], B[k * w + q], s0);
    s1 = fma(A[(q + 1) * w + i], B[k * w + q + 1], s1);
    s2 = fma(A[(q + 2) * w + i], B[k * w + q + 2], s2);
    s3 = fma(A[(q + 3) * w + i], B[k * w + q + 3], s3);
  }
  for (; q <= k; ++q) s0 = fma(A[q * w + i], B[k * w + q], s0);
  return (s0 + s1) + (s2 + s3);
}

template <int W>
__global__ void __launch_bounds__(kThreads, 1)
    k_orth_cluster(double* __restrict__ Y, int64_t ldy, int64_t rows, int w, int rpc, int shifted, double shift_coef,
                   double* __restrict__ Rout, double* __restrict__ Rw /* 3 w*w global scratch */,
                   DevStatus* status) {
  constexpr int ld = oc_ld(W);
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  extern __shared__ double osm[];
  double* Ri = osm;                 // W x ld  (R^-1, col-major: Ri[n*ld + k] = R^-1(k, n))
  double* G = Ri + W * ld;          // W x W   (Gram partial, col-major; on CTA 0 the reduced G)
  double* bc = G + W * W;           // 4*64    scratch of the factorisation
  double* Yc = bc + 4 * 64;         // rpc x ld (this CTA's rows, row-major)
  __shared__ int fast;
  __shared__ int mode;   // how Ri is to be applied: 0 = explicit R^-1 (DMMA), 1 = R (row solve)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t r0 = (int64_t)crank * rpc;
  const int nr = (int)max((int64_t)0, min((int64_t)rpc, rows - r0));
  OT(0);
  // ---- load this CTA's rows (W/8 x 8 independent loads in flight per thread)
  for (int i = tid; i < rpc; i += kThreads) {
#pragma unroll
    for (int c0 = 0; c0 < W; c0 += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (c0 + u < w && i < nr) ? Y[(int64_t)(c0 + u) * ldy + r0 + i] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) Yc[i * ld + c0 + u] = v[u];
    }
  }
  __syncthreads();
  OT(1);
  const int npass = shifted ? 3 : 2;
  double* R1 = Rw;             // R of the guard pass (global scratch, w x w)
  double* Rc = Rw + w * w;     // R of the current pass
  double* R0 = Rw + 2 * w * w; // R of the shift pass (shifted only)
  for (int ps = 0; ps < npass; ++ps) {
    const int kind = shifted ? ps : ps + 1;  // PASS_SHIFT / PASS_GUARD / PASS_SECOND
    if (ps > 0) {
      if (mode) solve_rows<W>(Yc, Ri, rpc, tid);
      else apply_rinv<W>(Yc, Ri, rpc, warp, g, t4, nullptr, 0, 0, 0);
      __syncthreads();
    }
    gram_tiles<W>(Yc, rpc, G, warp, g, t4);
    OT(2 + 6 * ps);
#ifdef RSVD_ORTH_GRAM_TWICE  // probe only: the same Gram again (warm instruction cache)
    if (ps == 0) {
      gram_tiles<W>(Yc, rpc, G, warp, g, t4);
      OT(31);
    }
#endif
    cluster.sync();
    OT(3 + 6 * ps);
    // all-reduce over the whole cluster: upper-triangle entry e (W*W <= C * kThreads, so at most
    // one per thread) is summed by one thread of one CTA (partials of CTA 0..C-1, in that order),
    // and after a barrier (every partial read) written into the G of EVERY CTA.  Each CTA then
    // factors the same bits with the same code, so R and R^-1 are identical on all CTAs and no
    // CTA copies R^-1 from CTA 0 (that DSMEM broadcast through one SM's port cost 7.7k / 25k
    // cycles per pass at W = 32 / 64).
    {
      static_assert(W * W <= kCluster * kThreads, "one Gram entry per thread");
      const int e = crank * kThreads + tid;
      const int i = e % W, jj = e / W;
      const bool own = e < W * W && i <= jj;
      double sum = 0.0;
      if (own) {
        double v[kCluster];
#pragma unroll
        for (int k = 0; k < kCluster; ++k) v[k] = (k < C) ? cluster.map_shared_rank(G, k)[e] : 0.0;
        sum = v[0];
#pragma unroll
        for (int k = 1; k < kCluster; ++k) sum += v[k];
        if (jj >= w) sum = (i == jj) ? 1.0 : 0.0;
      }
      cluster.sync();  // every partial has been read
      if (own)
        for (int k = 0; k < C; ++k) cluster.map_shared_rank(G, k)[e] = sum;
    }
    cluster.sync();    // every sum has landed
    {
      // bookkeeping warps (>= CW): mirror, second-pass test; factorisation warps (< CW) wait
      constexpr int CW = chol_warps<W>();
      const int bt = tid - 32 * CW, nbt = kThreads - 32 * CW;
      if (warp >= CW && bt == 0) {
        fast = (kind == PASS_SECOND) ? 1 : 0;
        mode = (kind == PASS_SECOND) ? 0 : 1;
      }
      __syncthreads();
      if (warp >= CW)
        for (int e = bt; e < W * W; e += nbt) {
          const int i = e % W, jj = e / W;
          if (i > jj) G[e] = G[i * W + jj];
        }
      __syncthreads();
      OT(4 + 6 * ps);
      if (kind == PASS_SECOND) {
        if (warp >= CW)
          for (int e = bt; e < W * W; e += nbt) {
            const int i = e % W, k = e / W;
            if (G[i * W + i] != 0.0 && G[k * W + k] != 0.0) {
              const double E = G[e] - (i == k ? 1.0 : 0.0);
              if (!(fabs(E) <= 1e-8)) fast = 0;
            }
          }
        __syncthreads();
      }
      if (fast) {
        if (warp >= CW)
          for (int e = bt; e < W * W; e += nbt) {
            const int i = e % W, k = e / W;
            const bool dz = G[i * W + i] == 0.0 || G[k * W + k] == 0.0;
            double r = 0.0, ri = 0.0;
            if (!dz && i <= k) {
              const double E = G[e] - (i == k ? 1.0 : 0.0);
              r = (i == k) ? 1.0 + 0.5 * E : E;
              ri = (i == k) ? 1.0 - 0.5 * E : -E;
            }
            if (crank == 0 && i < w && k < w) Rc[k * w + i] = r;
            Ri[k * ld + i] = ri;
          }
      } else if (warp < CW) {
        double shift = 0.0;
        if (kind == PASS_SHIFT) {
          double tr = 0.0;
          for (int jj = 0; jj < w; ++jj) tr += G[jj * W + jj];
          shift = shift_coef * tr;
        }
        const double tol = (kind == PASS_SHIFT) ? 0.0 : 1e-12;
        double* Rdst = crank != 0 ? nullptr : (kind == PASS_GUARD) ? R1 : (kind == PASS_SHIFT) ? R0 : Rc;
        const int cnt = chol_inv_cols<W>(G, w, shift, tol, Rdst, Ri, ld, bc);
        if (tid == 0) mode = 1;
        if (tid == 0 && crank == 0 && kind == PASS_GUARD && cnt && status) atomicAdd(&status->deficient, cnt);
      }
      __syncthreads();
      OT(5 + 6 * ps);
    }
    OT(6 + 6 * ps);
    __syncthreads();
  }
  OT(20);
  // ---- final apply, write Q over Y
  if (mode) {
    solve_rows<W>(Yc, Ri, rpc, tid);
    __syncthreads();
    for (int i = tid; i < nr; i += kThreads)
      for (int c = 0; c < w; ++c) Y[(int64_t)c * ldy + r0 + i] = Yc[i * ld + c];
  } else {
    apply_rinv<W>(Yc, Ri, rpc, warp, g, t4, Y + r0, ldy, nr, w);
  }
  OT(28);
  // R_out = R_2 R_1 (R_2 R_1 R_0 when shifted; upper triangular products), CTA 0
  if (Rout && crank == 0) {
    __syncthreads();
    OT(29);
    // both factors in shared memory: G is free on CTA 0 now, and so is the row buffer Yc after the
    // final apply.  When Yc holds a W x W block the products run on DMMA (W-padded, zero outside
    // w x w); tiny blocks keep the scalar dot products with the second factor in global memory
    // (a dependent loop over global loads costs an L2 round trip per step).
    if ((int64_t)rpc * ld >= (int64_t)W * W) {
      auto stage = [&](double* dst, const double* src) {
        // 8 independent L2 loads in flight per thread (a load -> store loop pays one round trip
        // per element)
        for (int e0 = tid; e0 < W * W; e0 += 8 * kThreads) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * kThreads, i = e % W, k = e / W;
            v[u] = (e < W * W && i < w && k < w) ? src[k * w + i] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * kThreads;
            if (e < W * W) dst[e] = v[u];
          }
        }
      };
      if (shifted) {  // R_1 <- R_1 R_0
        stage(G, R1);
        stage(Yc, R0);
        __syncthreads();
        triu_product_dmma<W>(G, Yc, w, R1, warp, g, t4);
        __syncthreads();
      }
      stage(G, Rc);   // R_out = R_2 R_1
      stage(Yc, R1);
      __syncthreads();
      OT(30);
      triu_product_dmma<W>(G, Yc, w, Rout, warp, g, t4);
    } else {
      if (shifted) {
        // R_1 <- R_1 R_0
        for (int e = tid; e < w * w; e += kThreads) G[e] = R1[e];
        __syncthreads();
        for (int e = tid; e < w * w; e += kThreads) {
          const int i = e % w, k = e / w;
          R1[e] = (i <= k) ? triu_dot(G, R0, w, i, k) : 0.0;
        }
        __syncthreads();
      }
      // R_out = R_2 R_1
      for (int e = tid; e < w * w; e += kThreads) G[e] = Rc[e];
      __syncthreads();
      OT(30);
      for (int e = tid; e < w * w; e += kThreads) {
        const int i = e % w, k = e / w;
        Rout[e] = (i <= k) ? triu_dot(G, R1, w, i, k) : 0.0;
      }
    }
  }
  OT(21);
  // no trailing cluster barrier: the last remote (DSMEM) accesses are the Gram-sum writes of the
  // last pass, which complete before that pass's cluster.sync
  OT(22);
}

template <int W>
int launch_w(double* Y, int64_t ldy, int64_t rows, int w, int shifted, double shift_coef, double* Rout, double* Rw,
             DevStatus* status, cudaStream_t st) {
  int rpc = (int)((rows + kCluster - 1) / kCluster);
  rpc = (rpc + 15) / 16 * 16;  // gram_tiles steps 16 rows at a time without a bounds predicate
  if (rpc > oc_rows_max(W)) return RSVD_E_ARG;
  const size_t smem = (size_t)(oc_fixed(W) + rpc * oc_ld(W)) * 8;
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_orth_cluster<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
    cudaFuncSetAttribute(k_orth_cluster<W>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kCluster);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_orth_cluster<W>, Y, ldy, rows, w, rpc, shifted, shift_coef, Rout, Rw,
                                     status);
  return e == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

}  // namespace

// true if the block fits the one-launch cluster path
bool orth_cluster_fits(int64_t rows, int w) {
  if (w < 1 || w > 64) return false;
  static constexpr int rmax[8] = {oc_rows_max(8),  oc_rows_max(16), oc_rows_max(24), oc_rows_max(32),
                                  oc_rows_max(40), oc_rows_max(48), oc_rows_max(56), oc_rows_max(64)};
  return rows <= (int64_t)kCluster * rmax[(w + 7) / 8 - 1];
}

int launch_orth_cluster(double* Y, int64_t ldy, int64_t rows, int w, int shifted, double shift_coef, double* Rout,
                        double* Rw, DevStatus* status, cudaStream_t st) {
  if (!orth_cluster_fits(rows, w)) return RSVD_E_ARG;
  switch ((w + 7) / 8) {
    case 1: return launch_w<8>(Y, ldy, rows, w, shifted, shift_coef, Rout, Rw, status, st);
    case 2: return launch_w<16>(Y, ldy, rows, w, shifted, shift_coef, Rout, Rw, status, st);
    case 3: return launch_w<24>(Y, ldy, rows, w, shifted, shift_coef, Rout, Rw, status, st);
    case 4: return launch_w<32>(Y, ldy, rows, w, shifted, shift_coef, Rout, Rw, status, st);
    case 5: return launch_w<40>(Y, ldy, rows, w, shifted, shift_coef, Rout, Rw, status, st);
    case 6: return launch_w<48>(Y, ldy, rows, w, shifted, shift_coef, Rout, Rw, status, st);
    case 7: return launch_w<56>(Y, ldy, rows, w, shifted, shift_coef, Rout, Rw, status, st);
    default: return launch_w<64>(Y, ldy, rows, w, shifted, shift_coef, Rout, Rw, status, st);
  }
}

}  // namespace rsvd
