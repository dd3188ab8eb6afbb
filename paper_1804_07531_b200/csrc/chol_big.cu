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
#include "common.cuh"
#include "internal.h"

namespace rsvd {
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

}  // namespace rsvd
