// Minimum-variance l_c for the single pass (Eq. MinVar).
//
// After the one view, the trial spectra lambda_{1..k}(l_c), l_c = 0..p, come from ONE QR of
// M = Phi^T Q_c U_c (l2 x l, U_c = right factor of the SVD of R_c, so Q_c U_c are the left singular
// vectors of Y_c).  QR is nested in the column count, so trial l_c's least-squares
// factor is the leading w = k + l_c block: C_w = Qh[:, :w] Rh[:w, :w] and
// X(l_c)^T = Y_r Qh_w Rh_w^-T.  With Y_r = Q_y R_y its singular values are those of the small
//     B_t = R_y Qh_w (Rh^-1)[:w, :w]^T = Z[:, :w] (Rh^-1)[:w, :w]^T,   Z = R_y Qh   (l2 x w).
// k_minvar_trials: one CTA per trial forms B_t and runs a values-only one-sided Jacobi on it.
// k_minvar_select: Var[s(l_c)] (unbiased, reading R19) and the argmin, smallest l_c on ties,
// with 0/0 = 1 and a/0 = inf (reading R20) -> an int in device memory.
// k_mask_cols: zero the columns j >= k + l_c of Q_c and C, so that the rest of Alg. 7 runs at
// the fixed width l with exact zero trailing columns (same result as truncating to k + l_c).
#include <atomic>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace rsvd {
namespace {

constexpr int kTrialThreads = 256;
constexpr int kTrialWarps = kTrialThreads / 32;
constexpr int kTrialMaxSweeps = 40;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// B (l2 x w, col-major, ld l2) lives in shared memory when it fits, else in the global scratch.
__global__ void __launch_bounds__(kTrialThreads) k_minvar_trials(const double* __restrict__ Z, int l2, int l,
                                                                  const double* __restrict__ Rhi, int k,
                                                                  double* __restrict__ lam, double* scratch,
                                                                  int use_smem) {
  extern __shared__ __align__(16) double smem[];
  const int t = blockIdx.x;
  const int w = k + t;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* B = use_smem ? smem : scratch + (int64_t)t * l2 * l;
  __shared__ double nrm[kMaxW32];
  __shared__ int rotated;
  // B[:, j] = sum_{i=j}^{w-1} Z[:, i] Rhi[j, i]   (Rhi upper triangular, ld l)
  for (int e = tid; e < l2 * w; e += kTrialThreads) {
    const int r = e % l2, j = e / l2;
    double acc = 0.0;
    for (int i = j; i < w; ++i) acc = fma(Z[(int64_t)i * l2 + r], Rhi[(int64_t)i * l + j], acc);
    B[(int64_t)j * l2 + r] = acc;
  }
  __syncthreads();
  // one-sided Jacobi, round-robin ordering (n players, n even; player n-1 fixed)
  const int n = (w + 1) & ~1;
  const double tol = 2.220446049250313e-16 * l2;  // dot-product rounding floor
  for (int sweep = 0; sweep < kTrialMaxSweeps && n > 1; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < n - 1; ++r) {
      for (int q = warp; q < n / 2; q += kTrialWarps) {
        int a, b;
        if (q == 0) {
          a = n - 1;
          b = r;
        } else {
          a = (r + q) % (n - 1);
          b = (r - q + n - 1) % (n - 1);
        }
        if (a >= w || b >= w) continue;
        const int i = min(a, b), j = max(a, b);
        double* bi = B + (int64_t)i * l2;
        double* bj = B + (int64_t)j * l2;
        double sa = 0.0, sb = 0.0, sc = 0.0;
        for (int e = lane; e < l2; e += 32) {
          const double x = bi[e], y = bj[e];
          sa = fma(x, x, sa);
          sb = fma(y, y, sb);
          sc = fma(x, y, sc);
        }
        sa = warp_sum(sa);
        sb = warp_sum(sb);
        sc = warp_sum(sc);
        if (sc == 0.0 || fabs(sc) <= tol * sqrt(sa * sb)) continue;
        const double zeta = (sb - sa) / (2.0 * sc);
        const double tt = (zeta != 0.0) ? copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta)) : 1.0;
        const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
        for (int e = lane; e < l2; e += 32) {
          const double x = bi[e], y = bj[e];
          bi[e] = cs * x - sn * y;
          bj[e] = sn * x + cs * y;
        }
        if (lane == 0) rotated = 1;
      }
      __syncthreads();
    }
    const int any = rotated;
    __syncthreads();
    if (!any) break;
  }
  // lambda = column norms, top k in descending order (ties by index)
  for (int j = warp; j < w; j += kTrialWarps) {
    double s = 0.0;
    for (int e = lane; e < l2; e += 32) s = fma(B[(int64_t)j * l2 + e], B[(int64_t)j * l2 + e], s);
    s = warp_sum(s);
    if (lane == 0) nrm[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < w; j += kTrialThreads) {
    int rank = 0;
    const double v = nrm[j];
    for (int i = 0; i < w; ++i) rank += (nrm[i] > v) || (nrm[i] == v && i < j);
    if (rank < k) lam[(int64_t)t * k + rank] = v;
  }
}

__device__ double ratio(double a, double b) {
  if (b > 0.0) return a / b;
  return (a == 0.0) ? 1.0 : INFINITY;
}

// lam: (p + 1) x k row-major (trial-major).  Same summation order as the oracle's minvar_select.
__global__ void k_minvar_select(const double* __restrict__ lam, int k, int p, int* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int best = 0;
  double best_var = INFINITY;
  for (int lc = 0; lc < p; ++lc) {
    const int j0 = lc > 0 ? lc - 1 : lc;
    const int cnt = (lc + 1 - j0 + 1) * k;
    double sum = 0.0;
    bool finite = true;
    for (int j = j0; j <= lc + 1; ++j)
      for (int i = 0; i < k; ++i) {
        const double s = ratio(lam[j * k + i], lam[lc * k + i]);
        finite = finite && isfinite(s);
        sum += s;
      }
    double var = INFINITY;
    if (finite) {
      const double mu = sum / cnt;
      double ss = 0.0;
      for (int j = j0; j <= lc + 1; ++j)
        for (int i = 0; i < k; ++i) {
          const double d = ratio(lam[j * k + i], lam[lc * k + i]) - mu;
          ss += d * d;
        }
      var = ss / (cnt - 1);
    }
    if (lc == 0 || var < best_var) {
      best = lc;
      best_var = var;
    }
  }
  *out = best;
}

__global__ void k_mask_cols(double* __restrict__ X, int64_t ld, int64_t rows, int w, int k,
                            const int* __restrict__ lc) {
  const int keep = k + *lc;
  const int64_t total = rows * (int64_t)(w - keep);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % rows;
    const int j = keep + (int)(e / rows);
    X[(int64_t)j * ld + r] = 0.0;
  }
}

}  // namespace

int64_t minvar_scratch(int l2, int l, int p) {
  return (int64_t)(p + 1) * l2 * l;
}

int launch_minvar_trials(const double* Z, int l2, int l, const double* Rhi, int k, int p, double* lam,
                         double* scratch, cudaStream_t st) {
  if (l > kMaxW32 || k < 1 || p < 0 || l2 < l) return RSVD_E_ARG;
  const size_t bytes = (size_t)l2 * l * 8;
  const int use_smem = bytes <= 200 * 1024 ? 1 : 0;
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_minvar_trials, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_minvar_trials<<<p + 1, kTrialThreads, use_smem ? bytes : 0, st>>>(Z, l2, l, Rhi, k, lam, scratch, use_smem);
  return cudaGetLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

int launch_minvar_select(const double* lam, int k, int p, int* out, cudaStream_t st) {
  k_minvar_select<<<1, 32, 0, st>>>(lam, k, p, out);
  return cudaGetLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

int launch_mask_cols(double* X, int64_t ld, int64_t rows, int w, int k, const int* lc, cudaStream_t st) {
  if (rows <= 0 || w <= k) return RSVD_OK;
  const int64_t total = rows * (int64_t)(w - k);
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  k_mask_cols<<<blocks, 256, 0, st>>>(X, ld, rows, w, k, lc);
  return cudaGetLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

}  // namespace rsvd
