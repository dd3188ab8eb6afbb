// Kernels that run between the matrix views (PAPER.md P:69 qr/chol, P:67 tsvd, P:159 lift):
//   slot sums (deterministic split-K reduction), Gram / cross products, guarded Cholesky with
//   pseudo-inverse of R (CholeskyQR2 building block), tall-skinny x small GEMM, one-sided
//   Jacobi SVD of the small core.  All fp64.
#include <atomic>
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <cstdlib>

namespace rsvd {

// ------------------------------------------------------------------ slot sum
__global__ void k_slot_sum(const double* __restrict__ in, int64_t ldi, int64_t slot_stride, int S, int64_t rows, int w,
                           double* __restrict__ out, int64_t ldo) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r >= rows || c >= w) return;
  const double* p = in + (int64_t)c * ldi + r;
  // loads in groups of 4 (in flight together), summed in slot order: same bits as a plain loop
  double s = p[0];
  int k = 1;
  for (; k + 4 <= S; k += 4) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = p[(int64_t)(k + u) * slot_stride];
#pragma unroll
    for (int u = 0; u < 4; ++u) s += v[u];
  }
  for (; k < S; ++k) s += p[(int64_t)k * slot_stride];
  out[(int64_t)c * ldo + r] = s;
}

int launch_slot_sum(const double* in, int64_t ldi, int64_t slot_stride, int S, int64_t rows, int w, double* out,
                    int64_t ldo, cudaStream_t st) {
  if (rows <= 0 || w <= 0) return RSVD_OK;
  dim3 grid((unsigned)((rows + 255) / 256), (unsigned)w);
  k_slot_sum<<<grid, 256, 0, st>>>(in, ldi, slot_stride, S, rows, w, out, ldo);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

// fp32 partial slots (the tf32 views' accumulation chunks) summed in fp64, in slot order
__global__ void k_slot_sum_f32(const float* __restrict__ in, int64_t ldi, int64_t slot_stride, int S, int64_t rows,
                               int w, double* __restrict__ out, int64_t ldo) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r >= rows || c >= w) return;
  const float* p = in + (int64_t)c * ldi + r;
  double s = (double)p[0];
  int k = 1;
  for (; k + 8 <= S; k += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = p[(int64_t)(k + u) * slot_stride];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += (double)v[u];
  }
  for (; k < S; ++k) s += (double)p[(int64_t)k * slot_stride];
  out[(int64_t)c * ldo + r] = s;
}

int launch_slot_sum_f32(const float* in, int64_t ldi, int64_t slot_stride, int S, int64_t rows, int w, double* out,
                        int64_t ldo, cudaStream_t st) {
  if (rows <= 0 || w <= 0) return RSVD_OK;
  dim3 grid((unsigned)((rows + 255) / 256), (unsigned)w);
  k_slot_sum_f32<<<grid, 256, 0, st>>>(in, ldi, slot_stride, S, rows, w, out, ldo);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

// ------------------------------------------------------------------ cross Gram  G = Xa^T Xb
// grid.x = row slots, grid.y = 64x64 output blocks (bi, bj).  256 threads, 4x4 register tile.
constexpr int kGR = 32;  // rows per smem tile
__global__ void __launch_bounds__(256) k_cross_gram(const double* __restrict__ Xa, int64_t lda_, int a,
                                                    const double* __restrict__ Xb, int64_t ldb, int b, int64_t rows,
                                                    int64_t rows_per_slot, double* __restrict__ slots, int nbj) {
  __shared__ double sa[kGR][64 + 2];
  __shared__ double sb[kGR][64 + 2];
  const int slot = blockIdx.x;
  const int bi = blockIdx.y / nbj, bj = blockIdx.y % nbj;
  const int i0 = bi * 64, j0 = bj * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = (int64_t)slot * rows_per_slot;
  const int64_t r1 = min(rows, r0 + rows_per_slot);
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int64_t rr = r0; rr < r1; rr += kGR) {
    // load: 64 columns x kGR rows of each operand (coalesced along rows)
    for (int e = threadIdx.x; e < 64 * kGR; e += 256) {
      const int col = e / kGR, row = e % kGR;
      const int64_t r = rr + row;
      const bool okr = r < r1;
      sa[row][col] = (okr && i0 + col < a) ? Xa[(int64_t)(i0 + col) * lda_ + r] : 0.0;
      sb[row][col] = (okr && j0 + col < b) ? Xb[(int64_t)(j0 + col) * ldb + r] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int row = 0; row < kGR; ++row) {
      double va[4], vb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) va[i] = sa[row][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) vb[j] = sb[row][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(va[i], vb[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* out = slots + (int64_t)slot * a * b;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gi = i0 + ty + 16 * i, gj = j0 + tx + 16 * j;
      if (gi < a && gj < b) out[(int64_t)gj * a + gi] = acc[i][j];
    }
}

int gram_slots(int64_t rows) {
  // 64 rows per slot: the per-slot loop over rows is a dependent latency chain, so more, shorter
  // slots finish sooner (C2's 4000-row Grams: 16 -> 63 CTAs); the slots are summed in order
  int64_t s = (rows + 63) / 64;
  if (s < 1) s = 1;
  if (s > 148) s = 148;
  return (int)s;
}

int launch_cross_gram(const double* Xa, int64_t lda_, int a, const double* Xb, int64_t ldb, int b, int64_t rows,
                      double* slots, int nslots, cudaStream_t st) {
  const int nbi = (a + 63) / 64, nbj = (b + 63) / 64;
  const int64_t rps = (rows + nslots - 1) / nslots;
  dim3 grid((unsigned)nslots, (unsigned)(nbi * nbj));
  k_cross_gram<<<grid, 256, 0, st>>>(Xa, lda_, a, Xb, ldb, b, rows, rps, slots, nbj);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

__global__ void k_slots_reduce_small(const double* __restrict__ slots, int nslots, int64_t count, double* __restrict__ G) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  // four interleaved partial sums (slot k goes to sum k % 4), combined in a fixed order: the loads
  // of a group are independent, so they are in flight together (deterministic: the order is fixed)
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int k = 0;
  for (; k + 3 < nslots; k += 4) {
    s0 += slots[(int64_t)k * count + i];
    s1 += slots[(int64_t)(k + 1) * count + i];
    s2 += slots[(int64_t)(k + 2) * count + i];
    s3 += slots[(int64_t)(k + 3) * count + i];
  }
  for (; k < nslots; ++k) s0 += slots[(int64_t)k * count + i];
  G[i] = (s0 + s1) + (s2 + s3);
}

int launch_slots_reduce_small(const double* slots, int nslots, int64_t count, double* G, cudaStream_t st) {
  k_slots_reduce_small<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(slots, nslots, count, G);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

// ------------------------------------------------------------------ guarded Cholesky
// G = R^T R (R upper).  Pivot j is "deficient" when d_j <= tol * ref_j with ref_j the reference
// squared norm of column j (G_jj itself, or the pre-projection norm for block Gram-Schmidt) —
// then row j of R is zero and column j of Rinv is zero (the column drops out of Q).
// Rinv is the upper-triangular inverse restricted to the kept columns.
constexpr int kCholMaxW = 160;
__global__ void __launch_bounds__(1024) k_chol(const double* __restrict__ G, const double* __restrict__ ref, int w,
                                               double tol, double shift_coef, double* __restrict__ R,
                                               double* __restrict__ Rinv, DevStatus* status) {
  extern __shared__ double S[];  // w*w (col-major), then deficient flags
  int* defi = reinterpret_cast<int*>(S + w * w);
  __shared__ double s_shift;
  __shared__ int s_fast;
  __shared__ double s_ref[kCholMaxW];   // guard references: a global load per pivot would sit on
                                        // the pivot chain (an L2 round trip per column)
  const int tid = threadIdx.x, nt = blockDim.x;
  if (ref == nullptr && shift_coef == 0.0 && chol_near_identity(G, w, R, Rinv, status, &s_fast)) return;
  for (int e = tid; e < w * w; e += nt) S[e] = G[e];
  for (int j = tid; j < w; j += nt) s_ref[j] = ref ? ref[j] : G[j * w + j];
  if (tid == 0) {
    // shifted CholeskyQR (Fukaya et al.): G + s I, s = shift_coef * ||Y||_F^2 >= shift_coef ||Y||_2^2
    double tr = 0.0;
    for (int j = 0; j < w; ++j) tr += G[j * w + j];
    s_shift = shift_coef * tr;
  }
  __syncthreads();
  if (shift_coef > 0.0) {
    for (int j = tid; j < w; j += nt) S[j * w + j] += s_shift;
    __syncthreads();
  }
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  for (int j = 0; j < w; ++j) {
    // every thread derives the pivot itself (no broadcast barrier); rsqrt gives 1/R_jj and R_jj
    const double d = S[j * w + j];
    const double rf = ref ? s_ref[j] : (s_ref[j] + s_shift * (shift_coef > 0.0));
    const bool def = !(d > tol * rf) || !(rf > 0.0);
    const double inv = def ? 0.0 : rsqrt_nr(d);
    // row j of R: R(j,i) = S(j,i) / R_jj, i > j  (S(j,i) at S[i*w + j])
    for (int i = j + 1 + tid; i < w; i += nt) S[i * w + j] *= inv;
    __syncthreads();  // row j complete; everyone has read S(j,j)
    if (tid == 0) {
      S[j * w + j] = def ? 0.0 : d * inv;
      defi[j] = def ? 1 : 0;
    }
    // trailing update of the upper triangle: S(i,k) -= R(j,i) R(j,k), j < i <= k
    // (warp per column k, lanes over rows i)
    if (!def)
      for (int k = j + 1 + warp; k < w; k += nwarp) {
        const double rjk = S[k * w + j];
        for (int i = j + 1 + lane; i <= k; i += 32) S[k * w + i] = fma(-S[i * w + j], rjk, S[k * w + i]);
      }
    __syncthreads();
  }
  // write R (upper, zero below)
  for (int e = tid; e < w * w; e += nt) {
    const int i = e % w, k = e / w;
    R[e] = (i <= k) ? S[k * w + i] : 0.0;
  }
  __syncthreads();
  // R^-1 in place, row by row from the bottom: X(i,j) = -(sum_{k=i+1..j} R(i,k) X(k,j)) / R(i,i);
  // each element's dot product split over lpe lanes (shuffle reduction)
  const int lpe = (w <= nt / 8) ? 8 : 4;
  const int el = tid / lpe, sl = tid % lpe;
  for (int i = w - 1; i >= 0; --i) {
    const int j = i + el;
    double x = 0.0;
    const bool act = (el < w - i);
    const bool live = act && !defi[i];
    double s = 0.0;
    if (live)
      for (int k = i + 1 + sl; k <= j; k += lpe) s = fma(S[k * w + i], S[j * w + k], s);
    __syncwarp();
    for (int o = lpe >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, lpe);
    if (live) {
      const double rii = S[i * w + i];
      x = (j == i) ? 1.0 / rii : -s / rii;
    }
    __syncthreads();
    if (act && sl == 0) S[j * w + i] = x;
    __syncthreads();
  }
  for (int e = tid; e < w * w; e += nt) {
    const int i = e % w, k = e / w;
    Rinv[e] = (i <= k) ? S[k * w + i] : 0.0;
  }
  if (tid == 0 && status) {
    int cnt = 0;
    for (int j = 0; j < w; ++j) cnt += defi[j];
    if (cnt) atomicAdd(&status->deficient, cnt);
  }
}

int launch_chol_cl(const double* G, const double* ref, int w, double tol, double* R, double* Rinv, DevStatus* status,
                   cudaStream_t st, double shift_coef);
int launch_chol_big(const double* G, const double* ref, int w, double tol, double* R, double* Rinv,
                    DevStatus* status, cudaStream_t st, double shift_coef);

static int chol_cl_from() {
  static const int v = [] {
    const char* e = getenv("RSVD_CHOL_CL_FROM");
    return e ? atoi(e) : 65;
  }();
  return v;
}

// launch_chol_ref takes the cluster kernel for this width: it reads only G's upper triangle
bool chol_reads_upper_only(int w) { return chol_cl_from() > 0 && w >= chol_cl_from() && w >= 33 && w <= 512; }

int launch_chol_ref(const double* G, const double* ref, int w, double tol, double* R, double* Rinv,
                    DevStatus* status, cudaStream_t st, double shift_coef) {
  static const int big_from = [] {
    const char* e = getenv("RSVD_CHOL_BIG_FROM");
    return e ? atoi(e) : kCholMaxW + 1;
  }();
  // the cluster kernel above RSVD_CHOL_CL_FROM (default 65; 0 disables it)
  if (chol_reads_upper_only(w)) return launch_chol_cl(G, ref, w, tol, R, Rinv, status, st, shift_coef);
  if (w > kCholMaxW || w >= big_from) return launch_chol_big(G, ref, w, tol, R, Rinv, status, st, shift_coef);
  if (w < 1) return RSVD_E_ARG;
  const size_t smem = (size_t)w * w * 8 + (size_t)w * 4 + 16;
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, kCholMaxW * kCholMaxW * 8 + kCholMaxW * 4 + 16);
    attr = true;
  }
  // 1024 threads: a 128 / 256-thread CTA (fewer warps per barrier) measured slower at w = 30
  // (C2 single pass: 2 x 22.4 us vs 2 x 20.0 us), the pivot chain is not barrier-bound
  k_chol<<<1, 1024, smem, st>>>(G, ref, w, tol, shift_coef, R, Rinv, status);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

int launch_chol(const double* G, int w, double* R, double* Rinv, double* /*Racc*/, DevStatus* status,
                cudaStream_t st) {
  return launch_chol_ref(G, nullptr, w, 1e-12, R, Rinv, status, st, 0.0);
}

// ------------------------------------------------------------------ tall-skinny x small GEMM
// out(rows x c) (=|-=) in(rows x w) M(w x c).  One thread per row, 16 output columns per CTA.
constexpr int kTsCC = 16;
__global__ void __launch_bounds__(128) k_ts_gemm(const double* __restrict__ in, int64_t ldi, int64_t rows, int w,
                                                 const double* __restrict__ M, int64_t ldm, int c,
                                                 double* __restrict__ out, int64_t ldo, int mode) {
  extern __shared__ double Ms[];  // w x kTsCC (row-major by k)
  const int c0 = blockIdx.y * kTsCC;
  for (int e = threadIdx.x; e < w * kTsCC; e += blockDim.x) {
    const int k = e / kTsCC, cc = e % kTsCC;
    Ms[e] = (c0 + cc < c) ? M[(int64_t)(c0 + cc) * ldm + k] : 0.0;
  }
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double acc[kTsCC];
#pragma unroll
  for (int i = 0; i < kTsCC; ++i) acc[i] = 0.0;
  for (int k = 0; k < w; ++k) {
    const double x = in[(int64_t)k * ldi + r];
    const double2* mrow = reinterpret_cast<const double2*>(Ms + k * kTsCC);
#pragma unroll
    for (int i = 0; i < kTsCC / 2; ++i) {
      const double2 mv = mrow[i];
      acc[2 * i] = fma(x, mv.x, acc[2 * i]);
      acc[2 * i + 1] = fma(x, mv.y, acc[2 * i + 1]);
    }
  }
#pragma unroll
  for (int i = 0; i < kTsCC; ++i) {
    if (c0 + i < c) {
      double* o = out + (int64_t)(c0 + i) * ldo + r;
      *o = mode ? (*o - acc[i]) : acc[i];
    }
  }
}

int launch_ts_gemm(const double* in, int64_t ldi, int64_t rows, int w, const double* M, int64_t ldm, int c,
                   double* out, int64_t ldo, int mode, cudaStream_t st) {
  if (rows <= 0 || c <= 0) return RSVD_OK;
  if (w > 1024) return RSVD_E_ARG;
  dim3 grid((unsigned)((rows + 127) / 128), (unsigned)((c + kTsCC - 1) / kTsCC));
  const size_t smem = (size_t)w * kTsCC * 8;
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_ts_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 * kTsCC * 8);
    attr = true;
  }
  k_ts_gemm<<<grid, 128, smem, st>>>(in, ldi, rows, w, M, ldm, c, out, ldo, mode);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

// ------------------------------------------------------------------ one-sided Jacobi SVD
// Hestenes: W = M J with plane rotations on column pairs (parallel round-robin ordering, one
// warp per pair) until every pair satisfies |w_p . w_q| <= tol sqrt(|w_p|^2 |w_q|^2).
// M = (W S^-1) S J^T  ->  left vectors W_j / s_j, right vectors J, values s_j = |W_j|.
constexpr int kJacThreads = 1024;
constexpr int kJacMaxC = 512;
// RPL: rows (and J entries) per lane held in registers during a rotation (r, ce <= 32 RPL): every
// load of a column pair is issued before any store (a load -> rotate -> store loop serialises on
// the possible aliasing of the two columns)
template <int RPL>
__global__ void __launch_bounds__(kJacThreads) k_jacobi(const double* __restrict__ M, int64_t ldm, int trans, int r,
                                                        int c, double* __restrict__ Ul, double* __restrict__ Sv,
                                                        double* __restrict__ Vr, double* __restrict__ gW,
                                                        double* __restrict__ gJ, int w_in_smem, int j_in_smem,
                                                        double tol, int max_sweeps, int want_j, DevStatus* status) {
  extern __shared__ double sm[];
  const int ce = c + (c & 1);  // even number of columns (pad with a zero column)
  double* W = w_in_smem ? sm : gW;
  double* J = j_in_smem ? (sm + (w_in_smem ? (int64_t)r * ce : 0)) : gJ;
  __shared__ int rotated;
  __shared__ double sval[kJacMaxC];
  __shared__ int srank[kJacMaxC];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  for (int e = tid; e < r * ce; e += nt) {
    const int i = e % r, j = e / r;
    double v = 0.0;
    if (j < c) v = trans ? M[(int64_t)i * ldm + j] : M[(int64_t)j * ldm + i];
    W[(int64_t)j * r + i] = v;
  }
  if (want_j)
    for (int e = tid; e < ce * ce; e += nt) J[e] = ((e % ce) == (e / ce)) ? 1.0 : 0.0;
  __syncthreads();
  int sweep = 0;
  bool converged = false;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < ce - 1; ++round) {
      for (int pi = warp; pi < ce / 2; pi += nwarp) {
        int p, q;
        if (pi == 0) {
          p = round;
          q = ce - 1;
        } else {
          p = (round + pi) % (ce - 1);
          q = (round - pi + (ce - 1)) % (ce - 1);
        }
        if (p > q) { const int tt = p; p = q; q = tt; }
        double* wp = W + (int64_t)p * r;
        double* wq = W + (int64_t)q * r;
        double xr[RPL], yr[RPL];
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          const int i = lane + 32 * t;
          xr[t] = (i < r) ? wp[i] : 0.0;
          yr[t] = (i < r) ? wq[i] : 0.0;
        }
        double a = 0.0, b = 0.0, cc = 0.0;
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          a = fma(xr[t], xr[t], a);
          b = fma(yr[t], yr[t], b);
          cc = fma(xr[t], yr[t], cc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          cc += __shfl_xor_sync(0xffffffffu, cc, o);
        }
        if (cc != 0.0 && fabs(cc) > tol * sqrt(a * b)) {
          // t = tan(theta), the smaller root of t^2 + 2 zeta t - 1 = 0, zeta = (b - a) / (2 c):
          // t = sign(d) e / (|d| + sqrt(d^2 + e^2)) with d = b - a, e = 2c.  Formed in fp32 from
          // the fp64 ratio when it is in range (any t gives an exactly orthogonal fp64 rotation,
          // cs = rsqrt(1 + t^2), sn = cs t; an approximate angle only leaves a ~1e-7 fraction of
          // the off-diagonal for the next sweep) — as in k_jacobi_small
          const double d = b - a, e = 2.0 * cc;
          const double ad = fabs(d), ae = fabs(e);
          double t;
          if (ad > 1e-30 && ad < 1e30 && ae > 1e-30 && ae < 1e30) {
            const float rf = (float)e / (float)ad;
            t = copysign(1.0, d) * (double)(rf / (1.0f + sqrtf(fmaf(rf, rf, 1.0f))));
          } else {
            t = copysign(1.0, d) * e / (ad + sqrt(fma(d, d, e * e)));
          }
          const double cs = rsqrt_nr(fma(t, t, 1.0));
          const double sn = cs * t;
#pragma unroll
          for (int t = 0; t < RPL; ++t) {
            const int i = lane + 32 * t;
            if (i < r) {
              wp[i] = cs * xr[t] - sn * yr[t];
              wq[i] = sn * xr[t] + cs * yr[t];
            }
          }
          if (want_j) {
            double* jp = J + (int64_t)p * ce;
            double* jq = J + (int64_t)q * ce;
            double xj[RPL], yj[RPL];
#pragma unroll
            for (int t = 0; t < RPL; ++t) {
              const int i = lane + 32 * t;
              xj[t] = (i < ce) ? jp[i] : 0.0;
              yj[t] = (i < ce) ? jq[i] : 0.0;
            }
#pragma unroll
            for (int t = 0; t < RPL; ++t) {
              const int i = lane + 32 * t;
              if (i < ce) {
                jp[i] = cs * xj[t] - sn * yj[t];
                jq[i] = sn * xj[t] + cs * yj[t];
              }
            }
          }
          if (lane == 0) rotated = 1;
        }
        __syncwarp();
      }
      __syncthreads();
    }
    if (!rotated) {
      converged = true;
      ++sweep;
      break;
    }
  }
  // singular values and descending ranks (ties broken by index)
  for (int j = warp; j < ce; j += nwarp) {
    const double* wj = W + (int64_t)j * r;
    double s = 0.0;
    for (int i = lane; i < r; i += 32) s = fma(wj[i], wj[i], s);
    s = warp_sum(s);
    if (lane == 0) sval[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < ce; j += nt) {
    const double sj = sval[j];
    int rk = 0;
    for (int i = 0; i < ce; ++i) {
      const double si = sval[i];
      rk += (si > sj) || (si == sj && i < j);
    }
    srank[j] = rk;
  }
  __syncthreads();
  for (int e = tid; e < r * ce; e += nt) {
    const int i = e % r, j = e / r;
    const int rk = srank[j];
    if (rk < c) {
      const double sj = sval[j];
      Ul[(int64_t)rk * r + i] = sj > 0.0 ? W[(int64_t)j * r + i] / sj : 0.0;
    }
  }
  if (want_j) {
    for (int e = tid; e < ce * ce; e += nt) {
      const int i = e % ce, j = e / ce;
      const int rk = srank[j];
      if (rk < c && i < c) Vr[(int64_t)rk * c + i] = J[(int64_t)j * ce + i];
    }
  } else {
    // right vectors from the left ones (B = W J^T, W = U S -> J = B^T U S^-1), as in k_jacobi_small
    for (int e = tid; e < c * ce; e += nt) {
      const int a = e % c, j = e / c;
      const int rk = srank[j];
      if (rk < c) {
        const double sj = sval[j];
        double sacc = 0.0;
        if (sj > 0.0)
          for (int i = 0; i < r; ++i) {
            const double bia = trans ? M[(int64_t)i * ldm + a] : M[(int64_t)a * ldm + i];
            sacc = fma(bia, W[(int64_t)j * r + i], sacc);
          }
        Vr[(int64_t)rk * c + a] = sj > 0.0 ? sacc / (sj * sj) : 0.0;
      }
    }
  }
  for (int j = tid; j < ce; j += nt)
    if (srank[j] < c) Sv[srank[j]] = sval[j];
  if (tid == 0 && status) {
    status->jacobi_sweeps = sweep;
    if (!converged) atomicAdd(&status->jacobi_fail, 1);
  }
}

// Medium cores (64 < c <= 128, r <= 128): the k_jacobi_small round (arithmetic round-robin pairs,
// padded W stride, MUFU angle, lagged J rotations) with 8 lanes x 16 rows per pair and J always
// accumulated (stride ce; in shared memory when W and J fit, else in the global scratch).
// WJ = 0: no J; right vectors B^T U S^-1 from the input in global memory (leading triplets only,
// as k_jacobi_small); 4 lanes x 32 rows per pair was the fastest no-J layout (tools/jac_small_probe).
template <int LPP, int RW, int WJ>
__global__ void __launch_bounds__(LPP == 4 ? 256 : 512) k_jacobi_mid(const double* __restrict__ M, int64_t ldm, int trans, int r, int c,
                                                    double* __restrict__ Ul, double* __restrict__ Sv,
                                                    double* __restrict__ Vr, double* __restrict__ gJ, int j_in_smem,
                                                    double tol, int max_sweeps, DevStatus* status) {
  constexpr int RS = LPP * RW + 4;
  extern __shared__ double jm_dyn[];
  const int ce = c + (c & 1);
  double* W = jm_dyn;                                 // ce x RS
  // WJ = 2: J in shared memory (a compile-time choice keeps the shared address space: LDS, not
  // generic loads); WJ = 1: J in the global scratch
  double* J = (WJ == 2) ? jm_dyn + (int64_t)ce * RS : gJ;   // ce x ce
  (void)j_in_smem;
  __shared__ double sval[128];
  __shared__ int srank[128];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int grp = tid / LPP, sl = tid % LPP;
  const unsigned gmask = ((1u << LPP) - 1u) << (tid & 31 & ~(LPP - 1));
  const int npairs = ce >> 1, m1 = ce - 1;
  for (int e = tid; e < ce * RS; e += nt) {
    const int i = e % RS, j = e / RS;
    double v = 0.0;
    if (i < r && j < c) v = trans ? M[(int64_t)i * ldm + j] : M[(int64_t)j * ldm + i];
    W[e] = v;
  }
  if (WJ)
    for (int e = tid; e < ce * ce; e += nt) J[e] = ((e % ce) == (e / ce)) ? 1.0 : 0.0;
  __syncthreads();
  const double tol2 = tol * tol;
  int sweep = 0;
  bool converged = false;
  int pj_p = 0, pj_q = 0, pj_on = 0;
  double pj_cs = 1.0, pj_sn = 0.0;
  auto apply_pending_j = [&]() {
    if (WJ && pj_on) {
      double* jp = J + (int64_t)pj_p * ce;
      double* jq = J + (int64_t)pj_q * ce;
      for (int k = sl; k < ce; k += LPP) {
        const double u = jp[k], v = jq[k];
        jp[k] = pj_cs * u - pj_sn * v;
        jq[k] = pj_sn * u + pj_cs * v;
      }
      pj_on = 0;
    }
  };
  const bool active = grp < npairs;
  for (; sweep < max_sweeps; ++sweep) {
    int rotated = 0, big = 0;
    for (int round = 0; round < m1; ++round) {
      {
        // every lane of every warp runs the round (inactive groups read column 0 and never
        // store): a warp that reaches the group shuffles diverged takes the serialised BRA.DIV
        // path (tools/jac_small_probe.cu: thousands of cycles per round instead of ~100)
        int p, q;
        {
          int pp = round + grp;
          if (pp >= m1) pp -= m1;
          int qq = round - grp;
          if (qq < 0) qq += m1;
          p = grp == 0 ? round : min(pp, qq);
          q = grp == 0 ? m1 : max(pp, qq);
          if (!active) p = q = 0;
        }
        double* wp = W + p * RS;
        double* wq = W + q * RS;
        double x[RW], y[RW];
#pragma unroll
        for (int t = 0; t < RW; ++t) {
          x[t] = wp[sl + LPP * t];
          y[t] = wq[sl + LPP * t];
        }
        double a0 = 0.0, b0 = 0.0, c0 = 0.0, a1 = 0.0, b1 = 0.0, c1 = 0.0;
#pragma unroll
        for (int t = 0; t < RW; t += 2) {
          a0 = fma(x[t], x[t], a0);
          b0 = fma(y[t], y[t], b0);
          c0 = fma(x[t], y[t], c0);
          a1 = fma(x[t + 1], x[t + 1], a1);
          b1 = fma(y[t + 1], y[t + 1], b1);
          c1 = fma(x[t + 1], y[t + 1], c1);
        }
        double a = a0 + a1, b = b0 + b1, cc = c0 + c1;
        __syncwarp();
#pragma unroll
        for (int o = LPP / 2; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o, LPP);
          b += __shfl_xor_sync(0xffffffffu, b, o, LPP);
          cc += __shfl_xor_sync(0xffffffffu, cc, o, LPP);
        }
        apply_pending_j();
        if (active && cc * cc > tol2 * (a * b) && cc != 0.0) {
          rotated = 1;
          big |= (cc * cc > 1e-20 * (a * b)) ? 1 : 0;
          const double d = b - a;
          double rd, rsq, rt;
          asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(fmax(fabs(d), 1e-300)));
          const double rho = fmin(fmax(2.0 * cc * rd, -1e100), 1e100);
          const double s1 = fma(rho, rho, 1.0);
          asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rsq) : "d"(s1));
          asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rt) : "d"(fma(s1, rsq, 1.0)));
          const double t = (d < 0.0 ? -rho : rho) * rt;
          const double cs = rsqrt_nr(fma(t, t, 1.0));
          const double sn = cs * t;
#pragma unroll
          for (int k = 0; k < RW; ++k) {
            wp[sl + LPP * k] = cs * x[k] - sn * y[k];
            wq[sl + LPP * k] = sn * x[k] + cs * y[k];
          }
          if (WJ) { pj_p = p; pj_q = q; pj_cs = cs; pj_sn = sn; pj_on = 1; }
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) {
      converged = true;
      ++sweep;
      break;
    }
    // quadratic convergence: when no rotation of this sweep had |c| / sqrt(ab) above 1e-10, the
    // off-diagonal left is O(1e-20), far below tol, so the confirming sweep is skipped
    if (!__syncthreads_or(big)) {
      converged = true;
      ++sweep;
      break;
    }
  }
  if (active) apply_pending_j();
  __syncthreads();
  for (int j = grp; j < ce; j += (nt / LPP)) {
    double sacc = 0.0;
#pragma unroll
    for (int t = 0; t < RW; ++t) {
      const double v = W[j * RS + sl + LPP * t];
      sacc = fma(v, v, sacc);
    }
#pragma unroll
    for (int o = LPP / 2; o > 0; o >>= 1) sacc += __shfl_xor_sync(gmask, sacc, o, LPP);
    if (sl == 0) sval[j] = sqrt(sacc);
  }
  __syncthreads();
  for (int j = tid; j < ce; j += nt) {
    const double sj = sval[j];
    int rk = 0;
    for (int i = 0; i < ce; ++i) {
      const double si = sval[i];
      rk += (si > sj) || (si == sj && i < j);
    }
    srank[j] = rk;
  }
  __syncthreads();
  for (int e = tid; e < r * ce; e += nt) {
    const int i = e % r, j = e / r;
    const int rk = srank[j];
    if (rk < c) {
      const double sj = sval[j];
      Ul[(int64_t)rk * r + i] = sj > 0.0 ? W[j * RS + i] / sj : 0.0;
    }
  }
  if (WJ) {
    for (int e = tid; e < ce * ce; e += nt) {
      const int i = e % ce, j = e / ce;
      const int rk = srank[j];
      if (rk < c && i < c) Vr[(int64_t)rk * c + i] = J[(int64_t)j * ce + i];
    }
  } else {
    // right vectors B^T U S^-1 (B = the input as seen by the sweep, read from global memory):
    // 4 x 2 register blocks (a, j)
    const int na = (c + 3) / 4, nj = ce / 2;
    for (int e = tid; e < na * nj; e += nt) {
      const int a0 = 4 * (e % na), j0 = 2 * (e / na);
      double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      for (int i = 0; i < r; ++i) {
        const double w0 = W[j0 * RS + i], w1 = W[(j0 + 1) * RS + i];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int a = min(a0 + u, c - 1);
          const double bb = trans ? M[(int64_t)i * ldm + a] : M[(int64_t)a * ldm + i];
          acc[u][0] = fma(bb, w0, acc[u][0]);
          acc[u][1] = fma(bb, w1, acc[u][1]);
        }
      }
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int j = j0 + v, rk = srank[j];
        if (rk >= c) continue;
        const double sj = sval[j];
        const double inv = sj > 0.0 ? 1.0 / (sj * sj) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (a0 + u < c) Vr[(int64_t)rk * c + a0 + u] = acc[u][v] * inv;
      }
    }
  }
  for (int j = tid; j < ce; j += nt)
    if (srank[j] < c) Sv[srank[j]] = sval[j];
  if (tid == 0 && status) {
    status->jacobi_sweeps = sweep;
    if (!converged) atomicAdd(&status->jacobi_fail, 1);
  }
}

static bool getenv_flag_jac(const char* n) {
  const char* e = getenv(n);
  return e && *e && *e != '0';
}

int launch_jacobi_small(const double* M, int64_t ldm, int trans, int r, int c, double* Ul, double* S, double* Vr,
                        DevStatus* status, cudaStream_t st, int want_j);
int launch_jacobi_cluster(const double* M, int64_t ldm, int trans, int r, int c, double* Ul, double* S, double* Vr,
                          double* scratch, DevStatus* status, cudaStream_t st, int want_j);
int launch_jacobi_gcl(const double* M, int64_t ldm, int trans, int r, int c, double* Ul, double* S, double* Vr,
                      double* scratch, DevStatus* status, cudaStream_t st, int want_j);

// want_j = 0: right vectors formed as B^T U S^-1 at the end (leading triplets only accurate)
int launch_jacobi_t(const double* M, int64_t ldm, int trans, int r, int c, double* Ul, double* S, double* Vr,
                    double* scratch, DevStatus* status, cudaStream_t st, int want_j) {
  if (c < 1 || c > kJacMaxC || r < c || r > kJacMaxC) return RSVD_E_ARG;
  // want_j: 0 = no J, 1 = J everywhere, 2 = J in the 64 < c <= 128 path only
  // block Jacobi with the Gram inner solver on a cluster (jacobi_gcl.cu) for c > 64, and for
  // c > 32 when J is accumulated (measured, tools/core_probe.py: w = 60 with J 0.58 vs 0.81 ms,
  // w = 120 1.15 vs 2.03 ms, w = 250 2.9 vs 8.1 ms); RSVD_JACOBI_GCL_FROM overrides the width,
  // RSVD_JACOBI_OLD_CLUSTER=1 keeps the one-CTA / plane-rotation cluster kernels
  static const int gcl_from = [] {
    const char* e = getenv("RSVD_JACOBI_GCL_FROM");
    return e ? atoi(e) : 0;
  }();
  static const bool old_cluster = getenv_flag_jac("RSVD_JACOBI_OLD_CLUSTER");
  const bool use_gcl = gcl_from > 0 ? c >= gcl_from : (c > 64 || (c > 32 && want_j == 1));
  // the Gram-block kernel always accumulates J (+20% at w = 250): both factors then stay
  // orthonormal to ~1e-14 (B^T U S^-1 loses u sigma_1 / sigma_j on the trailing triplets, which the
  // full-size C4 Krylov check, k = 100 of l = 120, sees at the 1e-12 level)
  if (use_gcl && !old_cluster)
    return launch_jacobi_gcl(M, ldm, trans, r, c, Ul, S, Vr, scratch, status, st, 1);
  if (r <= 64) return launch_jacobi_small(M, ldm, trans, r, c, Ul, S, Vr, status, st, want_j == 1);
  static const int cl_from = [] {
    const char* e = getenv("RSVD_JACOBI_CLUSTER_FROM");
    return e ? atoi(e) : 129;
  }();
  if (c >= cl_from) return launch_jacobi_cluster(M, ldm, trans, r, c, Ul, S, Vr, scratch, status, st, want_j == 1);
  // 64 < c <= 128: J is accumulated when the caller asks for it (want_j != 0: the normal-matrix
  // and truncation cores, whose trailing vectors must stay orthonormal to rounding — C4's k = 100
  // core, sigma_100 / sigma_1 = 1e-3); otherwise right vectors as B^T U S^-1 (leading triplets)
  want_j = want_j ? 1 : 0;
  const int ce = c + (c & 1);
  if (r <= 128 && !getenv_flag_jac("RSVD_JACOBI_OLD_MID")) {
    static std::atomic<bool> mattr{false};
    if (!mattr) {
      cudaFuncSetAttribute(k_jacobi_mid<8, 16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      cudaFuncSetAttribute(k_jacobi_mid<8, 16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      cudaFuncSetAttribute(k_jacobi_mid<4, 32, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      mattr = true;
    }
    const double tolm = 2.220446049250313e-16 * sqrt((double)r);
    if (want_j) {
      const size_t wb = (size_t)ce * (8 * 16 + 4) * 8, jb = (size_t)ce * ce * 8;
      const int j_in = (wb + jb) <= 220 * 1024 ? 1 : 0;
      const int threads = ((8 * (ce / 2)) + 31) / 32 * 32;
      if (j_in)
        k_jacobi_mid<8, 16, 2><<<1, threads, wb + jb, st>>>(M, ldm, trans, r, c, Ul, S, Vr, scratch, 1, tolm, 60,
                                                            status);
      else
        k_jacobi_mid<8, 16, 1><<<1, threads, wb, st>>>(M, ldm, trans, r, c, Ul, S, Vr, scratch, 0, tolm, 60, status);
    } else {
      const size_t wb = (size_t)ce * (4 * 32 + 4) * 8;
      const int threads = ((4 * (ce / 2)) + 31) / 32 * 32;
      k_jacobi_mid<4, 32, 0><<<1, threads, wb, st>>>(M, ldm, trans, r, c, Ul, S, Vr, scratch, 0, tolm, 60, status);
    }
    return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
  }
  want_j = 1;   // the generic kernel below keeps the previous always-J behaviour
  const size_t wbytes = (size_t)r * ce * 8, jbytes = want_j ? (size_t)ce * ce * 8 : 0;
  const size_t budget = 200 * 1024;
  int w_in = wbytes <= budget ? 1 : 0;
  int j_in = (w_in ? wbytes + jbytes : jbytes) <= budget ? 1 : 0;
  const size_t smem = (w_in ? wbytes : 0) + (j_in ? jbytes : 0);
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_jacobi<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)budget);
    cudaFuncSetAttribute(k_jacobi<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)budget);
    attr = true;
  }
  const double tol = 2.220446049250313e-16 * sqrt((double)r);  // LAPACK dgesvj's CTOL
  if (r <= 128)
    k_jacobi<4><<<1, kJacThreads, smem, st>>>(M, ldm, trans, r, c, Ul, S, Vr, scratch, scratch + kJacMaxC * kJacMaxC,
                                              w_in, j_in, tol, 60, want_j, status);
  else
    k_jacobi<16><<<1, kJacThreads, smem, st>>>(M, ldm, trans, r, c, Ul, S, Vr, scratch, scratch + kJacMaxC * kJacMaxC,
                                               w_in, j_in, tol, 60, want_j, status);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

int launch_jacobi(const double* M, int64_t ldm, int r, int c, double* Ul, double* S, double* Vr, double* scratch,
                  DevStatus* status, cudaStream_t st) {
  return launch_jacobi_t(M, ldm, 0, r, c, Ul, S, Vr, scratch, status, st, 1);
}

// ------------------------------------------------------------------ guarded triangular inverse
// X = R^-1 for upper-triangular R (c x c, col-major), one thread per column j (back substitution
// x_i = -(sum_{t=i+1..j} R_it x_t) / R_ii).  A zero pivot R_ii (a column zeroed by the rank guard,
// whose row is zero too) gives a zero row and column of X: then X is exactly R^+.
__global__ void k_tri_inv(const double* __restrict__ R, int c, double* __restrict__ X) {
  for (int j = threadIdx.x; j < c; j += blockDim.x) {
    double* x = X + (int64_t)j * c;
    for (int i = c - 1; i > j; --i) x[i] = 0.0;
    const double rjj = R[(int64_t)j * c + j];
    x[j] = rjj != 0.0 ? 1.0 / rjj : 0.0;
    for (int i = j - 1; i >= 0; --i) {
      const double rii = R[(int64_t)i * c + i];
      double s = 0.0;
      for (int t = i + 1; t <= j; ++t) s = fma(R[(int64_t)t * c + i], x[t], s);
      x[i] = rii != 0.0 ? -s / rii : 0.0;
    }
  }
}

// The same inverse for c <= 64 with R staged in shared memory and one warp per column j of X,
// column-oriented: b = e_j; for i = j..0: x_i = b_i / R_ii, then b_t -= R_ti x_i (t < i, lanes
// over t, rows t and t + 32 in two registers).  The chain is one shuffle, one division and one
// fma per step (the thread-per-column loop above paid an L2 round trip per dot-product term:
// ~20 us at c = 30).  Zero pivots give zero rows / columns, as above.
__global__ void __launch_bounds__(1024) k_tri_inv_warp(const double* __restrict__ R, int c, double* __restrict__ X) {
  __shared__ double Rs[64 * 65];
  const int ld = c + 1;
  for (int e = threadIdx.x; e < c * c; e += blockDim.x) {
    const int i = e % c, k = e / c;
    Rs[k * ld + i] = R[e];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = threadIdx.x >> 5; j < c; j += nw) {
    double b0 = lane == j ? 1.0 : 0.0, b1 = lane + 32 == j ? 1.0 : 0.0;
    for (int i = j; i >= 0; --i) {
      const double bi = __shfl_sync(0xffffffffu, i < 32 ? b0 : b1, i & 31);
      const double rii = Rs[i * ld + i];
      const double xi = rii != 0.0 ? bi / rii : 0.0;
      if (lane == i) b0 = xi;
      if (lane + 32 == i) b1 = xi;
      if (lane < i) b0 = fma(-Rs[i * ld + lane], xi, b0);
      if (lane + 32 < i) b1 = fma(-Rs[i * ld + lane + 32], xi, b1);
    }
    if (lane < c) X[(int64_t)j * c + lane] = lane <= j ? b0 : 0.0;
    if (lane + 32 < c) X[(int64_t)j * c + lane + 32] = lane + 32 <= j ? b1 : 0.0;
  }
}

int launch_tri_inv(const double* R, int c, double* Rinv, DevStatus* /*status*/, cudaStream_t st) {
  if (c < 1) return RSVD_E_ARG;
  if (c <= 64) {
    k_tri_inv_warp<<<1, 32 * min(c, 32), 0, st>>>(R, c, Rinv);
  } else {
    k_tri_inv<<<1, 128, 0, st>>>(R, c, Rinv);
  }
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

// ------------------------------------------------------------------ pseudo-inverse / scaling
// Tp (w x w) = V diag(s^+) U^T from T = U diag(s) V^T (U, V w x w col-major, s descending);
// s_i <= rcut * s_0 is dropped.  One thread per output entry.
__global__ void k_pinv_svd(const double* __restrict__ U, const double* __restrict__ s,
                           const double* __restrict__ V, int w, double rcut, double* __restrict__ Tp) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= w * w) return;
  const int i = e % w, j = e / w;
  const double cut = rcut * s[0];
  double acc = 0.0;
  for (int t = 0; t < w; ++t) {
    const double st = s[t];
    if (st > cut && st > 0.0) acc = fma(V[(int64_t)t * w + i] / st, U[(int64_t)t * w + j], acc);
  }
  Tp[e] = acc;
}

int launch_pinv_svd(const double* U, const double* s, const double* V, int w, double rcut, double* Tp,
                     cudaStream_t st) {
  k_pinv_svd<<<(w * w + 255) / 256, 256, 0, st>>>(U, s, V, w, rcut, Tp);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

__global__ void k_scale_cols(double* __restrict__ X, int64_t ld, int rows, int cols, const double* __restrict__ d) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int i = e % rows, j = e / rows;
  X[(int64_t)j * ld + i] *= d[j];
}

int launch_scale_cols(double* X, int64_t ld, int rows, int cols, const double* d, cudaStream_t st) {
  if (rows * cols == 0) return RSVD_OK;
  k_scale_cols<<<(rows * cols + 255) / 256, 256, 0, st>>>(X, ld, rows, cols, d);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

// ------------------------------------------------------------------ small dense helpers
__global__ void k_small_gemm(int ta, int tb, int m, int n, int k, const double* __restrict__ A, int64_t lda_,
                             const double* __restrict__ B, int64_t ldb, double* __restrict__ C, int64_t ldc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= m || j >= n) return;
  double s = 0.0;
  // operands loaded 8 k at a time (in flight together), accumulated in k order
  int p = 0;
  for (; p + 8 <= k; p += 8) {
    double a[8], b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a[u] = ta ? A[(int64_t)i * lda_ + p + u] : A[(int64_t)(p + u) * lda_ + i];
      b[u] = tb ? B[(int64_t)(p + u) * ldb + j] : B[(int64_t)j * ldb + p + u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) s = fma(a[u], b[u], s);
  }
  for (; p < k; ++p) {
    const double a = ta ? A[(int64_t)i * lda_ + p] : A[(int64_t)p * lda_ + i];
    const double b = tb ? B[(int64_t)p * ldb + j] : B[(int64_t)j * ldb + p];
    s = fma(a, b, s);
  }
  C[(int64_t)j * ldc + i] = s;
}

int launch_small_gemm(int ta, int tb, int m, int n, int k, const double* A, int64_t lda_, const double* B,
                      int64_t ldb, double* C, int64_t ldc, cudaStream_t st) {
  dim3 grid((unsigned)((m + 127) / 128), (unsigned)n);
  k_small_gemm<<<grid, 128, 0, st>>>(ta, tb, m, n, k, A, lda_, B, ldb, C, ldc);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

__global__ void k_copy_cols(const double* __restrict__ src, int64_t lds, double* __restrict__ dst, int64_t ldd,
                            int64_t rows) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r < rows) dst[(int64_t)c * ldd + r] = src[(int64_t)c * lds + r];
}

int launch_copy_cols(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int cols,
                     cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return RSVD_OK;
  dim3 grid((unsigned)((rows + 255) / 256), (unsigned)cols);
  k_copy_cols<<<grid, 256, 0, st>>>(src, lds, dst, ldd, rows);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

// n-side sharding (rsvd_api.cu Exec::gather_n / reduce_scatter_n): a column-major n x w block F
// (ld ldf) <-> the chunked layout of the collectives, chunk q = global rows [q cs, (q + 1) cs) as
// a column-major cs x w block at buf + q cs w (rows >= n zero in the chunked copy)
__global__ void k_rows_chunk(double* __restrict__ F, int64_t ldf, int64_t n, double* __restrict__ buf, int64_t cs,
                             int w, int64_t total, int to_chunks) {
  const int64_t gr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (gr >= total) return;
  const int64_t q = gr / cs, il = gr - q * cs;
  double* b = buf + q * cs * w + (int64_t)j * cs + il;
  if (to_chunks) *b = gr < n ? F[(int64_t)j * ldf + gr] : 0.0;
  else if (gr < n) F[(int64_t)j * ldf + gr] = *b;
}

int launch_rows_chunk(double* F, int64_t ldf, int64_t n, double* buf, int64_t cs, int nchunks, int w, int to_chunks,
                      cudaStream_t st) {
  const int64_t total = cs * nchunks;
  if (total <= 0 || w <= 0) return RSVD_OK;
  k_rows_chunk<<<dim3((unsigned)((total + 255) / 256), (unsigned)w), 256, 0, st>>>(F, ldf, n, buf, cs, w, total,
                                                                                    to_chunks);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

__global__ void k_fill(double* dst, int64_t n, double v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = v;
}

int launch_fill(double* dst, int64_t count, double v, cudaStream_t st) {
  if (count <= 0) return RSVD_OK;
  k_fill<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(dst, count, v);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

__global__ void k_square(double* S, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) S[i] = S[i] * S[i];
}

int launch_square(double* S, int n, cudaStream_t st) {
  k_square<<<(n + 127) / 128, 128, 0, st>>>(S, n);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

// Block Gram-Schmidt rank guard with a pre-projection reference: column j of X (rows x w) is
// numerically dependent on the previous blocks when its projected remainder is at the rounding
// level of the projection, |x_j|^2 <= tol * ref_j (ref = squared norm before projecting).  Such
// columns are set to exactly zero (they then stay zero through the shifted and the guarded
// Cholesky passes); their count goes to status->deficient.  G: the w x w Gram after projection.
__global__ void k_zero_dep_cols(double* __restrict__ X, int64_t ld, int64_t rows, int w, const double* __restrict__ G,
                                int64_t gstride, const double* __restrict__ ref, double tol, DevStatus* status) {
  const int j = blockIdx.y;
  if (j >= w) return;
  if (!(G[(int64_t)j * gstride] <= tol * ref[j])) return;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    X[(int64_t)j * ld + r] = 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0 && status) atomicAdd(&status->deficient, 1);
}

int launch_zero_dep_cols(double* X, int64_t ld, int64_t rows, int w, const double* G, const double* ref, double tol,
                         DevStatus* status, cudaStream_t st, int64_t gstride) {
  if (rows <= 0 || w <= 0) return RSVD_OK;
  const unsigned bx = (unsigned)std::min<int64_t>((rows + 255) / 256, 64);
  k_zero_dep_cols<<<dim3(bx, (unsigned)w), 256, 0, st>>>(X, ld, rows, w, G, gstride < 0 ? w + 1 : gstride, ref, tol,
                                                          status);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

// squared column norms d[j] = sum_r X(r, j)^2 (the diagonal of X^T X without forming it): one CTA
// per column, fixed-order per-thread sums and a fixed reduction tree (deterministic)
__global__ void __launch_bounds__(256) k_colnorm2(const double* __restrict__ X, int64_t ld, int64_t rows,
                                                  double* __restrict__ d) {
  __shared__ double part[8];
  const int j = blockIdx.x, tid = threadIdx.x;
  const double* x = X + (int64_t)j * ld;
  double s0 = 0.0, s1 = 0.0;
  int64_t r = tid;
  for (; r + 256 < rows; r += 512) {
    const double a = x[r], b = x[r + 256];
    s0 = fma(a, a, s0);
    s1 = fma(b, b, s1);
  }
  if (r < rows) s0 = fma(x[r], x[r], s0);
  double s = warp_sum(s0 + s1);
  if ((tid & 31) == 0) part[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += part[i];
    d[j] = t;
  }
}

int launch_colnorm2(const double* X, int64_t ld, int64_t rows, int w, double* d, cudaStream_t st) {
  if (w <= 0) return RSVD_OK;
  k_colnorm2<<<w, 256, 0, st>>>(X, ld, rows, d);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

// diag of a (w x w) matrix -> vector
__global__ void k_diag(const double* G, int w, double* d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < w) d[i] = G[(int64_t)i * w + i];
}

int launch_diag(const double* G, int w, double* d, cudaStream_t st) {
  k_diag<<<(w + 127) / 128, 128, 0, st>>>(G, w, d);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

}  // namespace rsvd

// ------------------------------------------------------------------ peak probes (roofline denominators)
namespace rsvd {
// FP64 DMMA issue-rate probe: 8 independent accumulator chains per warp, operands in registers.
__global__ void __launch_bounds__(256) k_probe_dmma(double* sink, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) sink[threadIdx.x] = s;
}

// streaming read probe: 128-bit loads, grid-stride, sum into a sink
__global__ void __launch_bounds__(512) k_probe_read(const double2* __restrict__ p, int64_t n2, double* sink) {
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    const double2 v0 = __ldcs(p + i), v1 = __ldcs(p + i + stride), v2 = __ldcs(p + i + 2 * stride),
                  v3 = __ldcs(p + i + 3 * stride);
    acc += v0.x + v0.y + v1.x + v1.y + v2.x + v2.y + v3.x + v3.y;
  }
  for (; i < n2; i += stride) {
    const double2 v = __ldcs(p + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.0) sink[0] = acc;
}

int probe_peaks(int sms, cudaStream_t st, double* dmma_tflops, double* read_gbs) {
  double* sink = nullptr;
  cudaMalloc(&sink, 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  const int blocks = sms * 4;
  k_probe_dmma<<<blocks, 256, 0, st>>>(sink, 100);  // warm-up
  cudaEventRecord(e0, st);
  k_probe_dmma<<<blocks, 256, 0, st>>>(sink, iters);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256.0 * 8.0 * iters * (blocks * 256 / 32);
  *dmma_tflops = flops / (ms * 1e-3) / 1e12;
  // read probe over 4 GiB
  const size_t bytes = (size_t)4 << 30;
  void* buf = nullptr;
  *read_gbs = 0;
  if (cudaMalloc(&buf, bytes) == cudaSuccess) {
    cudaMemsetAsync(buf, 0, bytes, st);
    const int64_t n2 = (int64_t)(bytes / 16);
    k_probe_read<<<sms * 4, 512, 0, st>>>((const double2*)buf, n2, sink);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0, st);
      k_probe_read<<<sms * 4, 512, 0, st>>>((const double2*)buf, n2, sink);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    *read_gbs = (double)bytes / (best * 1e-3) / 1e9;
    cudaFree(buf);
  } else {
    cudaGetLastError();
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  return cudaGetLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}
}  // namespace rsvd

// =====================================================================================
// Fused CholeskyQR pass for w <= 64 (one launch):
//   [apply]  Y_out = Y_in * Rin        (if Rin != null; Rin = R^-1 of the previous pass)
//   [gram]   partial G = Y_out^T Y_out over this CTA's rows  -> slot[blockIdx.x]
//   [finish] the last CTA to arrive sums the slots in fixed order, factors
//            G (+ shift I) = R^T R with the rank guard, and writes R and R^-1.
// Deterministic: every slot is summed in index order by one thread per entry.
// =====================================================================================
namespace rsvd {

#ifdef RSVD_PHASE_TIMING
__device__ unsigned long long g_phase[16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PHASE(i) do { if (threadIdx.x == 0) g_phase[i] = gtimer(); } while (0)
#define CYC(i) do { if (threadIdx.x == 0) g_phase[i] = clock64(); } while (0)
#define PHASE_MAX(i) do { if (threadIdx.x == 0) atomicMax(&g_phase[i], gtimer()); } while (0)
#define PHASE_MIN(i) do { if (threadIdx.x == 0) atomicMin(&g_phase[i], gtimer()); } while (0)
#else
#define PHASE(i) do {} while (0)
#define CYC(i) do {} while (0)
#define PHASE_MAX(i) do {} while (0)
#define PHASE_MIN(i) do {} while (0)
#endif
constexpr int kFW = 64;          // max width of the fused path

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---------------------------------------------------------------------------------------
// CTA-wide guarded Cholesky (upper, G = R^T R) + inverse for w <= 64, in shared memory.
//   S  (col-major, ld w): G on entry (diagonal already shifted), R on exit (upper part)
//   X  (col-major, ld w): scratch, R^-1 on exit
// One barrier per pivot: every thread recomputes the pivot's 1/sqrt; the trailing update uses
// the unscaled row (S(i,k) -= S(j,i) S(j,k) / d_j); rows are scaled at the end.
// ---------------------------------------------------------------------------------------
__device__ void cta_chol_inv(double* S, double* X, int w, const double* ref, double tol, int* defi,
                             double* invd, double* Rout, double* Rinv_out, DevStatus* status) {
  // S, X: col-major with odd leading dimension lw (bank-conflict-free column walks)
  const int lw = w | 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 thread grid over (row i, column k)
  CYC(8);
  for (int j = 0; j < w; ++j) {
    // issue every shared load of this step before the pivot math: the stores below cannot alias
    // them (they touch rows/columns > j only), so nothing serialises behind the rsqrt.
    const double d = S[j * lw + j];
    double sji[4], sjk[4], tg[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = ty + 16 * a;
      sji[a] = (i > j && i < w) ? S[i * lw + j] : 0.0;
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int k = tx + 16 * b;
      sjk[b] = (k > j && k < w) ? S[k * lw + j] : 0.0;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = ty + 16 * a, k = tx + 16 * b;
        tg[a][b] = (i > j && k >= i && k < w) ? S[k * lw + i] : 0.0;
      }
    const bool def = !(d > tol * ref[j]) || !(ref[j] > 0.0);
    const double inv = def ? 0.0 : rsqrt_nr(d);
    if (tid == 0) { defi[j] = def; invd[j] = inv; }
    const double inv2 = inv * inv;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = ty + 16 * a, k = tx + 16 * b;
        if (!def && i > j && k >= i && k < w) S[k * lw + i] = fma(-sji[a] * inv2, sjk[b], tg[a][b]);
      }
    __syncthreads();
  }
  CYC(9);
  // scale rows: R(j,k) = S(j,k) / sqrt(d_j) (k >= j); zero below the diagonal and deficient rows
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = ty + 16 * a;
    if (i < w) {
      const double sc = defi[i] ? 0.0 : invd[i];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int k = tx + 16 * b;
        if (k < w) {
          const double v = (i <= k) ? S[k * lw + i] * sc : 0.0;
          S[k * lw + i] = v;
          Rout[k * w + i] = v;
        }
      }
    }
  }
  __syncthreads();
  CYC(10);
  // X = R^-1 row by row from the bottom: X(i,i) = 1/R(i,i), X(i,j) = -(sum_k R(i,k) X(k,j)) / R(i,i).
  // Four threads share a column j (k split four ways, shuffle-combined) so each chain is short.
  const int j = tid >> 2, part = tid & 3;
  // 1/R(i,i) = 1/sqrt(d_i) * ... : R(i,i) = d_i * invd_i, so 1/R(i,i) = 1 / (d_i invd_i); computed
  // for all i at once (off the row loop's critical path), stored in the ref slot no longer needed
  double* rinvs = const_cast<double*>(ref);
  for (int i = tid; i < w; i += nt) rinvs[i] = defi[i] ? 0.0 : 1.0 / S[i * lw + i];
  __syncthreads();
  for (int i = w - 1; i >= 0; --i) {
    const double rinv = rinvs[i];
    double sacc = 0.0;
    if (j < w && j > i && rinv != 0.0) {
      const double* srow = S + i;          // R(i,k) at srow[k * lw]
      const double* xcol = X + j * lw;     // X(k,j) at xcol[k]
      double s0 = 0.0, s1 = 0.0;
      int k = i + 1 + part;
      for (; k + 4 <= j; k += 8) {
        s0 = fma(srow[k * lw], xcol[k], s0);
        s1 = fma(srow[(k + 4) * lw], xcol[k + 4], s1);
      }
      for (; k <= j; k += 4) s0 = fma(srow[k * lw], xcol[k], s0);
      sacc = s0 + s1;
    }
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
    if (j < w && part == 0) X[j * lw + i] = (j == i) ? rinv : (j > i ? -sacc * rinv : 0.0);
    __syncthreads();
  }
  CYC(11);
  for (int e = tid; e < w * w; e += nt) {
    const int i = e % w, k = e / w;
    Rinv_out[e] = X[k * lw + i];
  }
  if (tid == 0 && status) {
    int cnt = 0;
    for (int jj = 0; jj < w; ++jj) cnt += defi[jj];
    if (cnt) atomicAdd(&status->deficient, cnt);
  }
}

// smem row stride for a w-wide tile: >= 8*ceil(w/8), == 4 (mod 16) so that the m8n8k4 fragment
// loads (8 rows x 4 consecutive columns, or 4 rows x 8 consecutive columns) are conflict free
__host__ __device__ inline int cq_ld(int w) {
  const int wp = (w + 7) / 8 * 8;
  return wp + ((4 - wp % 16) + 16) % 16;
}
constexpr int kChunkBytes = 64 * 1024;   // staged row chunk (and its output buffer)
__host__ __device__ inline int cholqr_chunk_rows(int w) {
  int r = kChunkBytes / (cq_ld(w) * 8);
  r -= r % 8;
  return r < 8 ? 8 : r;
}

// One CholeskyQR pass over rows split among CTAs (each CTA a contiguous chunk):
//   [apply]  O = T * Rin  (T = staged rows of Yin; Rin = R^-1 of the previous pass)  -> Yout
//   [gram]   partial G = O^T O (upper 8x8 tiles by FP64 DMMA)  -> slot[blockIdx.x]
//   [finish] last CTA: fixed-order slot sum, then either the first-order closed form (second
//            pass with |G - I| <= 1e-8) or the guarded Cholesky + inverse.
__global__ void __launch_bounds__(256) k_cholqr_pass(const double* __restrict__ Yin, int64_t ldi,
                                                     double* __restrict__ Yout, int64_t ldo, int64_t rows, int w,
                                                     int64_t rows_per_cta, const double* __restrict__ Rin,
                                                     double* __restrict__ slots, unsigned* counter, double tol,
                                                     double shift_coef, int second_pass, double* __restrict__ Rout,
                                                     double* __restrict__ Rinv_out, DevStatus* status) {
  extern __shared__ double cq_dyn[];
  const int ld = cq_ld(w);
  const int WP = (w + 7) / 8 * 8;
  const int NT = WP / 8;                         // 8-wide tiles per side
  const int CR = cholqr_chunk_rows(w);
  double* T = cq_dyn;                            // CR x ld   (staged input rows)
  double* O = T + CR * ld;                       // CR x ld   (applied rows)
  double* Rs = O + CR * ld;                      // WP x ld   (Rin^T: Rs[n*ld + k] = Rin(k, n))
  __shared__ double refd[kFW], invd[kFW];
  __shared__ int defi[kFW];
  __shared__ unsigned ticket;
  __shared__ int fastpath;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  PHASE_MIN(0);
  const bool apply = Rin != nullptr;
  if (apply)
    for (int n = 0; n < WP; ++n)
      for (int k = tid; k < ld; k += 256) Rs[n * ld + k] = (n < w && k < w && k <= n) ? Rin[n * w + k] : 0.0;
  // this warp's upper-triangle Gram tiles (bi <= bj): tile index q = warp, warp+8, ...
  const int ntiles = NT * (NT + 1) / 2;
  double gacc[5][2];
#pragma unroll
  for (int u = 0; u < 5; ++u) gacc[u][0] = gacc[u][1] = 0.0;
  int tbi[5], tbj[5];
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    int q = warp + 8 * u, bi = 0;
    while (q >= NT - bi && bi < NT) { q -= NT - bi; ++bi; }
    tbi[u] = bi;
    tbj[u] = bi + q;
  }
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  for (int64_t rr = r0; rr < r1; rr += CR) {
    const int nr = (int)min((int64_t)CR, r1 - rr);
    const int nr8 = (nr + 7) & ~7;
    for (int c = 0; c < WP; ++c) {
      const double* src = Yin + (int64_t)c * ldi + rr;
      for (int i = tid; i < nr8; i += 256) {
        if (i < nr && c < w) cp_async8(T + i * ld + c, src + i);
        else T[i * ld + c] = 0.0;
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const double* Gsrc = T;
    if (apply) {
      // O = T Rin: warp takes 8-row m-tiles; all n-tiles per m-tile; K = WP
      for (int mt = warp; mt < nr8 / 8; mt += 8) {
        double oc[8][2];
#pragma unroll
        for (int n = 0; n < 8; ++n) oc[n][0] = oc[n][1] = 0.0;
        for (int k0 = 0; k0 < WP; k0 += 4) {
          const double a = T[(mt * 8 + g) * ld + k0 + t4];
#pragma unroll
          for (int n = 0; n < 8; ++n)
            if (n < NT) dmma(oc[n][0], oc[n][1], a, Rs[(n * 8 + g) * ld + k0 + t4]);
        }
#pragma unroll
        for (int n = 0; n < 8; ++n)
          if (n < NT) {
            const int row = mt * 8 + g, c0 = n * 8 + 2 * t4;
            *reinterpret_cast<double2*>(O + row * ld + c0) = make_double2(oc[n][0], oc[n][1]);
            if (row < nr) {
              if (c0 < w) Yout[(int64_t)c0 * ldo + rr + row] = oc[n][0];
              if (c0 + 1 < w) Yout[(int64_t)(c0 + 1) * ldo + rr + row] = oc[n][1];
            }
          }
      }
      __syncthreads();
      Gsrc = O;
    }
    // Gram tiles: G(bi, bj) += Src[:, bi-block]^T Src[:, bj-block]  (K = rows)
    for (int k0 = 0; k0 < nr8; k0 += 4) {
#pragma unroll
      for (int u = 0; u < 5; ++u) {
        if (warp + 8 * u < ntiles) {
          const double a = Gsrc[(k0 + t4) * ld + tbi[u] * 8 + g];
          const double b = Gsrc[(k0 + t4) * ld + tbj[u] * 8 + g];
          dmma(gacc[u][0], gacc[u][1], a, b);
        }
      }
    }
    __syncthreads();
  }
  double* slot = slots + (int64_t)blockIdx.x * w * w;
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    if (warp + 8 * u < ntiles) {
      const int i = tbi[u] * 8 + g;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = tbj[u] * 8 + 2 * t4 + h;
        if (i < w && j < w) {
          slot[j * w + i] = gacc[u][h];
          slot[i * w + j] = gacc[u][h];
        }
      }
    }
  }
  __threadfence();
  __syncthreads();
  PHASE_MAX(1);
  if (tid == 0) ticket = atomicAdd(counter, 1u);
  __syncthreads();
  if (ticket != gridDim.x - 1) return;
  // ---------------- finisher (last CTA): fixed-order slot sum into S (reuses T)
  __threadfence();
  PHASE(2);
  double* S = T;
  double* X = O;
  const int Gn = gridDim.x;
  for (int e0 = tid; e0 < w * w; e0 += 512) {
    const int e1 = e0 + 256;
    double a[8], b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = b[u] = 0.0;
    int k = 0;
    for (; k + 8 <= Gn; k += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a[u] += __ldcg(&slots[(int64_t)(k + u) * w * w + e0]);
        if (e1 < w * w) b[u] += __ldcg(&slots[(int64_t)(k + u) * w * w + e1]);
      }
    }
    for (; k < Gn; ++k) {
      a[0] += __ldcg(&slots[(int64_t)k * w * w + e0]);
      if (e1 < w * w) b[0] += __ldcg(&slots[(int64_t)k * w * w + e1]);
    }
    S[e0] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    if (e1 < w * w) S[e1] = ((b[0] + b[1]) + (b[2] + b[3])) + ((b[4] + b[5]) + (b[6] + b[7]));
  }
  if (tid == 0) { *counter = 0u; fastpath = second_pass; }
  __syncthreads();
  PHASE(3);
  if (second_pass) {
    // G = Q1^T Q1 = I + E (CholeskyQR's second pass).  With max|E| <= 1e-8 the first-order
    // factor R2 = I + triu(E,1) + diag(E)/2 and R2^-1 = I - triu(E,1) - diag(E)/2 are exact to
    // O(|E|^2) <= 1e-16.  Columns zeroed by the first pass (G_jj == 0) stay zero.
    for (int k = 0; k < w; ++k)
      for (int i = tid; i < w; i += 256) {
        if (S[i * w + i] == 0.0 || S[k * w + k] == 0.0) continue;
        const double E = S[k * w + i] - (i == k ? 1.0 : 0.0);
        if (!(fabs(E) <= 1e-8)) fastpath = 0;
      }
    __syncthreads();
    if (fastpath) {
      int cnt = 0;
      for (int k = 0; k < w; ++k)
        for (int i = tid; i < w; i += 256) {
          const int e = k * w + i;
          const bool dz = S[i * w + i] == 0.0 || S[k * w + k] == 0.0;
          double r = 0.0, ri = 0.0;
          if (!dz && i <= k) {
            const double E = S[e] - (i == k ? 1.0 : 0.0);
            r = (i == k) ? 1.0 + 0.5 * E : E;
            ri = (i == k) ? 1.0 - 0.5 * E : -E;
          }
          Rout[e] = r;
          Rinv_out[e] = ri;
          if (i == k && dz) ++cnt;
        }
      if (cnt && status) atomicAdd(&status->deficient, cnt);
      PHASE(4);
      return;
    }
  }
  // re-layout S to the odd leading dimension used by cta_chol_inv (X as scratch)
  const int lw = w | 1;
  for (int e = tid; e < w * w; e += 256) X[e] = S[e];
  __syncthreads();
  for (int e = tid; e < w * w; e += 256) {
    const int i = e % w, k = e / w;
    S[k * lw + i] = X[e];
  }
  __syncthreads();
  if (tid < 32) {
    double tr = 0.0;
    for (int j = tid; j < w; j += 32) tr += S[j * lw + j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
    const double shift = shift_coef * tr;
    for (int j = tid; j < w; j += 32) {
      refd[j] = S[j * lw + j] + shift;
      S[j * lw + j] += shift;
    }
  }
  __syncthreads();
  cta_chol_inv(S, X, w, refd, tol, defi, invd, Rout, Rinv_out, status);
  PHASE(4);
}

int cholqr_smem_bytes(int w) { return (2 * cholqr_chunk_rows(w) * cq_ld(w) + ((w + 7) / 8 * 8) * cq_ld(w)) * 8; }

int cholqr_pass_ctas(int64_t rows) {
  int64_t g = (rows + 255) / 256;
  if (g > 148) g = 148;
  if (g < 1) g = 1;
  return (int)g;
}

int launch_cholqr_pass(const double* Yin, int64_t ldi, double* Yout, int64_t ldo, int64_t rows, int w,
                       const double* Rin, double* slots, unsigned* counter, double tol, double shift_coef,
                       int second_pass, double* R, double* Rinv, DevStatus* status, cudaStream_t st) {
  if (w < 1 || w > kFW) return RSVD_E_ARG;
  const int G = cholqr_pass_ctas(rows);
  const int64_t rpc = (rows + G - 1) / G;
  const int smem = cholqr_smem_bytes(w);
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_cholqr_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_cholqr_pass<<<G, 256, smem, st>>>(Yin, ldi, Yout, ldo, rows, w, rpc, Rin, slots, counter, tol, shift_coef,
                                      second_pass, R, Rinv, status);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

}  // namespace rsvd

// =====================================================================================
// One-sided Jacobi for small cores (r <= 64 rows, c <= 64 columns): W and J live in shared
// memory, one warp per column pair, round-robin pair table precomputed, rows-per-lane fixed at
// compile time.  The rotation angle t is computed in fp32 from the fp64 ratio (any t gives an
// exactly orthogonal rotation because cs = rsqrt(1 + t^2) and sn = cs t are formed in fp64; an
// approximate angle only leaves a ~1e-7 fraction of the off-diagonal, which the next sweep removes).
// =====================================================================================
namespace rsvd {

// LPP lanes per column pair, RW rows per lane (r <= LPP * RW); WJ: accumulate J (rotations lag one
// round: they touch only J, and the barrier keeps each column's order).  Pair indices are computed
// arithmetically (round-robin, player ce-1 fixed) and W's column stride is padded by 4 doubles to
// spread the banks.  B200: the round is a latency chain (load, dots, butterfly, angle, rotate,
// barrier); the angle uses the approximate fp64 MUFU ops (rcp/rsqrt.approx.f64): any t gives an
// exactly orthogonal rotation because cs = rsqrt(1 + t^2) (full precision) and sn = cs t.
template <int LPP, int RW, int WJ>
__global__ void __launch_bounds__(256) k_jacobi_small(const double* __restrict__ M, int64_t ldm, int trans, int r,
                                                      int c, double* __restrict__ Ul, double* __restrict__ Sv,
                                                      double* __restrict__ Vr, double tol, int max_sweeps,
                                                      DevStatus* status) {
  constexpr int RS = LPP * RW + 4;     // padded column stride of W
  extern __shared__ double jac_dyn[];
  double* W = jac_dyn;                 // 64 x RS
  double* J = jac_dyn + 64 * RS;       // 64 x 64 (WJ); else the input B (64 x RS) for the epilogue
  __shared__ double sval[64];
  __shared__ int srank[64];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int grp = tid / LPP, sl = tid % LPP;       // pair group and its sub-lane
  const unsigned gmask = (LPP == 32 ? 0xffffffffu : ((1u << LPP) - 1u)) << (tid & 31 & ~(LPP - 1));
  const int ce = c + (c & 1);
  const int npairs = ce >> 1, m1 = ce - 1;
  for (int e = tid; e < 64 * RS; e += nt) {
    const int i = e % RS, j = e / RS;
    double v = 0.0;
    if (i < r && j < c) v = trans ? M[(int64_t)i * ldm + j] : M[(int64_t)j * ldm + i];
    W[e] = v;
    if (!WJ) J[e] = v;
  }
  if (WJ)
    for (int e = tid; e < 64 * 64; e += nt) J[e] = ((e & 63) == (e >> 6)) ? 1.0 : 0.0;
  __syncthreads();
  const double tol2 = tol * tol;
  int sweep = 0;
  bool converged = false;
  int pj_p = 0, pj_q = 0, pj_on = 0;
  double pj_cs = 1.0, pj_sn = 0.0;
  auto apply_pending_j = [&]() {
    if (WJ && pj_on) {
      double* jp = J + pj_p * 64;
      double* jq = J + pj_q * 64;
      for (int k = sl; k < ce; k += LPP) {
        const double u = jp[k], v = jq[k];
        jp[k] = pj_cs * u - pj_sn * v;
        jq[k] = pj_sn * u + pj_cs * v;
      }
      pj_on = 0;
    }
  };
  const bool active = grp < npairs;
  for (; sweep < max_sweeps; ++sweep) {
    int rotated = 0, big = 0;
    for (int round = 0; round < m1; ++round) {
      {
        // every lane of every warp runs the round (inactive groups read column 0 and never
        // store): a warp that reaches the group shuffles diverged takes the serialised BRA.DIV
        // path (tools/jac_small_probe.cu: thousands of cycles per round instead of ~100)
        int p, q;
        {
          int pp = round + grp;
          if (pp >= m1) pp -= m1;
          int qq = round - grp;
          if (qq < 0) qq += m1;
          p = grp == 0 ? round : min(pp, qq);
          q = grp == 0 ? m1 : max(pp, qq);
          if (!active) p = q = 0;
        }
        double* wp = W + p * RS;
        double* wq = W + q * RS;
        double x[RW], y[RW];
#pragma unroll
        for (int t = 0; t < RW; ++t) {
          x[t] = wp[sl + LPP * t];
          y[t] = wq[sl + LPP * t];
        }
        double a0 = 0.0, b0 = 0.0, c0 = 0.0, a1 = 0.0, b1 = 0.0, c1 = 0.0;
#pragma unroll
        for (int t = 0; t < RW; t += 2) {
          a0 = fma(x[t], x[t], a0);
          b0 = fma(y[t], y[t], b0);
          c0 = fma(x[t], y[t], c0);
          if (t + 1 < RW) {
            a1 = fma(x[t + 1], x[t + 1], a1);
            b1 = fma(y[t + 1], y[t + 1], b1);
            c1 = fma(x[t + 1], y[t + 1], c1);
          }
        }
        double a = a0 + a1, b = b0 + b1, cc = c0 + c1;
        __syncwarp();
#pragma unroll
        for (int o = LPP / 2; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o, LPP);
          b += __shfl_xor_sync(0xffffffffu, b, o, LPP);
          cc += __shfl_xor_sync(0xffffffffu, cc, o, LPP);
        }
        apply_pending_j();
        if (active && cc * cc > tol2 * (a * b) && cc != 0.0) {
          rotated = 1;
          big |= (cc * cc > 1e-20 * (a * b)) ? 1 : 0;
          // rho = 2c / |b - a|, t = sign(b - a) rho / (1 + sqrt(1 + rho^2)), approximate fp64 MUFU ops
          const double d = b - a;
          double rd, rsq, rt;
          asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(fmax(fabs(d), 1e-300)));
          const double rho = fmin(fmax(2.0 * cc * rd, -1e100), 1e100);
          const double s1 = fma(rho, rho, 1.0);
          asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rsq) : "d"(s1));
          asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rt) : "d"(fma(s1, rsq, 1.0)));
          const double t = (d < 0.0 ? -rho : rho) * rt;
          const double cs = rsqrt_nr(fma(t, t, 1.0));
          const double sn = cs * t;
#pragma unroll
          for (int k = 0; k < RW; ++k) {
            wp[sl + LPP * k] = cs * x[k] - sn * y[k];
            wq[sl + LPP * k] = sn * x[k] + cs * y[k];
          }
          if (WJ) { pj_p = p; pj_q = q; pj_cs = cs; pj_sn = sn; pj_on = 1; }
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) {
      converged = true;
      ++sweep;
      break;
    }
    // quadratic convergence: when no rotation of this sweep had |c| / sqrt(ab) above 1e-10, the
    // off-diagonal left is O(1e-20), far below tol, so the confirming sweep is skipped
    if (!__syncthreads_or(big)) {
      converged = true;
      ++sweep;
      break;
    }
  }
  if (active) apply_pending_j();
  __syncthreads();
  for (int j = grp; j < ce; j += (nt / LPP)) {
    double sacc = 0.0;
#pragma unroll
    for (int t = 0; t < RW; ++t) {
      const double v = W[j * RS + sl + LPP * t];
      sacc = fma(v, v, sacc);
    }
#pragma unroll
    for (int o = LPP / 2; o > 0; o >>= 1) sacc += __shfl_xor_sync(gmask, sacc, o, LPP);
    if (sl == 0) sval[j] = sqrt(sacc);
  }
  __syncthreads();
  for (int j = tid; j < ce; j += nt) {
    const double sj = sval[j];
    int rk = 0;
    for (int i = 0; i < ce; ++i) {
      const double si = sval[i];
      rk += (si > sj) || (si == sj && i < j);
    }
    srank[j] = rk;
  }
  __syncthreads();
  for (int e = tid; e < r * ce; e += nt) {
    const int i = e % r, j = e / r;
    const int rk = srank[j];
    if (rk < c) {
      const double sj = sval[j];
      Ul[(int64_t)rk * r + i] = sj > 0.0 ? W[j * RS + i] / sj : 0.0;
    }
  }
  if (WJ) {
    for (int e = tid; e < c * ce; e += nt) {
      const int i = e % c, j = e / c;
      const int rk = srank[j];
      if (rk < c) Vr[(int64_t)rk * c + i] = J[j * 64 + i];
    }
  } else {
    // right vectors from the left ones: B = W J^T with W = U S  ->  J = B^T U S^-1 (B = the
    // input as seen by the sweep, staged in the J area).  Accurate to ~u sigma_1 / sigma_j, i.e.
    // for the leading triplets the algorithms use (the rsvd_core_svd primitive accumulates J
    // instead).  4 x 2 register blocks (a, j) from shared memory.
    const double* Bs = J;
    const int na = (c + 3) / 4, nj = ce / 2;
    for (int e = tid; e < na * nj; e += nt) {
      const int a0 = 4 * (e % na), j0 = 2 * (e / na);
      double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      for (int i = 0; i < r; ++i) {
        const double w0 = W[j0 * RS + i], w1 = W[(j0 + 1) * RS + i];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double bb = Bs[min(a0 + u, 63) * RS + i];
          acc[u][0] = fma(bb, w0, acc[u][0]);
          acc[u][1] = fma(bb, w1, acc[u][1]);
        }
      }
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int j = j0 + v, rk = srank[j];
        if (rk >= c) continue;
        const double sj = sval[j];
        const double inv = sj > 0.0 ? 1.0 / (sj * sj) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (a0 + u < c) Vr[(int64_t)rk * c + a0 + u] = acc[u][v] * inv;
      }
    }
  }
  for (int j = tid; j < ce; j += nt)
    if (srank[j] < c) Sv[srank[j]] = sval[j];
  if (tid == 0 && status) {
    status->jacobi_sweeps = sweep;
    if (!converged) atomicAdd(&status->jacobi_fail, 1);
  }
}

int launch_jacobi_small(const double* M, int64_t ldm, int trans, int r, int c, double* Ul, double* S, double* Vr,
                        DevStatus* status, cudaStream_t st, int want_j) {
  if (c < 1 || c > 64 || r < c || r > 64) return RSVD_E_ARG;
  const int ce = c + (c & 1);
  const double tol = 2.220446049250313e-16 * sqrt((double)r);
  const int smem = 2 * 64 * (64 + 4) * 8;  // W and J (or the staged input B), stride <= 68
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_jacobi_small<8, 4, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_jacobi_small<8, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_jacobi_small<4, 16, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_jacobi_small<4, 16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  // measured on B200 (tools/jac_small_probe.cu): r <= 32 -> 8 lanes x 4 rows per pair,
  // r <= 64 -> 4 lanes x 16 rows (one warp per SMSP; 8 x 8 was 10-20% slower)
  if (r <= 32) {
    const int threads = ((8 * (ce / 2)) + 31) / 32 * 32;
    if (want_j) k_jacobi_small<8, 4, 1><<<1, threads, smem, st>>>(M, ldm, trans, r, c, Ul, S, Vr, tol, 60, status);
    else k_jacobi_small<8, 4, 0><<<1, threads, smem, st>>>(M, ldm, trans, r, c, Ul, S, Vr, tol, 60, status);
  } else {
    const int threads = ((4 * (ce / 2)) + 31) / 32 * 32;
    if (want_j) k_jacobi_small<4, 16, 1><<<1, threads, smem, st>>>(M, ldm, trans, r, c, Ul, S, Vr, tol, 60, status);
    else k_jacobi_small<4, 16, 0><<<1, threads, smem, st>>>(M, ldm, trans, r, c, Ul, S, Vr, tol, 60, status);
  }
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

}  // namespace rsvd

#ifdef RSVD_PHASE_TIMING
namespace rsvd {
void read_phases(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_phase, sizeof(unsigned long long) * 16); }
void reset_phases() {
  unsigned long long init[16];
  for (int i = 0; i < 16; ++i) init[i] = (i == 0) ? ~0ull : 0ull;
  cudaMemcpyToSymbol(g_phase, init, sizeof(init));
}
}  // namespace rsvd
#endif

// ------------------------------------------------------------------ Nystrom helpers (Alg. 4)
namespace rsvd {
namespace {
// out[0] = 2.2e-16 * sqrt(lambda_max(G)) for the symmetric psd G (w x w): ||Y_r||_2 from its
// Gram by power iteration (fixed 200 iterations, Rayleigh quotient; deterministic), line 9.
__global__ void __launch_bounds__(256) k_nys_nu(const double* __restrict__ G, int w, double* __restrict__ out) {
  __shared__ double x[512], y[512], red[8];
  const int tid = threadIdx.x;
  for (int i = tid; i < w; i += 256) x[i] = 1.0 + 1e-3 * i;   // generic start, not orthogonal to the top space
  __syncthreads();
  double rq = 0.0;
  for (int it = 0; it < 200; ++it) {
    for (int i = tid; i < w; i += 256) {
      double s = 0.0;
      for (int k = 0; k < w; ++k) s = fma(G[(int64_t)k * w + i], x[k], s);
      y[i] = s;
    }
    __syncthreads();
    double nn = 0.0, xy = 0.0;
    for (int i = tid; i < w; i += 256) { nn = fma(y[i], y[i], nn); xy = fma(x[i], y[i], xy); }
    nn = warp_sum(nn);
    xy = warp_sum(xy);
    if ((tid & 31) == 0) { red[tid >> 5] = nn; }
    __syncthreads();
    double tn = 0.0;
    for (int q = 0; q < 8; ++q) tn += red[q];
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = xy;
    __syncthreads();
    double txy = 0.0;
    for (int q = 0; q < 8; ++q) txy += red[q];
    double txx = 0.0;
    for (int k = 0; k < w; ++k) txx = fma(x[k], x[k], txx);
    rq = (txx > 0.0) ? txy / txx : 0.0;
    const double sc = tn > 0.0 ? rsqrt(tn) : 0.0;
    __syncthreads();
    for (int i = tid; i < w; i += 256) x[i] = y[i] * sc;
    __syncthreads();
  }
  if (tid == 0) out[0] = 2.2e-16 * sqrt(fmax(rq, 0.0));
}
// Y += nu * Q  (column-major rows x w), nu read from device memory
__global__ void k_axpy_dev(double* __restrict__ Y, int64_t ldy, const double* __restrict__ Q, int64_t ldq, int64_t rows,
                           int w, const double* __restrict__ nu) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r < rows && c < w) Y[(int64_t)c * ldy + r] = fma(nu[0], Q[(int64_t)c * ldq + r], Y[(int64_t)c * ldy + r]);
}
// S (w x w) = (B + B^T) / 2
__global__ void k_symmetrize(const double* __restrict__ B, int w, double* __restrict__ S) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= w * w) return;
  const int i = e % w, j = e / w;
  S[e] = 0.5 * (B[e] + B[(int64_t)i * w + j]);
}
// lam2[i] = max(lam[i]^2 - nu, 0)   (line 15); lam2 may alias lam
__global__ void k_nys_eig(const double* lam, int k, const double* __restrict__ nu, double* lam2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) lam2[i] = fmax(lam[i] * lam[i] - nu[0], 0.0);
}
}  // namespace

int launch_nys_nu(const double* G, int w, double* out, cudaStream_t st) {
  if (w < 1 || w > 512) return RSVD_E_ARG;
  k_nys_nu<<<1, 256, 0, st>>>(G, w, out);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}
int launch_axpy_dev(double* Y, int64_t ldy, const double* Q, int64_t ldq, int64_t rows, int w, const double* nu,
                    cudaStream_t st) {
  if (rows <= 0 || w <= 0) return RSVD_OK;
  k_axpy_dev<<<dim3((unsigned)((rows + 255) / 256), (unsigned)w), 256, 0, st>>>(Y, ldy, Q, ldq, rows, w, nu);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}
int launch_symmetrize(const double* B, int w, double* S, cudaStream_t st) {
  k_symmetrize<<<(w * w + 255) / 256, 256, 0, st>>>(B, w, S);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}
int launch_nys_eig(const double* lam, int k, const double* nu, double* lam2, cudaStream_t st) {
  k_nys_eig<<<(k + 255) / 256, 256, 0, st>>>(lam, k, nu, lam2);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}
}  // namespace rsvd

namespace rsvd {
namespace {
__global__ void k_sub_cols(const double* __restrict__ T, int64_t ldt, double* __restrict__ out, int64_t ldo,
                           int64_t rows, int c) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (r < rows && j < c) out[(int64_t)j * ldo + r] -= T[(int64_t)j * ldt + r];
}
__global__ void k_add_cols(const double* __restrict__ T, int64_t ldt, double* __restrict__ out, int64_t ldo,
                           int64_t rows, int c) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (r < rows && j < c) out[(int64_t)j * ldo + r] += T[(int64_t)j * ldt + r];
}
}  // namespace
int launch_add_cols(const double* T, int64_t ldt, double* out, int64_t ldo, int64_t rows, int c, cudaStream_t st) {
  if (rows <= 0 || c <= 0) return RSVD_OK;
  k_add_cols<<<dim3((unsigned)((rows + 255) / 256), (unsigned)c), 256, 0, st>>>(T, ldt, out, ldo, rows, c);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}
int launch_sub_cols(const double* T, int64_t ldt, double* out, int64_t ldo, int64_t rows, int c, cudaStream_t st) {
  if (rows <= 0 || c <= 0) return RSVD_OK;
  k_sub_cols<<<dim3((unsigned)((rows + 255) / 256), (unsigned)c), 256, 0, st>>>(T, ldt, out, ldo, rows, c);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}
}  // namespace rsvd
