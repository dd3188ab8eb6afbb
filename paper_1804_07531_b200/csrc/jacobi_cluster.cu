// Core SVD (tsvd of the w x w core; Alg. 9) for cores too
// wide for one CTA's shared memory (64 < w <= 512): block one-sided (Hestenes) Jacobi on a
// thread-block cluster.
//
// W = M (r x c, zero-padded to nb*b columns) lives in global memory (L2 resident, <= 2 MB).
// The nb = 2C column blocks of b columns are paired by a round-robin tournament; in each block
// round cluster CTA k loads its block pair (2b columns) into shared memory, runs one cyclic
// sweep of plane rotations over those 2b columns (round-robin, one warp per column pair),
// writes the pair back in place and meets the other CTAs at a cluster barrier.  2C-1 block
// rounds make one outer sweep, in which every column pair of W meets at least once; outer
// sweeps repeat until no pair needed a rotation (|w_p.w_q| <= tol |w_p||w_q|, tol = sqrt(r) u,
// LAPACK dgesvj's threshold — the same test as the one-CTA kernels).
// Deterministic: fixed pairing and summation order, independent of timing.
// Outputs as the other Jacobi kernels: sigma_j = |W_j| sorted descending, Ul = W_j / sigma_j,
// Vr = J (want_j, rotations accumulated in global memory) or Vr = B^T Ul S^-1.
#include <atomic>
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace rsvd {
namespace {

constexpr int kMaxC = 512;
constexpr int kThreads = 512;   // 16 warps: one per column pair of a 32-column block pair

__device__ __forceinline__ void pair_of(int round, int k, int n, int* p, int* q) {
  // round-robin tournament on n (even) players, round in [0, n-1), pair k in [0, n/2)
  int a, b;
  if (k == 0) {
    a = round;
    b = n - 1;
  } else {
    a = (round + k) % (n - 1);
    b = (round - k + (n - 1)) % (n - 1);
  }
  *p = a < b ? a : b;
  *q = a < b ? b : a;
}


template <int RPL>
__global__ void __launch_bounds__(kThreads, 1)
    k_jacobi_cluster(const double* __restrict__ M, int64_t ldm, int trans, int r, int c, int b, int nb,
                     double* __restrict__ Ul, double* __restrict__ Sv, double* __restrict__ Vr,
                     double* __restrict__ W, double* __restrict__ J, int ldj, double* __restrict__ sval_g,
                     int* __restrict__ flags, double tol, int max_sweeps, int want_j, DevStatus* status) {
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  extern __shared__ double sW[];          // 2b columns x r rows (column j at sW[j * r])
  __shared__ int s_rot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = kThreads / 32;
  const int ncol = nb * b;                 // padded column count
  // ---- W = B (B = M or M^T), zero-padded; J = I
  for (int64_t e = (int64_t)rank * kThreads + tid; e < (int64_t)r * ncol; e += (int64_t)C * kThreads) {
    const int i = (int)(e % r), j = (int)(e / r);
    double v = 0.0;
    if (j < c) v = trans ? M[(int64_t)i * ldm + j] : M[(int64_t)j * ldm + i];
    W[e] = v;
  }
  if (want_j)
    for (int64_t e = (int64_t)rank * kThreads + tid; e < (int64_t)ncol * ldj; e += (int64_t)C * kThreads) {
      const int i = (int)(e % ldj), j = (int)(e / ldj);
      J[e] = (i == j) ? 1.0 : 0.0;
    }
  if (rank == 0 && tid == 0) flags[0] = flags[1] = 0;
  __threadfence();
  cluster.sync();

  const int b2 = 2 * b;
  int sweep = 0;
  bool converged = false;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) s_rot = 0;
    int rotated = 0;
    for (int br = 0; br < nb - 1; ++br) {
      int P, Q;
      pair_of(br, rank, nb, &P, &Q);
      // load blocks P, Q -> local columns [0, b) and [b, 2b): column loops, 8 loads in flight
      for (int lj0 = 0; lj0 < b2; lj0 += 8)
        for (int i = tid; i < r; i += kThreads) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int lj = lj0 + u;
            const int gj = (lj < b ? P * b + lj : Q * b + (lj - b));
            v[u] = (lj < b2) ? W[(int64_t)gj * r + i] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (lj0 + u < b2) sW[(lj0 + u) * r + i] = v[u];
        }
      __syncthreads();
      // one cyclic sweep over the 2b local columns
      for (int ir = 0; ir < b2 - 1; ++ir) {
        for (int pk = warp; pk < b; pk += nwarp) {
          int p, q;
          pair_of(ir, pk, b2, &p, &q);
          double* wp = sW + p * r;
          double* wq = sW + q * r;
          // the lane's slice of both columns in registers: every load is issued before any
          // store (a load -> rotate -> store loop serialises on the possible aliasing)
          double x[RPL], y[RPL];   // RPL = rows per lane (r <= 32 RPL)
#pragma unroll
          for (int t = 0; t < RPL; ++t) {
            const int i = lane + 32 * t;
            x[t] = (i < r) ? wp[i] : 0.0;
            y[t] = (i < r) ? wq[i] : 0.0;
          }
          double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0, c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int t = 0; t < RPL; t += 2) {
            a0 = fma(x[t], x[t], a0);
            b0 = fma(y[t], y[t], b0);
            c0 = fma(x[t], y[t], c0);
            a1 = fma(x[t + 1], x[t + 1], a1);
            b1 = fma(y[t + 1], y[t + 1], b1);
            c1 = fma(x[t + 1], y[t + 1], c1);
          }
          double a = a0 + a1, bb = b0 + b1, cc = c0 + c1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            bb += __shfl_xor_sync(0xffffffffu, bb, o);
            cc += __shfl_xor_sync(0xffffffffu, cc, o);
          }
          if (cc != 0.0 && cc * cc > tol * tol * (a * bb)) {
            // rho = 2c / |b - a|, t = sign(b - a) rho / (1 + sqrt(1 + rho^2)) from the approximate
            // fp64 MUFU ops: any t gives an exactly orthogonal rotation (cs full precision)
            const double d = bb - a;
            double rd, rsq, rt;
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(fmax(fabs(d), 1e-300)));
            const double rho = fmin(fmax(2.0 * cc * rd, -1e100), 1e100);
            const double s1 = fma(rho, rho, 1.0);
            asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rsq) : "d"(s1));
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rt) : "d"(fma(s1, rsq, 1.0)));
            const double t = (d < 0.0 ? -rho : rho) * rt;
            const double cs = rsqrt(fma(t, t, 1.0));
            const double sn = cs * t;
#pragma unroll
            for (int k = 0; k < RPL; ++k) {
              const int i = lane + 32 * k;
              if (i < r) {
                wp[i] = cs * x[k] - sn * y[k];
                wq[i] = sn * x[k] + cs * y[k];
              }
            }
            if (want_j) {
              const int gp = p < b ? P * b + p : Q * b + (p - b);
              const int gq = q < b ? P * b + q : Q * b + (q - b);
              double* jp = J + (int64_t)gp * ldj;
              double* jq = J + (int64_t)gq * ldj;
              for (int i = lane; i < ncol; i += 32) {
                const double x = jp[i], y = jq[i];
                jp[i] = cs * x - sn * y;
                jq[i] = sn * x + cs * y;
              }
            }
            rotated = 1;
          }
          __syncwarp();
        }
        __syncthreads();
      }
      // write the pair back in place (each block is owned by exactly one CTA per block round)
      for (int lj = 0; lj < b2; ++lj) {
        const int gj = (lj < b ? P * b + lj : Q * b + (lj - b));
        for (int i = tid; i < r; i += kThreads) W[(int64_t)gj * r + i] = sW[lj * r + i];
      }
      __threadfence();
      cluster.sync();
    }
    // convergence: OR of every CTA's rotation flag (flags[sweep & 1], reset one sweep ahead)
    if (rotated) s_rot = 1;
    __syncthreads();
    if (tid == 0) {
      if (s_rot) atomicOr(&flags[sweep & 1], 1);
      if (rank == 0) flags[(sweep + 1) & 1] = 0;
    }
    __threadfence();
    cluster.sync();
    const int any = *((volatile int*)&flags[sweep & 1]);
    cluster.sync();  // everyone has read the flag before it is reset next sweep
    if (!any) {
      converged = true;
      ++sweep;
      break;
    }
  }
  // ---- singular values (column norms), descending ranks, outputs
  for (int j = rank * nwarp + warp; j < ncol; j += C * nwarp) {
    const double* wj = W + (int64_t)j * r;
    double s = 0.0;
    for (int i = lane; i < r; i += 32) s = fma(wj[i], wj[i], s);
    s = warp_sum(s);
    if (lane == 0) sval_g[j] = sqrt(s);
  }
  __threadfence();
  cluster.sync();
  for (int j = rank * kThreads + tid; j < ncol; j += C * kThreads) {
    const double sj = sval_g[j];
    int rk = 0;
    for (int i = 0; i < ncol; ++i) {
      const double si = sval_g[i];
      rk += (si > sj) || (si == sj && i < j);
    }
    if (rk < c) {
      Sv[rk] = sj;
      reinterpret_cast<int*>(sval_g + kMaxC)[rk] = j;  // rank -> column
    }
  }
  __threadfence();
  cluster.sync();
  const int* col_of = reinterpret_cast<const int*>(sval_g + kMaxC);
  for (int64_t e = (int64_t)rank * kThreads + tid; e < (int64_t)r * c; e += (int64_t)C * kThreads) {
    const int i = (int)(e % r), rk = (int)(e / r);
    const int j = col_of[rk];
    const double sj = sval_g[j];
    Ul[(int64_t)rk * r + i] = sj > 0.0 ? W[(int64_t)j * r + i] / sj : 0.0;
  }
  if (want_j) {
    for (int64_t e = (int64_t)rank * kThreads + tid; e < (int64_t)c * c; e += (int64_t)C * kThreads) {
      const int i = (int)(e % c), rk = (int)(e / c);
      Vr[(int64_t)rk * c + i] = J[(int64_t)col_of[rk] * ldj + i];
    }
  } else {
    // right vectors from the left ones (B = W J^T, W = U S  ->  J = B^T U S^-1), leading triplets
    for (int64_t e = (int64_t)rank * kThreads + tid; e < (int64_t)c * c; e += (int64_t)C * kThreads) {
      const int a = (int)(e % c), rk = (int)(e / c);
      const int j = col_of[rk];
      const double sj = sval_g[j];
      double s = 0.0;
      if (sj > 0.0)
        for (int i = 0; i < r; ++i) {
          const double bia = trans ? M[(int64_t)i * ldm + a] : M[(int64_t)a * ldm + i];
          s = fma(bia, W[(int64_t)j * r + i], s);
        }
      Vr[(int64_t)rk * c + a] = sj > 0.0 ? s / (sj * sj) : 0.0;
    }
  }
  if (rank == 0 && tid == 0 && status) {
    status->jacobi_sweeps = sweep;
    if (!converged) atomicAdd(&status->jacobi_fail, 1);
  }
}

}  // namespace

// scratch (doubles) needed by launch_jacobi_cluster
int64_t jacobi_cluster_scratch(int r, int c) {
  (void)c;
  return (int64_t)r * kMaxC + (int64_t)kMaxC * kMaxC + 2 * kMaxC + 64;
}

int launch_jacobi_cluster(const double* M, int64_t ldm, int trans, int r, int c, double* Ul, double* S, double* Vr,
                          double* scratch, DevStatus* status, cudaStream_t st, int want_j) {
  if (c < 1 || c > kMaxC || r < c || r > kMaxC) return RSVD_E_ARG;
  const int C = c <= 256 ? 8 : 16;
  const int nb = 2 * C;
  const int b = (c + nb - 1) / nb;      // <= 16
  const int ncol = nb * b;
  double* W = scratch;
  double* J = W + (int64_t)r * kMaxC;
  double* sval = J + (int64_t)kMaxC * kMaxC;
  int* flags = reinterpret_cast<int*>(sval + 2 * kMaxC);
  const size_t smem = (size_t)2 * b * r * 8;
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_jacobi_cluster<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 16 * kMaxC * 8);
    cudaFuncSetAttribute(k_jacobi_cluster<8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_jacobi_cluster<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 16 * kMaxC * 8);
    cudaFuncSetAttribute(k_jacobi_cluster<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const double tol = 2.220446049250313e-16 * sqrt((double)r);
  // rows per lane as a compile-time count: r <= 256 -> 8 (C3's 140, C5's 250), else 16
  cudaError_t e = (r <= 256)
      ? cudaLaunchKernelEx(&cfg, k_jacobi_cluster<8>, M, ldm, trans, r, c, b, nb, Ul, S, Vr, W, J, ncol, sval, flags,
                           tol, 60, want_j, status)
      : cudaLaunchKernelEx(&cfg, k_jacobi_cluster<16>, M, ldm, trans, r, c, b, nb, Ul, S, Vr, W, J, ncol, sval,
                           flags, tol, 60, want_j, status);
  return e == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

}  // namespace rsvd
