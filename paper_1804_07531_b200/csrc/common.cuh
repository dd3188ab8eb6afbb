// Device-side building blocks shared by the rsvd kernels (sm_100a only).
//
//   * mbarrier + TMA (cp.async.bulk.tensor) producer/consumer pipeline primitives
//   * FP64 DMMA (mma.sync m8n8k4 .f64) — the only FP64 tensor-core path on sm_100
//     (tcgen05 has no f64 kind)
//   * the 128-byte TMA swizzle address map
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "rsvd kernels are written for sm_100a only"
#endif

namespace rsvd {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
// 2-D tiled load: box at (c0 = inner coordinate, c1 = outer coordinate) -> smem, completes
// transaction bytes on `bar`.  Out-of-bounds elements are zero-filled (and still counted).
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Byte offset of 16-byte chunk `chunk` (0..7) of row `row` inside a box whose rows are 128 B
// and which TMA wrote with CU_TENSOR_MAP_SWIZZLE_128B (box base 1024-B aligned): the chunk
// index is XOR-ed with (row mod 8).
__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t chunk) {
  return (row << 7) + ((chunk ^ (row & 7u)) << 4);
}

// ---------------------------------------------------------------- FP64 tensor core
// D(8x8) += A(8x4, row) * B(4x8, col).  Thread (g = lane>>2, t = lane&3) holds
// a = A[g][t], b = B[t][g], d0/d1 = D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Row permutation inside an 8-row MMA tile that makes the 128-bit fragment loads from
// 128B-swizzled tiles bank-conflict free: fragment row g lives in smem row perm8(g), so the
// quarter-warp {g=2i, g=2i+1} touches smem rows {i, i+4} whose swizzled chunks are disjoint.
__device__ __forceinline__ int perm8(int g) { return ((g & 1) << 2) | (g >> 1); }

// 1/sqrt(x) for x > 0 in fp64 without the IEEE div/sqrt subroutines: fp32 seed (scaled into
// range by a power of two) + two Newton steps (relative error ~1e-16).
__device__ __forceinline__ double fast_rsqrt(double x) {
  const int e = ilogb(x) & ~1;                 // even exponent so sqrt scales exactly
  const double xs = ldexp(x, -e);              // xs in [1, 4)
  double y = (double)rsqrtf((float)xs);
  y = y * fma(-0.5 * xs, y * y, 1.5);
  y = y * fma(-0.5 * xs, y * y, 1.5);
  return ldexp(y, -e / 2);
}
// 1/x in fp64: fp32 seed of the scaled value + two Newton steps
__device__ __forceinline__ double fast_rcp(double x) {
  const int e = ilogb(x);
  const double xs = ldexp(x, -e);              // |xs| in [1, 2)
  double y = (double)(1.0f / (float)xs);
  y = y * fma(-xs, y, 2.0);
  y = y * fma(-xs, y, 2.0);
  return ldexp(y, -e);
}

// 1/sqrt(d), d > 0 normal: the MUFU seed (rsqrt.approx.f64, ~2^-22) and one third-order Newton
// step (~2^-64 before rounding) — a short dependent chain, no slow-path branch of the IEEE rsqrt
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-d * y, y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace rsvd

#include "internal.h"
namespace rsvd {
// CholeskyQR's second pass: the Gram of an already nearly orthonormal block is G = I + E with tiny
// E.  When max |E| <= 1e-8 over the non-zero columns, R = I + triu(E, 1) + diag(E) / 2 and
// R^-1 = I - triu(E, 1) - diag(E) / 2 to O(|E|^2) = O(u); columns with a zero Gram diagonal (zeroed
// by an earlier guard) stay zero and count as deficient.  Called by every thread of the block with
// uniform arguments; returns true (R, Rinv written) when the closed form applies.
__device__ __forceinline__ bool chol_near_identity(const double* __restrict__ G, int w, double* __restrict__ R,
                                                   double* __restrict__ Rinv, DevStatus* status, int* s_flag) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) *s_flag = 1;
  __syncthreads();
  for (int e = tid; e < w * w; e += nt) {
    const int i = e % w, k = e / w;
    if (G[(int64_t)i * w + i] != 0.0 && G[(int64_t)k * w + k] != 0.0) {
      const double E = G[e] - (i == k ? 1.0 : 0.0);
      if (!(fabs(E) <= 1e-8)) *s_flag = 0;
    }
  }
  __syncthreads();
  if (!*s_flag) return false;
  int ndef = 0;
  for (int e = tid; e < w * w; e += nt) {
    const int i = e % w, k = e / w;
    const bool dz = G[(int64_t)i * w + i] == 0.0 || G[(int64_t)k * w + k] == 0.0;
    double r = 0.0, ri = 0.0;
    if (!dz && i <= k) {
      const double E = G[e] - (i == k ? 1.0 : 0.0);
      r = (i == k) ? 1.0 + 0.5 * E : E;
      ri = (i == k) ? 1.0 - 0.5 * E : -E;
    }
    R[e] = r;
    Rinv[e] = ri;
    if (i == k && G[e] == 0.0) ++ndef;
  }
  if (status && ndef) atomicAdd(&status->deficient, ndef);
  return true;
}
}  // namespace rsvd
