// Matrix-view kernels: the hot path of the pass-efficient randomized SVD (§4, §6, §7).
//
//   k_view_ax   Y = A X        range view          (Alg. 2 line 4 "A Q_r", Alg. 7 line 3a, Alg. 9 line 4)
//   k_view_aty  Z = A^T Y      co-range view       (Alg. 2 line 6 "A^* Q_c", Alg. 7 line 3b, Alg. 9 line 5)
//   k_view_fused  Y_c = A Omega and Y_r = A^T Phi from ONE read of every A tile (Alg. 7 line 3 a)+b))
//
// A is row-major (m x n, lda).  All tall-skinny operands are column-major ("each vector
// contiguous"): X^T is w x n, Y^T is w x m, with leading dimensions >= rows.  Tiles of A and of
// the skinny operands are staged by TMA (128B swizzle) through an mbarrier ring and consumed
// by FP64 DMMA (mma.sync m8n8k4) — sm_100 has no tcgen05 f64 kind.  One producer warp issues
// TMA; 8 consumer warps issue DMMA.  CTAs are persistent and walk "units" (a block of output
// rows x a range of the reduction dimension); each unit writes its partial result to its own
// slot so that the cross-unit sum is done later in a fixed order (bitwise deterministic).
#include <atomic>
#include "common.cuh"
#include "internal.h"

#include <cudaTypedefs.h>

#include <algorithm>

namespace rsvd {

constexpr int kNW = 8;             // consumer warps
constexpr int kThreads = (kNW + 1) * 32;
constexpr int kBK = 32;            // reduction-dimension elements per pipeline stage
constexpr int kSmemBudget = 200 * 1024;
constexpr int kNG = 4;             // n-tiles per B-fragment group
// k-loop unroll (of the 4 k-steps per stage) by width: unrolling lets the next step's fragment
// loads overlap the current DMMAs.  4 everywhere except WT 9..12, where two 8-row m-tiles per warp
// (MT = 2) double the accumulators and a full unroll spills.  Measured against the earlier
// 4/2/1 policy (tools/view_probe_ab.py): C3 20000 x 8000 w = 140 views -5%, C2 w = 60/120 -2/-3%.
template <int WT>
struct KUnroll { static constexpr int v = (WT >= 9 && WT <= 12) ? 2 : 4; };

// 1024-byte aligned base of the dynamic shared memory (128B-swizzled TMA tiles need it), formed by
// pointer arithmetic on the __shared__ array: an integer round trip (uintptr_t) would lose the
// address space and turn every operand load into a generic LD.E with 64-bit address math.
__device__ __forceinline__ uint8_t* smem_base_1024(uint8_t* raw) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(raw));
  return raw + ((1024u - (a & 1023u)) & 1023u);
}

// Per-CTA %globaltimer stamps of k_view_ax for tools/view_timeline.cu (compiled out otherwise):
// [0] start, [1] first stage consumed (warp 0), [2 + i] end of the CTA's unit i (warp 0, i < 6), [8] end.
#ifdef RSVD_VIEW_TIMING
__device__ unsigned long long g_view_t[160][9];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define VT(i) do { if (threadIdx.x == 0 && blockIdx.x < 160) g_view_t[blockIdx.x][i] = gtimer(); } while (0)
#else
#define VT(i) do {} while (0)
#endif

// =====================================================================================
// Y = A X     (M = rows of A, K = n, N = w)
// =====================================================================================
template <int WT>
struct AxCfg {
  static constexpr int MT = WT > 12 ? 1 : 2;   // 8-row MMA tiles per warp (register budget 168)
  static constexpr int BM = kNW * MT * 8;      // 128 rows per unit
  static constexpr int WP = WT * 8;            // padded width
  static constexpr int A_STAGE = BM * kBK * 8; // two 16-col boxes of BM x 128 B
  static constexpr int X_STAGE = WP * kBK * 8; // two 16-col boxes of WP x 128 B
  static constexpr int STAGE = A_STAGE + X_STAGE;
  static constexpr int STAGES = (kSmemBudget / STAGE) > 6 ? 6 : (kSmemBudget / STAGE);
  static constexpr int SMEM = STAGES * STAGE + 1024 + 2 * STAGES * 8;
};

template <int WT>
__global__ void __launch_bounds__(kThreads, 1)
    k_view_ax(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
              double* __restrict__ out, int64_t ldo, int64_t slot_stride, int rows, int w, int RB, int S,
              int KT, int KTS, int a_keep) {
  using C = AxCfg<WT>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_base_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  VT(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int U = RB * S;

  if (warp == kNW) {  // ---------------- TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmX);
      const uint64_t pa = a_keep ? policy_evict_last() : policy_evict_first(), px = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < U; u += gridDim.x) {
        const int rb = u / S, s = u % S;
        const int kt0 = s * KTS, kt1 = min(KT, kt0 + KTS);
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * C::STAGE;
          mbar_arrive_expect_tx(&full[stage], C::STAGE);
          const int k0 = kt * kBK;
          tma_load_2d(st, &tmA, &full[stage], k0, rb * C::BM, pa);
          tma_load_2d(st + C::BM * 128, &tmA, &full[stage], k0 + 16, rb * C::BM, pa);
          tma_load_2d(st + C::A_STAGE, &tmX, &full[stage], k0, 0, px);
          tma_load_2d(st + C::A_STAGE + C::WP * 128, &tmX, &full[stage], k0 + 16, 0, px);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  // ---------------- DMMA consumers
  const int g = lane >> 2, t = lane & 3, pg = perm8(g);
  double acc[C::MT][WT][2];
  int stage = 0;
  uint32_t phase = 0;
#ifdef RSVD_VIEW_TIMING
  int nu = 0;
#endif
  for (int u = blockIdx.x; u < U; u += gridDim.x) {
    const int rb = u / S, s = u % S;
    const int kt0 = s * KTS, kt1 = min(KT, kt0 + KTS);
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < WT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    for (int kt = kt0; kt < kt1; ++kt) {
      mbar_wait(&full[stage], phase);
#ifdef RSVD_VIEW_TIMING
      if (nu == 0 && kt == kt0) VT(1);
#endif
      const uint8_t* As = smem + stage * C::STAGE;
      const uint8_t* Xs = As + C::A_STAGE;
#pragma unroll (KUnroll<WT>::v)
      for (int kk = 0; kk < 4; ++kk) {   // 4 x 8 k per stage; thread t owns k = 8kk + {2t, 2t+1}
        const int box = kk >> 1;
        const uint32_t q = ((kk & 1) << 2) + t;
        double2 a[C::MT];
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt)
          a[mt] = *reinterpret_cast<const double2*>(As + box * C::BM * 128 + sw128(warp * C::MT * 8 + mt * 8 + pg, q));
        // n-tiles in groups of kNG: bounds the live B fragments; x- then y-halves give
        // MT*kNG independent DMMAs between dependent ones
#pragma unroll
        for (int n0 = 0; n0 < WT; n0 += kNG) {
          double2 b[kNG];
#pragma unroll
          for (int j = 0; j < kNG; ++j)
            if (n0 + j < WT) b[j] = *reinterpret_cast<const double2*>(Xs + box * C::WP * 128 + sw128((n0 + j) * 8 + pg, q));
#pragma unroll
          for (int j = 0; j < kNG; ++j)
#pragma unroll
            for (int mt = 0; mt < C::MT; ++mt)
              if (n0 + j < WT) dmma(acc[mt][n0 + j][0], acc[mt][n0 + j][1], a[mt].x, b[j].x);
#pragma unroll
          for (int j = 0; j < kNG; ++j)
#pragma unroll
            for (int mt = 0; mt < C::MT; ++mt)
              if (n0 + j < WT) dmma(acc[mt][n0 + j][0], acc[mt][n0 + j][1], a[mt].y, b[j].y);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    // epilogue: fragment (g, 2t / 2t+1) of tile (mt, nt) is Y[row perm8(g)][col t / 4+t]
    double* o = out + (int64_t)s * slot_stride;
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt) {
      const int r = rb * C::BM + warp * C::MT * 8 + mt * 8 + pg;
      if (r < rows) {
#pragma unroll
        for (int nt = 0; nt < WT; ++nt) {
          const int c0 = nt * 8 + t, c1 = c0 + 4;
          if (c0 < w) o[(int64_t)c0 * ldo + r] = acc[mt][nt][0];
          if (c1 < w) o[(int64_t)c1 * ldo + r] = acc[mt][nt][1];
        }
      }
    }
#ifdef RSVD_VIEW_TIMING
    if (nu < 6) VT(2 + nu);
    ++nu;
#endif
  }
  VT(8);
}

// =====================================================================================
// Z = A^T Y   (M = n (columns of A), K = rows of A, N = w)
// =====================================================================================
template <int WT>
struct AtyCfg {
  static constexpr int MT = WT > 12 ? 1 : 2;
  static constexpr int BN = kNW * MT * 8;        // 128 columns of A per unit
  static constexpr int WP = WT * 8;
  static constexpr int A_STAGE = kBK * BN * 8;   // BN/16 boxes of kBK x 128 B
  static constexpr int Y_STAGE = WP * kBK * 8;
  static constexpr int STAGE = A_STAGE + Y_STAGE;
  static constexpr int STAGES = (kSmemBudget / STAGE) > 6 ? 6 : (kSmemBudget / STAGE);
  static constexpr int SMEM = STAGES * STAGE + 1024 + 2 * STAGES * 8;
};

template <int WT>
__global__ void __launch_bounds__(kThreads, 1)
    k_view_aty(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmY,
               double* __restrict__ out, int64_t ldo, int64_t slot_stride, int ncols, int w, int CB, int S,
               int KT, int KTS) {
  using C = AtyCfg<WT>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_base_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int U = CB * S;

  if (warp == kNW) {
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmY);
      const uint64_t pa = policy_evict_first(), py = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < U; u += gridDim.x) {
        const int cb = u / S, s = u % S;
        const int kt0 = s * KTS, kt1 = min(KT, kt0 + KTS);
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * C::STAGE;
          mbar_arrive_expect_tx(&full[stage], C::STAGE);
          const int r0 = kt * kBK;
#pragma unroll
          for (int b = 0; b < C::BN / 16; ++b)
            tma_load_2d(st + b * kBK * 128, &tmA, &full[stage], cb * C::BN + b * 16, r0, pa);
          tma_load_2d(st + C::A_STAGE, &tmY, &full[stage], r0, 0, py);
          tma_load_2d(st + C::A_STAGE + C::WP * 128, &tmY, &full[stage], r0 + 16, 0, py);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  const int g = lane >> 2, t = lane & 3, pg = perm8(g);
  double acc[C::MT][WT][2];
  int stage = 0;
  uint32_t phase = 0;
  for (int u = blockIdx.x; u < U; u += gridDim.x) {
    const int cb = u / S, s = u % S;
    const int kt0 = s * KTS, kt1 = min(KT, kt0 + KTS);
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < WT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    for (int kt = kt0; kt < kt1; ++kt) {
      mbar_wait(&full[stage], phase);
      const uint8_t* As = smem + stage * C::STAGE;
      const uint8_t* Ys = As + C::A_STAGE;
#pragma unroll (KUnroll<WT>::v)
      for (int kk = 0; kk < 4; ++kk) {
        const int r0 = kk * 8 + 2 * t;     // rows of A (the reduction index) this thread feeds
        const int boxy = kk >> 1;
        const uint32_t q = ((kk & 1) << 2) + t;
        double a0[C::MT], a1[C::MT];
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) {
          const int c = warp * C::MT * 8 + mt * 8 + g;  // column of A inside the unit
          const uint8_t* base = As + (c >> 4) * kBK * 128 + ((c & 1) << 3);
          const uint32_t ch = (c & 15) >> 1;
          a0[mt] = *reinterpret_cast<const double*>(base + sw128(r0, ch));
          a1[mt] = *reinterpret_cast<const double*>(base + sw128(r0 + 1, ch));
        }
#pragma unroll
        for (int n0 = 0; n0 < WT; n0 += kNG) {
          double2 b[kNG];
#pragma unroll
          for (int j = 0; j < kNG; ++j)
            if (n0 + j < WT) b[j] = *reinterpret_cast<const double2*>(Ys + boxy * C::WP * 128 + sw128((n0 + j) * 8 + pg, q));
#pragma unroll
          for (int j = 0; j < kNG; ++j)
#pragma unroll
            for (int mt = 0; mt < C::MT; ++mt)
              if (n0 + j < WT) dmma(acc[mt][n0 + j][0], acc[mt][n0 + j][1], a0[mt], b[j].x);
#pragma unroll
          for (int j = 0; j < kNG; ++j)
#pragma unroll
            for (int mt = 0; mt < C::MT; ++mt)
              if (n0 + j < WT) dmma(acc[mt][n0 + j][0], acc[mt][n0 + j][1], a1[mt], b[j].y);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    double* o = out + (int64_t)s * slot_stride;
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt) {
      const int col = cb * C::BN + warp * C::MT * 8 + mt * 8 + g;
      if (col < ncols) {
#pragma unroll
        for (int nt = 0; nt < WT; ++nt) {
          const int c0 = nt * 8 + t, c1 = c0 + 4;
          if (c0 < w) o[(int64_t)c0 * ldo + col] = acc[mt][nt][0];
          if (c1 < w) o[(int64_t)c1 * ldo + col] = acc[mt][nt][1];
        }
      }
    }
  }
}

// =====================================================================================
// Fused single-pass sketch: from each A tile (kBK rows x BN cols) read once,
//   Y_r[BN cols] += A_tile^T Phi[tile rows]     (accumulated in registers over the unit)
//   Y_c[tile rows] (+)= A_tile Omega[BN cols]   (per-tile partial, flushed every stage)
// Units are (column strip sb, row split s).  Y_r partials go to slot s, Y_c partials go to slot
// sb (deterministic mode) or are red.global.add-ed into one buffer (atomic mode).
// =====================================================================================
template <int L2T>
struct FusedCfg {
  static constexpr int BN = kNW * 8;            // 64 columns per strip (1 MMA tile per warp)
  static constexpr int LTMAX = 9;               // l <= 72
  static constexpr int L2P = L2T * 8;
  static constexpr int LPMAX = LTMAX * 8;
  static constexpr int A_STAGE = kBK * BN * 8;  // 4 boxes of kBK x 128 B (16 KB)
  static constexpr int P_STAGE = L2P * kBK * 8; // Phi^T tile, 2 boxes
  static constexpr int STAGE = A_STAGE + P_STAGE;
  static constexpr int OM_BYTES = LPMAX * BN * 8;  // Omega^T strip, 4 boxes of LP x 128 B
  static constexpr int STAGES = ((kSmemBudget - OM_BYTES) / STAGE) > 5 ? 5 : ((kSmemBudget - OM_BYTES) / STAGE);
  static constexpr int SMEM = STAGES * STAGE + OM_BYTES + 1024 + (2 * STAGES + 4) * 8;
};

// Shared-memory plan for one (L2T, LTC) instance: the Omega^T strip is sized by LTC (LP <= 16 LTC)
// and double-buffered when that still leaves 4 pipeline stages, so the next unit's strip is
// loaded while the current unit runs (otherwise every unit start waits one TMA round trip).
template <int L2T, int LTC>
struct FusedPlan {
  using B = FusedCfg<L2T>;
  static constexpr int OM_ONE = (LTC * 16 < B::LPMAX ? LTC * 16 : B::LPMAX) * B::BN * 8;
  static constexpr int OM_BUFS = (kSmemBudget - 2 * OM_ONE) / B::STAGE >= 4 ? 2 : 1;
  static constexpr int OM_BYTES = OM_BUFS * OM_ONE;
  static constexpr int ST = (kSmemBudget - OM_BYTES) / B::STAGE;
  static constexpr int STAGES = ST > 5 ? 5 : ST;
  static constexpr int SMEM = STAGES * B::STAGE + OM_BYTES + 1024 + (2 * STAGES + 4) * 8;
  static_assert(OM_ONE % 1024 == 0 && B::STAGE % 1024 == 0, "128B-swizzled TMA tiles need 1024 B alignment");
  static_assert(STAGES >= 2 && SMEM <= 227 * 1024, "fused shared-memory plan");
};

// LTC: Y_c n-tiles per warp (warp groups 0/1 take n-tiles g, g+2, ...; LTC = ceil(LT/2)) — a
// compile-time count, because predicated-off DMMAs still take issue slots
template <int L2T, int LTC>
__global__ void __launch_bounds__(kThreads, 1)
    k_view_fused(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmOm,
                 const __grid_constant__ CUtensorMap tmPhi, double* __restrict__ yc, int64_t ldyc,
                 int64_t yc_slot_stride, int yc_atomic, double* __restrict__ yr, int64_t ldyr,
                 int64_t yr_slot_stride, int rows, int ncols, int l, int LP, int l2, int NSB, int S, int KT,
                 int KTS) {
  using C = FusedCfg<L2T>;
  using P = FusedPlan<L2T, LTC>;
  constexpr int STAGES = P::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_base_1024(smem_raw);
  uint8_t* om0 = smem + STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(om0 + P::OM_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* om_full = empty + STAGES;   // [P::OM_BUFS]
  uint64_t* om_empty = om_full + 2;     // [P::OM_BUFS]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNW);
    }
    for (int b = 0; b < P::OM_BUFS; ++b) {
      mbar_init(&om_full[b], 1);
      mbar_init(&om_empty[b], kNW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int U = NSB * S;
  const int OM_TX = LP * C::BN * 8;

  if (warp == kNW) {
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmOm);
      tma_prefetch_desc(&tmPhi);
      const uint64_t pa = policy_evict_first(), pk = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0, ophase = 0;
      int ob = 0;
      for (int u = blockIdx.x; u < U; u += gridDim.x) {
        const int sb = u / S, s = u % S;
        // Omega^T strip for this unit (LP rows x BN cols) into buffer ob, released by the
        // consumers at unit end; with two buffers it is issued one unit ahead
        mbar_wait(&om_empty[ob], ophase ^ 1);
        mbar_arrive_expect_tx(&om_full[ob], OM_TX);
        uint8_t* om = om0 + ob * P::OM_ONE;
#pragma unroll
        for (int b = 0; b < C::BN / 16; ++b)
          tma_load_2d(om + b * LP * 128, &tmOm, &om_full[ob], sb * C::BN + b * 16, 0, pk);
        if (++ob == P::OM_BUFS) { ob = 0; ophase ^= 1; }
        const int kt0 = s * KTS, kt1 = min(KT, kt0 + KTS);
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * C::STAGE;
          mbar_arrive_expect_tx(&full[stage], C::STAGE);
          const int r0 = kt * kBK;
#pragma unroll
          for (int b = 0; b < C::BN / 16; ++b)
            tma_load_2d(st + b * kBK * 128, &tmA, &full[stage], sb * C::BN + b * 16, r0, pa);
          tma_load_2d(st + C::A_STAGE, &tmPhi, &full[stage], r0, 0, pk);
          tma_load_2d(st + C::A_STAGE + C::L2P * 128, &tmPhi, &full[stage], r0 + 16, 0, pk);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  const int g = lane >> 2, t = lane & 3, pg = perm8(g);
  const int LT = LP >> 3;
  // Y_c work split per stage: warp -> m-tile (warp & 3) of the 4 row tiles, n-tiles j = (warp>>2) + 2i
  // from a provably warp-uniform warp index, so the Y_c tile predicate below (nt < LT) is uniform
  // and the predicated mma.sync needs no WARPSYNC
  const int warp_u = __shfl_sync(0xffffffffu, warp, 0);
  const int yc_mt = warp_u & 3;
  const int yc_n0 = warp_u >> 2;
  double accr[L2T][2];
  int stage = 0;
  uint32_t phase = 0, ophase = 0;
  int ob = 0;
  for (int u = blockIdx.x; u < U; u += gridDim.x) {
    const int sb = u / S, s = u % S;
    const int kt0 = s * KTS, kt1 = min(KT, kt0 + KTS);
#pragma unroll
    for (int nt = 0; nt < L2T; ++nt) accr[nt][0] = accr[nt][1] = 0.0;
    mbar_wait(&om_full[ob], ophase);
    const uint8_t* om = om0 + ob * P::OM_ONE;
    for (int kt = kt0; kt < kt1; ++kt) {
      mbar_wait(&full[stage], phase);
      const uint8_t* As = smem + stage * C::STAGE;
      const uint8_t* Ps = As + C::A_STAGE;
      // Y_c first: its short dependent DMMA chain and its partial stores overlap the Y_r DMMAs
      // that follow (both k-loops fully unrolled: 113 -> 112 us, and 127 -> 113 us for the unroll)
      // ---- Y_c(tile rows) = A_tile Omega_strip  (ax pattern; K = BN = 64 -> 8 double-steps)
      {
        double accc[LTC][2];
#pragma unroll
        for (int i = 0; i < LTC; ++i) accc[i][0] = accc[i][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < C::BN / 8; ++kk) {
          const int box = kk >> 1;
          const uint32_t q = ((kk & 1) << 2) + t;
          const double2 a = *reinterpret_cast<const double2*>(As + box * kBK * 128 + sw128(yc_mt * 8 + pg, q));
          double2 b[LTC];
#pragma unroll
          for (int i = 0; i < LTC; ++i) {
            const int nt = yc_n0 + 2 * i;
            if (nt < LT) b[i] = *reinterpret_cast<const double2*>(om + box * LP * 128 + sw128(nt * 8 + pg, q));
          }
#pragma unroll
          for (int i = 0; i < LTC; ++i)
            if (yc_n0 + 2 * i < LT) dmma(accc[i][0], accc[i][1], a.x, b[i].x);
#pragma unroll
          for (int i = 0; i < LTC; ++i)
            if (yc_n0 + 2 * i < LT) dmma(accc[i][0], accc[i][1], a.y, b[i].y);
        }

        const int r = kt * kBK + yc_mt * 8 + pg;
        if (r < rows) {
          double* o = yc + (yc_atomic ? 0 : (int64_t)sb * yc_slot_stride);
#pragma unroll
          for (int i = 0; i < LTC; ++i) {
            const int nt = yc_n0 + 2 * i;
            if (nt < LT) {
              const int c0 = nt * 8 + t, c1 = c0 + 4;
              if (yc_atomic) {
                if (c0 < l) atomicAdd(&o[(int64_t)c0 * ldyc + r], accc[i][0]);
                if (c1 < l) atomicAdd(&o[(int64_t)c1 * ldyc + r], accc[i][1]);
              } else {
                if (c0 < l) o[(int64_t)c0 * ldyc + r] = accc[i][0];
                if (c1 < l) o[(int64_t)c1 * ldyc + r] = accc[i][1];
              }
            }
          }
        }
      }
      // ---- Y_r += A_tile^T Phi_tile  (aty pattern; this warp owns A columns warp*8 + g)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int r0 = kk * 8 + 2 * t;
        const int c = warp * 8 + g;
        const uint8_t* base = As + (c >> 4) * kBK * 128 + ((c & 1) << 3);
        const uint32_t ch = (c & 15) >> 1;
        const double a0 = *reinterpret_cast<const double*>(base + sw128(r0, ch));
        const double a1 = *reinterpret_cast<const double*>(base + sw128(r0 + 1, ch));
        const uint32_t q = ((kk & 1) << 2) + t;
        const uint8_t* pb = Ps + (kk >> 1) * C::L2P * 128;
#pragma unroll
        for (int n0 = 0; n0 < L2T; n0 += kNG) {
          double2 b[kNG];
#pragma unroll
          for (int j = 0; j < kNG; ++j)
            if (n0 + j < L2T) b[j] = *reinterpret_cast<const double2*>(pb + sw128((n0 + j) * 8 + pg, q));
#pragma unroll
          for (int j = 0; j < kNG; ++j)
            if (n0 + j < L2T) dmma(accr[n0 + j][0], accr[n0 + j][1], a0, b[j].x);
#pragma unroll
          for (int j = 0; j < kNG; ++j)
            if (n0 + j < L2T) dmma(accr[n0 + j][0], accr[n0 + j][1], a1, b[j].y);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&om_empty[ob]);
    if (++ob == P::OM_BUFS) { ob = 0; ophase ^= 1; }
    double* o = yr + (int64_t)s * yr_slot_stride;
    const int col = sb * C::BN + warp * 8 + g;
    if (col < ncols) {
#pragma unroll
      for (int nt = 0; nt < L2T; ++nt) {
        const int c0 = nt * 8 + t, c1 = c0 + 4;
        if (c0 < l2) o[(int64_t)c0 * ldyr + col] = accr[nt][0];
        if (c1 < l2) o[(int64_t)c1 * ldyr + col] = accr[nt][1];
      }
    }
  }
}

// =====================================================================================
// host side
// =====================================================================================
namespace {

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool get_encoder() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || fn == nullptr)
    return false;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

// 2-D fp64 tensor map over a row-major [outer x inner] array with row stride ld (elements),
// box = 16 inner elements (128 B, swizzled) x box_outer rows.
int make_map(CUtensorMap* map, const double* base, int64_t inner, int64_t outer, int64_t ld, int box_outer) {
  if (!get_encoder()) return RSVD_E_CUDA;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {16u, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? RSVD_OK : RSVD_E_CUDA;
}

// Choose the reduction split S for `nblk` output blocks of `kt` stage-tiles each so that the
// busiest persistent CTA's critical path (in tiles, + per-unit overhead) is minimal.
void choose_split(int nblk, int kt, int grid_cap, int max_split, int* S_out, int* KTS_out) {
  double best = 1e30;
  int bS = 1, bK = kt;
  for (int S = 1; S <= std::min(kt, max_split); ++S) {
    const int kts = (kt + S - 1) / S;
    const int s2 = (kt + kts - 1) / kts;
    const long U = (long)nblk * s2;
    const long G = std::min<long>(U, grid_cap);
    const long per = (U + G - 1) / G;
    const double cost = per * (kts + 2.5);
    if (cost < best - 1e-9) { best = cost; bS = s2; bK = kts; }
  }
  *S_out = bS;
  *KTS_out = bK;
}

template <int WT>
int launch_ax_t(const ViewArgs& a, cudaStream_t st) {
  using C = AxCfg<WT>;
  CUtensorMap tmA, tmX;
  if (make_map(&tmA, a.A, a.n, a.rows, a.lda, C::BM) || make_map(&tmX, a.X, a.n, a.w, a.ldx, C::WP))
    return RSVD_E_CUDA;
  const int RB = (int)((a.rows + C::BM - 1) / C::BM);
  const int KT = (int)((a.n + kBK - 1) / kBK);
  const int U = RB * a.S;
  const int grid = std::min(U, a.grid_cap);
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_view_ax<WT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  k_view_ax<WT><<<grid, kThreads, C::SMEM, st>>>(tmA, tmX, a.out, a.ldo, a.slot_stride, (int)a.rows, a.w, RB, a.S, KT,
                                                   a.KTS, a.a_keep);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

template <int WT>
int launch_aty_t(const ViewArgs& a, cudaStream_t st) {
  using C = AtyCfg<WT>;
  CUtensorMap tmA, tmY;
  if (make_map(&tmA, a.A, a.n, a.rows, a.lda, kBK) || make_map(&tmY, a.X, a.rows, a.w, a.ldx, C::WP))
    return RSVD_E_CUDA;
  const int CB = (int)((a.n + C::BN - 1) / C::BN);
  const int KT = (int)((a.rows + kBK - 1) / kBK);
  const int U = CB * a.S;
  const int grid = std::min(U, a.grid_cap);
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_view_aty<WT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  k_view_aty<WT><<<grid, kThreads, C::SMEM, st>>>(tmA, tmY, a.out, a.ldo, a.slot_stride, (int)a.n, a.w, CB, a.S, KT,
                                                    a.KTS);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

template <int L2T, int LTC>
int launch_fused_t(const FusedArgs& a, cudaStream_t st) {
  using C = FusedCfg<L2T>;
  const int LP = ((a.l + 7) / 8) * 8;
  CUtensorMap tmA, tmOm, tmPhi;
  if (make_map(&tmA, a.A, a.n, a.rows, a.lda, kBK) || make_map(&tmOm, a.Om, a.n, a.l, a.ldom, LP) ||
      make_map(&tmPhi, a.Phi, a.rows, a.l2, a.ldphi, C::L2P))
    return RSVD_E_CUDA;
  const int NSB = (int)((a.n + C::BN - 1) / C::BN);
  const int KT = (int)((a.rows + kBK - 1) / kBK);
  const int U = NSB * a.S;
  const int grid = std::min(U, a.grid_cap);
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_view_fused<L2T, LTC>, cudaFuncAttributeMaxDynamicSharedMemorySize, FusedPlan<L2T, LTC>::SMEM);
    attr = true;
  }
  k_view_fused<L2T, LTC><<<grid, kThreads, FusedPlan<L2T, LTC>::SMEM, st>>>(tmA, tmOm, tmPhi, a.yc, a.ldyc, a.yc_slot_stride, a.yc_atomic,
                                                       a.yr, a.ldyr, a.yr_slot_stride, (int)a.rows, (int)a.n, a.l,
                                                       LP, a.l2, NSB, a.S, KT, a.KTS);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

template <int... Is>
struct Seq {};

template <template <int> class F, typename Args, int... Is>
int dispatch(int WT, const Args& a, cudaStream_t st, Seq<Is...>) {
  int r = RSVD_E_ARG;
  ((WT == Is + 1 ? (r = F<Is + 1>::run(a, st), 0) : 0), ...);
  return r;
}

template <int WT>
struct AxRun { static int run(const ViewArgs& a, cudaStream_t st) { return launch_ax_t<WT>(a, st); } };
template <int WT>
struct AtyRun { static int run(const ViewArgs& a, cudaStream_t st) { return launch_aty_t<WT>(a, st); } };
template <int LTC>
struct FusedRunL {
  template <int L2T>
  struct R { static int run(const FusedArgs& a, cudaStream_t st) { return launch_fused_t<L2T, LTC>(a, st); } };
};

}  // namespace

// Plan the split of a view so that partial slots can be sized by the caller.
void plan_view(int kind, int64_t rows, int64_t n, int w, int grid_cap, int* S, int* KTS) {
  const int bm = ((w + 7) / 8 > 12) ? 64 : 128;
  if (kind == VIEW_AX) {
    const int RB = (int)((rows + bm - 1) / bm);
    const int KT = (int)((n + kBK - 1) / kBK);
    // one or two row blocks (a tall-skinny Gram X^T X as a view of X^T): split the long reduction
    // over every SM rather than 64 of them
    choose_split(RB, KT, grid_cap, RB <= 2 ? grid_cap : 64, S, KTS);
  } else if (kind == VIEW_ATY) {
    const int CB = (int)((n + bm - 1) / bm);
    const int KT = (int)((rows + kBK - 1) / kBK);
    choose_split(CB, KT, grid_cap, 64, S, KTS);
  } else {
    const int NSB = (int)((n + 63) / 64);
    const int KT = (int)((rows + kBK - 1) / kBK);
    choose_split(NSB, KT, grid_cap, 64, S, KTS);
  }
}

int launch_view_ax(const ViewArgs& a, cudaStream_t st) {
  const int WT = (a.w + 7) / 8;
  if (WT < 1 || WT > kMaxWT) return RSVD_E_ARG;
  return dispatch<AxRun>(WT, a, st, Seq<0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15>{});
}

int launch_view_aty(const ViewArgs& a, cudaStream_t st) {
  const int WT = (a.w + 7) / 8;
  if (WT < 1 || WT > kMaxWT) return RSVD_E_ARG;
  return dispatch<AtyRun>(WT, a, st, Seq<0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15>{});
}

int launch_view_fused(const FusedArgs& a, cudaStream_t st) {
  const int L2T = (a.l2 + 7) / 8;
  if (a.l < 1 || a.l > kFusedMaxL || L2T < 1 || L2T > kFusedMaxL2T) return RSVD_E_ARG;
  using S18 = Seq<0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17>;
  const int LTC = ((a.l + 7) / 8 + 1) / 2;  // 1..5 (l <= 72)
  switch (LTC) {
    case 1: return dispatch<FusedRunL<1>::template R>(L2T, a, st, S18{});
    case 2: return dispatch<FusedRunL<2>::template R>(L2T, a, st, S18{});
    case 3: return dispatch<FusedRunL<3>::template R>(L2T, a, st, S18{});
    case 4: return dispatch<FusedRunL<4>::template R>(L2T, a, st, S18{});
    default: return dispatch<FusedRunL<5>::template R>(L2T, a, st, S18{});
  }
}

}  // namespace rsvd

namespace rsvd {
int fused_strips(int64_t n) { return (int)((n + FusedCfg<1>::BN - 1) / FusedCfg<1>::BN); }
}  // namespace rsvd
