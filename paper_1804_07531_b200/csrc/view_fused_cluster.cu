// Fused single-pass sketch for wide sketches (l <= 128, l2 <= 256; C4's 120 / 240), fp64:
//   Y_c = A Omega  and  Y_r = A^T Phi  from ONE read of every A tile (Alg. 7 line 3 a)+b), P:667-669,
//   P:684 "performed independently in parallel").
//
// Thread-block cluster of CL CTAs (16, or 8 for narrow A).  CTA `rank` of the cluster owns one
// 64-column strip of A; the cluster covers CL adjacent strips (a strip group) and walks a row
// range of A in 16-row tiles.  Per tile, every CTA:
//   * Y_r[strip columns] += A_tile^T Phi_tile      (FP64 DMMA, accumulated in registers over the
//                                                   row range: no partial traffic);
//   * P = A_tile Omega_strip   (16 x l partial of Y_c over the strip's 64 columns) into its shared
//     memory, then the CL partials of the tile are summed ACROSS the cluster through distributed
//     shared memory: CTA `rank` reduces 16 / CL rows, reading them from the CL CTAs in rank order
//     (deterministic), and writes the reduced rows to the strip group's Y_c partial slot.
// So the Y_c partials leave the chip once per strip group (CL x 64 columns) instead of once per
// strip: partial traffic l / (64 CL) of A's bytes (C4: 0.12x written + 0.12x read back) instead of
// l / 64 (1.9x).  The partial buffers are double-buffered; mbarriers signalled remotely
// (mbarrier.arrive.release.cluster) say "partial ready" and "partial consumed".  The slots are
// summed in group order afterwards (k_slot_sum_rows), the Y_r row-split slots in split order.
#include <atomic>
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace rsvd {
namespace {

constexpr int kFNW = 8;                    // consumer warps
constexpr int kFThreads = (kFNW + 1) * 32; // + one TMA producer warp
constexpr int kFBK = 16;                   // rows of A per stage
constexpr int kFBN = 64;                   // columns per CTA strip
constexpr int kFSmem = 218 * 1024;

template <int L2T, int LTC>
struct FcPlan {
  static constexpr int L2P = L2T * 8;
  static constexpr int LPM = LTC * 32;                   // l padded to the warps' n-tile coverage (4 groups x LTC tiles)
  static constexpr int A_STAGE = kFBK * kFBN * 8;        // 4 boxes of 16 rows x 128 B
  static constexpr int P_STAGE = L2P * 128;              // Phi^T tile: L2P rows of 16 doubles
  static constexpr int STAGE = A_STAGE + P_STAGE;
  static constexpr int OM = LPM * 128 * 4;               // Omega^T strip: 4 boxes of LPM rows x 128 B
  static constexpr int PB = kFBK * LPM * 8;              // one Y_c partial buffer (16 rows x LPM, row-major)
  static constexpr int STAGES = (kFSmem - OM - 2 * PB - 512) / STAGE > 4 ? 4 : (kFSmem - OM - 2 * PB - 512) / STAGE;
  static constexpr int SMEM = STAGES * STAGE + OM + 2 * PB + 1024 + 512;
  static_assert(STAGES >= 2, "fused cluster plan needs two stages");
  static_assert(A_STAGE % 1024 == 0 && STAGE % 1024 == 0 && OM % 1024 == 0, "1024-B aligned swizzled tiles");
};

__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ double ld_dsmem(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Units: u = (strip group g, row split s), g = u / S.  Rows of split s: tiles [s KTS, (s+1) KTS).
template <int L2T, int LTC>
__global__ void __launch_bounds__(kFThreads, 1)
    k_view_fused_cl(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmOm,
                    const __grid_constant__ CUtensorMap tmPhi, double* __restrict__ yc_slots, int64_t ldys,
                    int64_t yc_slot_stride, double* __restrict__ yr, int64_t ldyr, int64_t yr_slot_stride, int rows,
                    int ncols, int l, int l2, int NG, int S, int KT, int KTS) {
  using P = FcPlan<L2T, LTC>;
  constexpr int STAGES = P::STAGES;
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int ncl = gridDim.x / CL, cid = blockIdx.x / CL;
  extern __shared__ uint8_t fc_raw[];
  uint8_t* smem = fc_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(fc_raw)) & 1023u)) & 1023u);
  uint8_t* om = smem + STAGES * P::STAGE;
  double* pbuf = reinterpret_cast<double*>(om + P::OM);         // [2][16][LPM]
  uint64_t* bars = reinterpret_cast<uint64_t*>(om + P::OM + 2 * P::PB);
  uint64_t* full = bars;
  uint64_t* empty = full + STAGES;
  uint64_t* om_full = empty + STAGES;
  uint64_t* om_empty = om_full + 1;
  uint64_t* pready = om_empty + 1;   // [2]: the CL partials of a tile are in the buffers
  uint64_t* pfree = pready + 2;      // [2]: the CL CTAs have read this CTA's buffer
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kFNW);
    }
    mbar_init(om_full, 1);
    mbar_init(om_empty, kFNW);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&pready[b], CL);
      mbar_init(&pfree[b], CL);
    }
    fence_barrier_init();
  }
  __syncthreads();
  cluster_sync_all();   // peers' mbarriers are initialised before any remote arrive
  const int U = NG * S;
  const int LT = (l + 7) >> 3;
  const int LPM = P::LPM;

  if (warp == kFNW) {
    // ------------------------------------------------------------ TMA producer (one lane)
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmOm);
      tma_prefetch_desc(&tmPhi);
      const uint64_t pa = policy_evict_first(), pk = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0, ophase = 0;
      for (int u = cid; u < U; u += ncl) {
        const int g = u / S, s = u % S;
        const int strip = g * CL + rank;
        mbar_wait(om_empty, ophase ^ 1);
        mbar_arrive_expect_tx(om_full, P::OM);
#pragma unroll
        for (int b = 0; b < 4; ++b) tma_load_2d(om + b * LPM * 128, &tmOm, om_full, strip * kFBN + b * 16, 0, pk);
        ophase ^= 1;
        const int kt0 = s * KTS, kt1 = min(KT, kt0 + KTS);
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * P::STAGE;
          mbar_arrive_expect_tx(&full[stage], P::STAGE);
          const int r0 = kt * kFBK;
#pragma unroll
          for (int b = 0; b < 4; ++b) tma_load_2d(st + b * kFBK * 128, &tmA, &full[stage], strip * kFBN + b * 16, r0, pa);
          tma_load_2d(st + P::A_STAGE, &tmPhi, &full[stage], r0, 0, pk);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ DMMA consumers
    const int g8 = lane >> 2, t = lane & 3, pg = perm8(g8);
    const int warp_u = __shfl_sync(0xffffffffu, warp, 0);
    const int yc_mt = warp_u & 1;          // Y_c m-tile (of the 2 in a 16-row tile)
    const int yc_n0 = warp_u >> 1;         // Y_c n-tiles yc_n0 + 4 i
    const int rpc = kFBK / CL;             // reduced rows per CTA per tile
    const uint32_t pbuf_s = smem_u32(pbuf);
    double accr[L2T][2];
    int stage = 0;
    uint32_t phase = 0, ophase = 0;
    int tile = 0;                          // tiles processed by this CTA (same sequence in the cluster)
    // Sum tile tt's CL partials (buffer tt & 1 of every CTA, rank order) for rows
    // [rank rpc, (rank+1) rpc) of the tile, store them in group gg's slot, release the buffers.
    auto reduce_tile = [&](int tt, int gg, int ktt) {
      const int bb = tt & 1;
      mbar_wait_cluster(&pready[bb], (tt >> 1) & 1);
      const int nel = rpc * l;
      double* slot = yc_slots + (int64_t)gg * yc_slot_stride;
      for (int e = threadIdx.x; e < nel; e += kFNW * 32) {
        const int rl = rank * rpc + e / l, c = e % l;
        const int grow = ktt * kFBK + rl;
        const uint32_t off = pbuf_s + (uint32_t)((bb * kFBK * LPM + rl * LPM + c) * 8);
        double v = 0.0;
        for (int q = 0; q < CL; ++q) v += ld_dsmem(mapa_u32(off, q));
        if (grow < rows) slot[(int64_t)grow * ldys + c] = v;
      }
      named_bar(1, kFNW * 32);
      if (threadIdx.x < CL) mbar_arrive_remote(mapa_u32(smem_u32(&pfree[bb]), threadIdx.x));
    };
    for (int u = cid; u < U; u += ncl) {
      const int g = u / S, s = u % S;
      const int strip = g * CL + rank;
      const int kt0 = s * KTS, kt1 = min(KT, kt0 + KTS);
#pragma unroll
      for (int nt = 0; nt < L2T; ++nt) accr[nt][0] = accr[nt][1] = 0.0;
      mbar_wait(om_full, ophase);
      ophase ^= 1;
      for (int kt = kt0; kt < kt1; ++kt, ++tile) {
        mbar_wait(&full[stage], phase);
        const uint8_t* As = smem + stage * P::STAGE;
        const uint8_t* Ps = As + P::A_STAGE;
        const int b = tile & 1;
        double* pb = pbuf + b * kFBK * LPM;
        // ---- Y_c partial of this tile: P = A_tile Omega_strip (16 x l), into buffer b
        {
          double accc[LTC][2];
#pragma unroll
          for (int i = 0; i < LTC; ++i) accc[i][0] = accc[i][1] = 0.0;
#pragma unroll
          for (int kk = 0; kk < kFBN / 8; ++kk) {
            const int box = kk >> 1;
            const uint32_t q = ((kk & 1) << 2) + t;
            const double2 a = *reinterpret_cast<const double2*>(As + box * kFBK * 128 + sw128(yc_mt * 8 + pg, q));
            double2 bb[LTC];
#pragma unroll
            for (int i = 0; i < LTC; ++i) {
              const int nt = yc_n0 + 4 * i;
              if (nt < LT) bb[i] = *reinterpret_cast<const double2*>(om + box * LPM * 128 + sw128(nt * 8 + pg, q));
            }
#pragma unroll
            for (int i = 0; i < LTC; ++i)
              if (yc_n0 + 4 * i < LT) dmma(accc[i][0], accc[i][1], a.x, bb[i].x);
#pragma unroll
            for (int i = 0; i < LTC; ++i)
              if (yc_n0 + 4 * i < LT) dmma(accc[i][0], accc[i][1], a.y, bb[i].y);
          }
          if (tile >= 2) mbar_wait_cluster(&pfree[b], ((tile >> 1) + 1) & 1);   // peers read buffer b (tile - 2)
          const int rr = yc_mt * 8 + pg;
#pragma unroll
          for (int i = 0; i < LTC; ++i) {
            const int nt = yc_n0 + 4 * i;
            if (nt < LT) {
              pb[rr * LPM + nt * 8 + t] = accc[i][0];
              pb[rr * LPM + nt * 8 + t + 4] = accc[i][1];
            }
          }
        }
        named_bar(1, kFNW * 32);
        // thread q signals peer q (the release fences run in parallel, one per thread)
        if (threadIdx.x < CL) mbar_arrive_remote(mapa_u32(smem_u32(&pready[b]), threadIdx.x));
        // ---- Y_r[strip columns] += A_tile^T Phi_tile   (this warp: A columns warp * 8 + g8)
#pragma unroll
        for (int kk = 0; kk < kFBK / 8; ++kk) {
          const int r0 = kk * 8 + 2 * t;
          const int c = warp * 8 + g8;
          const uint8_t* base = As + (c >> 4) * kFBK * 128 + ((c & 1) << 3);
          const uint32_t ch = (c & 15) >> 1;
          const double a0 = *reinterpret_cast<const double*>(base + sw128(r0, ch));
          const double a1 = *reinterpret_cast<const double*>(base + sw128(r0 + 1, ch));
          const uint32_t q = ((kk & 1) << 2) + t;
#pragma unroll
          for (int n0 = 0; n0 < L2T; n0 += 4) {
            double2 bb[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (n0 + j < L2T) bb[j] = *reinterpret_cast<const double2*>(Ps + sw128((n0 + j) * 8 + pg, q));
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (n0 + j < L2T) dmma(accr[n0 + j][0], accr[n0 + j][1], a0, bb[j].x);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (n0 + j < L2T) dmma(accr[n0 + j][0], accr[n0 + j][1], a1, bb[j].y);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        // ---- cluster reduction of this tile's Y_c partials (the lagged variant, one tile later,
        // measured slower: 465 vs 416 ms at C4)
        reduce_tile(tile, g, kt);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(om_empty);
      // ---- Y_r of this strip over the split's rows -> slot s
      double* o = yr + (int64_t)s * yr_slot_stride;
      const int col = strip * kFBN + warp * 8 + g8;
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
  // no CTA leaves while a peer may still read its partial buffers or arrive on its barriers
  __syncwarp();
  cluster_sync_all();
}

// out (column-major, ldo) = sum over NG row-major slots (rows x w, ld ldi, stride st) in slot order
__global__ void k_slot_sum_rows(const double* __restrict__ in, int64_t ldi, int64_t st, int NG, int64_t rows, int w,
                                double* __restrict__ out, int64_t ldo) {
  const int c = threadIdx.x % 32 + 32 * blockIdx.y;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (r >= rows || c >= w) return;
  const double* p = in + r * ldi + c;
  double s = p[0];
  for (int gi = 1; gi < NG; ++gi) s += p[(int64_t)gi * st];
  out[(int64_t)c * ldo + r] = s;
}

PFN_cuTensorMapEncodeTiled_v12000 g_enc_fc = nullptr;

int make_map_fc(CUtensorMap* map, const double* base, int64_t inner, int64_t outer, int64_t ld, int box_outer) {
  if (!g_enc_fc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr)
      return RSVD_E_CUDA;
    g_enc_fc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {16u, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = g_enc_fc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? RSVD_OK : RSVD_E_CUDA;
}

int cluster_size_for(int64_t n) {
  static const int force = [] {   // RSVD_FC_CL=8 / 16: A/B of the cluster size (measurement only)
    const char* e = getenv("RSVD_FC_CL");
    const int v = e ? atoi(e) : 0;
    return (v == 8 || v == 16) ? v : 0;
  }();
  if (force) return force;
  return (n + kFBN - 1) / kFBN >= 32 ? 16 : 8;
}

template <int L2T, int LTC>
int launch_fc_t(const FusedClArgs& a, cudaStream_t st) {
  using P = FcPlan<L2T, LTC>;
  CUtensorMap tmA, tmOm, tmPhi;
  if (make_map_fc(&tmA, a.A, a.n, a.rows, a.lda, kFBK) || make_map_fc(&tmOm, a.Om, a.n, a.l, a.ldom, P::LPM) ||
      make_map_fc(&tmPhi, a.Phi, a.rows, a.l2, a.ldphi, P::L2P))
    return RSVD_E_CUDA;
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_view_fused_cl<L2T, LTC>, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM);
    cudaFuncSetAttribute(k_view_fused_cl<L2T, LTC>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  const int CL = a.CL;
  const int KT = (int)((a.rows + kFBK - 1) / kFBK);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.nclusters * CL);
  cfg.blockDim = dim3(kFThreads);
  cfg.dynamicSmemBytes = P::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_view_fused_cl<L2T, LTC>, tmA, tmOm, tmPhi, a.yc_slots, a.ldys,
                                     a.yc_slot_stride, a.yr, a.ldyr, a.yr_slot_stride, (int)a.rows, (int)a.n, a.l, a.l2,
                                     a.NG, a.S, KT, a.KTS);
  return e == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

template <int... Is>
struct FcSeq {};
template <int LTC, int... Is>
int fc_dispatch(int L2T, const FusedClArgs& a, cudaStream_t st, FcSeq<Is...>) {
  int r = RSVD_E_ARG;
  ((L2T == Is ? (r = launch_fc_t<Is, LTC>(a, st), 0) : 0), ...);
  return r;
}
// supported Y_r widths in 8-column tiles (l2 padded up to the next one)
using FcL2 = FcSeq<8, 12, 16, 18, 24, 30, 32>;
constexpr int kFcL2[] = {8, 12, 16, 18, 24, 30, 32};

template <int L2T, int LTC>
int max_clusters_t(int CL) {
  using P = FcPlan<L2T, LTC>;
  cudaFuncSetAttribute(k_view_fused_cl<L2T, LTC>, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM);
  cudaFuncSetAttribute(k_view_fused_cl<L2T, LTC>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(kFThreads);
  cfg.dynamicSmemBytes = P::SMEM;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_view_fused_cl<L2T, LTC>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace

int fused_cl_l2t(int l2) {
  const int need = (l2 + 7) / 8;
  for (int v : kFcL2)
    if (v >= need) return v;
  return 0;
}
int fused_cl_ltc(int l) { return ((l + 7) / 8 + 3) / 4; }   // Y_c n-tiles per warp (4 warp groups)

bool fused_cl_supported(int l, int l2) { return l >= 1 && l <= 128 && l2 >= 1 && fused_cl_l2t(l2) > 0; }

// Plan: cluster size, co-resident clusters, strip groups NG, row splits S (minimising the busiest
// cluster's tile count), and the slot sizes the caller allocates.
void plan_fused_cl(int64_t rows, int64_t n, int l, int l2, int sms, FusedClArgs* a) {
  a->CL = cluster_size_for(n);
  const int NSB = (int)((n + kFBN - 1) / kFBN);
  a->NG = (NSB + a->CL - 1) / a->CL;
  static int cache[2][40] = {};   // max active clusters per (CL, L2T) (host-side, computed once)
  const int ci = a->CL == 16 ? 1 : 0, l2t = fused_cl_l2t(l2), ltc = fused_cl_ltc(l);
  int ncl = cache[ci][l2t];
  if (ncl == 0) {
    switch (ltc * 100 + l2t) {
#define FC_CASE(LTCV, L2V) \
  case LTCV * 100 + L2V: ncl = max_clusters_t<L2V, LTCV>(a->CL); break;
#define FC_ROW(LTCV) FC_CASE(LTCV, 8) FC_CASE(LTCV, 12) FC_CASE(LTCV, 16) FC_CASE(LTCV, 18) FC_CASE(LTCV, 24) \
  FC_CASE(LTCV, 30) FC_CASE(LTCV, 32)
      FC_ROW(1) FC_ROW(2) FC_ROW(3) FC_ROW(4)
#undef FC_ROW
#undef FC_CASE
      default: ncl = 0;
    }
    if (ncl < 1) ncl = std::max(1, sms / a->CL);
    cache[ci][l2t] = ncl;   // (per L2T: the plan's shared memory barely depends on LTC)
  }
  ncl = std::min(ncl, std::max(1, sms / a->CL));
  const int KT = (int)((rows + kFBK - 1) / kFBK);
  double best = 1e30;
  int bS = 1, bK = KT;
  for (int S = 1; S <= std::min(KT, 32); ++S) {
    const int kts = (KT + S - 1) / S;
    const int s2 = (KT + kts - 1) / kts;
    const long U = (long)a->NG * s2;
    const long G = std::min<long>(U, ncl);
    const long per = (U + G - 1) / G;
    const double cost = per * (kts + 6.0);
    if (cost < best - 1e-9) { best = cost; bS = s2; bK = kts; }
  }
  a->S = bS;
  a->KTS = bK;
  a->nclusters = (int)std::min<long>((long)a->NG * bS, ncl);
  if (getenv("RSVD_FC_DEBUG"))
    fprintf(stderr, "fused_cl plan: CL %d NG %d S %d KTS %d clusters %d (max active %d)\n", a->CL, a->NG, a->S, a->KTS,
            a->nclusters, ncl);
}

int launch_view_fused_cl(const FusedClArgs& a, cudaStream_t st) {
  const int L2T = fused_cl_l2t(a.l2), LTC = fused_cl_ltc(a.l);
  if (!L2T || LTC < 1 || LTC > 4) return RSVD_E_ARG;
  switch (LTC) {
    case 1: return fc_dispatch<1>(L2T, a, st, FcL2{});
    case 2: return fc_dispatch<2>(L2T, a, st, FcL2{});
    case 3: return fc_dispatch<3>(L2T, a, st, FcL2{});
    default: return fc_dispatch<4>(L2T, a, st, FcL2{});
  }
}

int launch_slot_sum_rows(const double* in, int64_t ldi, int64_t slot_stride, int NG, int64_t rows, int w, double* out,
                         int64_t ldo, cudaStream_t st) {
  if (rows <= 0 || w <= 0) return RSVD_OK;
  dim3 grid((unsigned)((rows + 7) / 8), (unsigned)((w + 31) / 32));
  k_slot_sum_rows<<<grid, 256, 0, st>>>(in, ldi, slot_stride, NG, rows, w, out, ldo);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

}  // namespace rsvd
