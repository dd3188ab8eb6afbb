// fp32 matrix views on the 5th-generation tensor cores (tcgen05, kind::tf32), 3xTF32 split.
//
//   k_view_tf32<VIEW_AX>   Y = A X       (Alg. 2 line 4 "A Q_r", Alg. 9 line 4)
//   k_view_tf32<VIEW_ATY>  Z = A^T Y     (Alg. 2 line 6 "A^* Q_c", Alg. 9 line 5)
//
// A is fp32 (the C5 configuration), row-major.  One TF32 product keeps 11 significant bits,
// which fails the fp32 parity tolerance, so every product is formed as
//     A X  ~  A_hi X_hi + A_hi X_lo + A_lo X_hi,      v_hi = rna_tf32(v), v_lo = rna_tf32(v - v_hi)
// (22-bit operands, the lo*lo term dropped), accumulated in fp32 in TMEM.
//
// Pipeline per CTA (persistent; units = (block of 128*MT output rows) x (reduction range)):
//   warp 0      TMA producer: raw A tile (fp32, SWIZZLE_64B) + the pre-split X_hi / X_lo tiles
//   warps 2..5  split the raw A tile in shared memory: hi in place, lo into its own buffer
//               (elementwise, so the swizzled layout TMA produced is kept), then release the
//               stage to the MMA warp; at the end of a unit they drain TMEM (tcgen05.ld) and
//               write the fp64 partial slot
//   warp 1      one elected lane issues tcgen05.mma (M = 128, N <= 256 per instruction) from
//               smem descriptors and commits stage release / accumulator-ready to mbarriers
// A x X: A tile is K-major (k contiguous).  A^T x Y: the A tile is read MN-major (the output
// index, A's column, is the contiguous one) — tcgen05 accepts MN-major tf32 operands.
#include <atomic>
#include "common.cuh"
#include "internal.h"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

namespace rsvd {
namespace {

constexpr int kBK = 16;          // fp32 per 64-byte swizzled row = reduction elements per stage
constexpr int kThreads = 192;    // 6 warps
constexpr int kMaxStages = 8;
constexpr int kSmemBudget = 200 * 1024;
// Stages accumulated in one fp32 TMEM accumulator before it is drained.  The tensor core's fp32
// accumulation is not round-to-nearest: its error is biased toward zero and grows with the number
// of accumulating MMAs (6 per stage).  Measured (tools/tf32_bias_probe.py, 20000 x 100000, w = 250):
// one accumulator over ~1500 stages shrinks every output by 4.7e-5 (the full C5, 6250 stages: every
// singular value 2.1e-4 low, above the fp32 parity tolerance 1e-4); 256-stage chunks 2.3e-5,
// 64-stage chunks 6e-6.  Each chunk is stored as its own fp32 partial slot (fire-and-forget stores,
// no read-modify-write in the kernel) and the slots are summed in fp64 afterwards.
constexpr int kTf32Chunk = 256;

__host__ __device__ constexpr int tmem_cols_for(int c) {
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

// Padded width: WP = NCH chunks of NW columns (NW a multiple of 16, <= 256: one MMA's N each)
__host__ __device__ inline void pad_width(int w, int* WP, int* NW) {
  const int w16 = (w + 15) / 16 * 16;
  const int nch = (w16 + 255) / 256;
  const int nw = ((w16 + nch - 1) / nch + 15) / 16 * 16;
  *NW = nw;
  *WP = nw * nch;
}

struct Geo {  // runtime geometry shared by host and device
  int MT, WP, NCH, NW;
  int a_bytes, x_bytes, stage_bytes, stages, tmem_cols;
  __host__ __device__ void init(int mt, int w) {
    MT = mt;
    pad_width(w, &WP, &NW);
    const int wp = WP;
    NCH = WP / NW;
    a_bytes = 128 * mt * kBK * 4;
    x_bytes = wp * kBK * 4;
    stage_bytes = 2 * a_bytes + 2 * x_bytes;
    stages = kSmemBudget / stage_bytes;
    if (stages > kMaxStages) stages = kMaxStages;
    tmem_cols = tmem_cols_for(mt * wp);
  }
  __host__ __device__ int smem() const { return stages * stage_bytes + 1024 + 256; }
};

// ---------------------------------------------------------------- tcgen05 helpers
// shared-memory matrix descriptor; layout 4 = SWIZZLE_64B (K-major operands), 1 = 128-byte
// swizzle with 32-byte atoms (the only layout tcgen05 takes for MN-major tf32 operands)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;          // descriptor version 1 (sm_100)
  d |= (uint64_t)layout << 61;
  return d;
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, M = 128, N = n
__device__ __forceinline__ uint32_t idesc_tf32(int n, int a_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- the view kernel
// KIND == VIEW_AX : out rows = rows of A (M), reduction over n.   tmA box {16 cols, 128 rows}
// KIND == VIEW_ATY: out rows = cols of A (M), reduction over rows. tmA box {32 cols, 16 rows},
//                   128B swizzle with 32B atoms (MN-major tf32 operand layout)
// tmXh / tmXl: X^T (resp. Y^T) pre-split, fp32 [w x K] with K contiguous, box {16, min(WP,256)}
// TRUNC: A_hi is A itself (the tensor core reads the upper 19 bits of the fp32 container, i.e.
// truncates to tf32), so the raw tile stays as TMA wrote it and only A_lo = A - trunc(A) (the
// low 13 mantissa bits, exact in fp32) is formed and stored; else A_hi = rna(A) in place and
// A_lo = rna(A - A_hi).  (RSVD_TF32_RNA=1 selects the rounded split for A/B.)
template <int KIND, int TRUNC>
__global__ void __launch_bounds__(kThreads, 1)
    k_view_tf32(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmXh,
                const __grid_constant__ CUtensorMap tmXl, float* __restrict__ out, int64_t ldo,
                int64_t slot_stride, int out_rows, int w, int MT, int NB, int S, int KT, int KTS, int kChunk) {
  Geo G;
  G.init(MT, w);
  const int WP = G.WP, NW = G.NW;
  extern __shared__ uint8_t smem_raw[];
  // aligned by pointer arithmetic on the __shared__ array (keeps the shared address space)
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G.stages * G.stage_bytes);
  uint64_t* conv = full + kMaxStages;
  uint64_t* empty = conv + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tbase_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int BM = 128 * MT;

  if (threadIdx.x == 0) {
    for (int s = 0; s < G.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tbase_slot)),
                 "r"(G.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tbase_slot;
  const int U = NB * S;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmXh);
      tma_prefetch_desc(&tmXl);
      // A x X reads each row of A in 64-byte k-chunks: with 256-byte L2 promotion the other three
      // chunks of a promoted line are used by the next three stages, so A must not be marked
      // evict-first there (ncu: 1.66x DRAM over-fetch with evict_first).  A^T x Y reads 128-byte
      // rows of 4 adjacent boxes per stage: evict_first is safe.
      const uint64_t pa = (KIND == VIEW_AX) ? policy_evict_normal() : policy_evict_first();
      const uint64_t px = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < U; u += gridDim.x) {
        const int blk = u / S, s = u % S;
        const int kt0 = s * KTS, kt1 = min(KT, kt0 + KTS);
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * G.stage_bytes;
          mbar_arrive_expect_tx(&full[stage], G.a_bytes + 2 * G.x_bytes);
          const int k0 = kt * kBK;
          if (KIND == VIEW_AX) {
            for (int t = 0; t < MT; ++t) tma_load_2d(st + t * 128 * 64, &tmA, &full[stage], k0, blk * BM + t * 128, pa);
          } else {
            for (int b = 0; b < BM / 32; ++b)
              tma_load_2d(st + b * (kBK * 128), &tmA, &full[stage], blk * BM + b * 32, k0, pa);
          }
          uint8_t* xh = st + 2 * G.a_bytes;
          uint8_t* xl = xh + G.x_bytes;
          for (int c = 0; c < WP; c += NW) {
            tma_load_2d(xh + c * 64, &tmXh, &full[stage], k0, c, px);
            tma_load_2d(xl + c * 64, &tmXl, &full[stage], k0, c, px);
          }
          if (++stage == G.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    int stage = 0;
    uint32_t phase = 0, tphase = 0;
    // A operand: K-major (AX) rows of 64 B, 8-row groups 512 B apart; MN-major (ATY) 32-column
    // boxes of kBK rows x 128 B side by side (LBO), 4-row K groups 512 B apart (SBO)
    const uint32_t a_lbo = (KIND == VIEW_AX) ? 16u : (uint32_t)(kBK * 128);
    const uint32_t a_ks = (KIND == VIEW_AX) ? 32u : 1024u;         // byte step per 8-wide k step
    const uint32_t a_tile = (KIND == VIEW_AX) ? 128u * 64u : 4u * (kBK * 128);  // per 128-row M tile
    const uint32_t a_lay = (KIND == VIEW_AX) ? 4u : 1u;
    for (int u = blockIdx.x; u < U; u += gridDim.x) {
      const int s = u % S;
      const int kt0 = s * KTS, kt1 = min(KT, kt0 + KTS);
      int kc0 = kt0;                         // first stage of the current accumulation chunk
      for (int kt = kt0; kt < kt1; ++kt) {
        if (kt == kc0) {                     // a new chunk: TMEM must have been drained
          if (lane == 0) mbar_wait(tempty, tphase ^ 1);
          tphase ^= 1;
          __syncwarp();
          tc_fence_after();
        }
        const bool chunk_end = (kt == kt1 - 1) || (kt - kc0 == kChunk - 1);
        if (lane == 0) {
          mbar_wait(&conv[stage], phase);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + stage * G.stage_bytes);
          const uint32_t ahi = st, alo = st + G.a_bytes, xh = st + 2 * G.a_bytes, xl = xh + G.x_bytes;
#pragma unroll
          for (int ks = 0; ks < kBK / 8; ++ks) {
            for (int t = 0; t < MT; ++t) {
              const uint64_t dah = sdesc(ahi + t * a_tile + ks * a_ks, a_lbo, 512, a_lay);
              const uint64_t dal = sdesc(alo + t * a_tile + ks * a_ks, a_lbo, 512, a_lay);
              const uint32_t id = idesc_tf32(NW, KIND == VIEW_ATY);
              for (int c = 0; c < G.NCH; ++c) {
                const uint64_t dxh = sdesc(xh + c * NW * 64 + ks * 32, 16, 512, 4);
                const uint64_t dxl = sdesc(xl + c * NW * 64 + ks * 32, 16, 512, 4);
                const uint32_t d = tbase + (uint32_t)(t * WP + c * NW);
                mma_tf32(d, dah, dxh, id, (kt > kc0 || ks > 0) ? 1u : 0u);
                mma_tf32(d, dah, dxl, id, 1u);
                mma_tf32(d, dal, dxh, id, 1u);
              }
            }
          }
          mma_commit(&empty[stage]);
          if (chunk_end) mma_commit(tfull);
        }
        __syncwarp();
        if (chunk_end) kc0 = kt + 1;
        if (++stage == G.stages) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ split + epilogue (warps 2..5)
    const int ct = threadIdx.x - 64;  // 0..127
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    int stage = 0;
    uint32_t phase = 0, tphase = 0;
    for (int u = blockIdx.x; u < U; u += gridDim.x) {
      const int blk = u / S, s = u % S;
      const int kt0 = s * KTS, kt1 = min(KT, kt0 + KTS);
      int kc0 = kt0;
      for (int kt = kt0; kt < kt1; ++kt) {
        mbar_wait(&full[stage], phase);
        uint8_t* st = smem + stage * G.stage_bytes;
        float4* raw = reinterpret_cast<float4*>(st);
        float4* lo = reinterpret_cast<float4*>(st + G.a_bytes);
        const int n4 = G.a_bytes / 16;
        if (TRUNC) {
          for (int i = ct; i < n4; i += 128) {
            const float4 v = raw[i];
            float4 l;
            l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
            l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
            l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
            l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
            lo[i] = l;
          }
        } else {
          for (int i = ct; i < n4; i += 128) {
            const float4 v = raw[i];
            float4 h, l;
            h.x = rna_tf32(v.x); l.x = rna_tf32(v.x - h.x);
            h.y = rna_tf32(v.y); l.y = rna_tf32(v.y - h.y);
            h.z = rna_tf32(v.z); l.z = rna_tf32(v.z - h.z);
            h.w = rna_tf32(v.w); l.w = rna_tf32(v.w - h.w);
            raw[i] = h;
            lo[i] = l;
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[stage]);
        if (++stage == G.stages) { stage = 0; phase ^= 1; }
        if (kt != kt1 - 1 && kt - kc0 != kChunk - 1) continue;
        // end of an accumulation chunk: drain TMEM (lane = output row inside the 128-row tile,
        // column = output column) into this chunk's fp32 partial slot
        const int cpu = (KTS + kChunk - 1) / kChunk;            // chunk slots per unit
        const int ci = (kc0 - kt0) / kChunk;
        const bool last = (kt == kt1 - 1);
        kc0 = kt + 1;
        mbar_wait(tfull, tphase);
        tphase ^= 1;
        tc_fence_after();
        float* o = out + (int64_t)(s * cpu + ci) * slot_stride;
        for (int t = 0; t < MT; ++t) {
          const int r = blk * BM + t * 128 + q * 32 + lane;
          for (int c0 = 0; c0 < WP; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(t * WP + c0), v);
            tmem_ld_wait();
            if (r < out_rows) {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (c0 + j < w) o[(int64_t)(c0 + j) * ldo + r] = __uint_as_float(v[j]);
            }
          }
          // a short last unit has fewer chunks than cpu: its unused slots hold zeros
          if (last && r < out_rows)
            for (int cz = ci + 1; cz < cpu; ++cz) {
              float* oz = out + (int64_t)(s * cpu + cz) * slot_stride;
              for (int c = 0; c < w; ++c) oz[(int64_t)c * ldo + r] = 0.0f;
            }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(G.tmem_cols) : "memory");
  }
}

// X (fp64, column-major rows x w, ld) -> X_hi, X_lo (fp32 tf32-rounded, column-major, ld32)
__global__ void k_split_tf32(const double* __restrict__ X, int64_t ld, int64_t rows, int w, float* __restrict__ hi,
                             float* __restrict__ lo, int64_t ld32) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r >= rows || c >= w) return;
  const double x = X[(int64_t)c * ld + r];
  const float h = rna_tf32((float)x);
  const float l = rna_tf32((float)(x - (double)h));
  hi[(int64_t)c * ld32 + r] = h;
  lo[(int64_t)c * ld32 + r] = l;
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode32 = nullptr;

int make_map32(CUtensorMap* map, const float* base, int64_t inner, int64_t outer, int64_t ld, int box_inner,
               int box_outer, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_64B) {
  if (!g_encode32) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr)
      return RSVD_E_CUDA;
    g_encode32 = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = g_encode32(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? RSVD_OK : RSVD_E_CUDA;
}

int mt_for(int w) {
  int wp, nw;
  pad_width(w, &wp, &nw);
  return wp <= 256 ? 2 : 1;
}

}  // namespace

void plan_view_tf32(int kind, int64_t rows, int64_t n, int w, int grid_cap, int* S, int* KTS) {
  const int bm = 128 * mt_for(w);
  const int64_t out_rows = kind == VIEW_AX ? rows : n;
  const int64_t K = kind == VIEW_AX ? n : rows;
  const int NB = (int)((out_rows + bm - 1) / bm);
  const int KT = (int)((K + kBK - 1) / kBK);
  // minimise the busiest CTA's tile count (+ a per-unit epilogue overhead in tiles)
  double best = 1e30;
  int bS = 1, bK = KT;
  for (int s = 1; s <= std::min(KT, 64); ++s) {
    const int kts = (KT + s - 1) / s;
    const int s2 = (KT + kts - 1) / kts;
    const long U = (long)NB * s2;
    const long Gd = std::min<long>(U, grid_cap);
    const long per = (U + Gd - 1) / Gd;
    const double cost = per * (kts + 8.0);
    if (cost < best - 1e-9) { best = cost; bS = s2; bK = kts; }
  }
  *S = bS;
  *KTS = bK;
}

int tf32_slots(int S, int KTS) { return S * ((KTS + kTf32Chunk - 1) / kTf32Chunk); }

int launch_split_tf32(const double* X, int64_t ld, int64_t rows, int w, float* hi, float* lo, int64_t ld32,
                      cudaStream_t st) {
  if (rows <= 0 || w <= 0) return RSVD_OK;
  dim3 grid((unsigned)((rows + 255) / 256), (unsigned)w);
  k_split_tf32<<<grid, 256, 0, st>>>(X, ld, rows, w, hi, lo, ld32);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

int launch_view_tf32(const ViewArgs32& a, cudaStream_t st) {
  if (a.w < 1 || a.w > kMaxW32) return RSVD_E_ARG;
  const int MT = mt_for(a.w);
  Geo G;
  G.init(MT, a.w);
  if (G.stages < 2) return RSVD_E_ARG;
  const int BM = 128 * MT;
  const bool ax = a.kind == VIEW_AX;
  const int64_t out_rows = ax ? a.rows : a.n;
  const int64_t K = ax ? a.n : a.rows;
  CUtensorMap tmA, tmXh, tmXl;
  if ((ax ? make_map32(&tmA, a.A, a.n, a.rows, a.lda, 16, 128)
         : make_map32(&tmA, a.A, a.n, a.rows, a.lda, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) ||
      make_map32(&tmXh, a.Xhi, K, a.w, a.ldx, 16, G.NW) || make_map32(&tmXl, a.Xlo, K, a.w, a.ldx, 16, G.NW))
    return RSVD_E_CUDA;
  const int NB = (int)((out_rows + BM - 1) / BM);
  const int KT = (int)((K + kBK - 1) / kBK);
  const int U = NB * a.S;
  const int grid = std::min(U, a.grid_cap);
  const int smem = G.smem();
  const int chunk = kTf32Chunk;
  static const bool rna = [] {
    const char* e = getenv("RSVD_TF32_RNA");
    return e && e[0] == '1';
  }();
  static std::atomic<bool> attr{false};
  if (!attr) {
    cudaFuncSetAttribute(k_view_tf32<VIEW_AX, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 2048);
    cudaFuncSetAttribute(k_view_tf32<VIEW_ATY, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 2048);
    cudaFuncSetAttribute(k_view_tf32<VIEW_AX, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 2048);
    cudaFuncSetAttribute(k_view_tf32<VIEW_ATY, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 2048);
    attr = true;
  }
#define TF32_LAUNCH(K, T)                                                                                        \
  k_view_tf32<K, T><<<grid, kThreads, smem, st>>>(tmA, tmXh, tmXl, a.out, a.ldo, a.slot_stride, (int)out_rows, \
                                                  a.w, MT, NB, a.S, KT, a.KTS, chunk)
  if (ax) {
    if (rna) TF32_LAUNCH(VIEW_AX, 0); else TF32_LAUNCH(VIEW_AX, 1);
  } else {
    if (rna) TF32_LAUNCH(VIEW_ATY, 0); else TF32_LAUNCH(VIEW_ATY, 1);
  }
#undef TF32_LAUNCH
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

}  // namespace rsvd

namespace rsvd {
namespace {
__global__ void k_f32_to_f64(const float* __restrict__ s, int64_t lds, double* __restrict__ d, int64_t ldd,
                             int64_t rows, int cols) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r < rows && c < cols) d[(int64_t)c * ldd + r] = (double)s[(int64_t)c * lds + r];
}
__global__ void k_f64_to_f32(const double* __restrict__ s, int64_t lds, float* __restrict__ d, int64_t ldd,
                             int64_t rows, int cols) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r < rows && c < cols) d[(int64_t)c * ldd + r] = (float)s[(int64_t)c * lds + r];
}
}  // namespace

int launch_f32_to_f64(const float* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int cols,
                      cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return RSVD_OK;
  k_f32_to_f64<<<dim3((unsigned)((rows + 255) / 256), (unsigned)cols), 256, 0, st>>>(src, lds, dst, ldd, rows, cols);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}
int launch_f64_to_f32(const double* src, int64_t lds, float* dst, int64_t ldd, int64_t rows, int cols,
                      cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return RSVD_OK;
  k_f64_to_f32<<<dim3((unsigned)((rows + 255) / 256), (unsigned)cols), 256, 0, st>>>(src, lds, dst, ldd, rows, cols);
  return cudaPeekAtLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}
}  // namespace rsvd
