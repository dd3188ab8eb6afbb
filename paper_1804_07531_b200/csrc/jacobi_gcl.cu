// Core SVD (tsvd of the w x w core; Alg. 9) by block
// one-sided Jacobi on a thread-block cluster with a Gram-matrix inner solver.
//
// W = M (r x c, zero-padded to nb*b columns) lives in global memory (L2 resident, <= 2 MB).  The
// nb = 2C column blocks of b columns (b a multiple of 4) are paired by a round-robin tournament;
// in each block round cluster CTA k
//   1. loads its block pair W_P = [W_P | W_Q] (r x 2b) into shared memory,
//   2. forms the fresh Gram G = W_P^T W_P (2b x 2b) on the FP64 tensor cores (DMMA m8n8k4),
//   3. if some column pair of the block pair fails |g_pq| <= tol sqrt(g_pp g_qq) (tol = sqrt(r) u,
//      dgesvj's threshold, the same test as the one-CTA kernels), runs one cyclic two-sided Jacobi
//      sweep on G (round-robin pairs, every 2x2 block of G updated by one thread per round, G
//      double-buffered), accumulating the rotations into J_l (2b x 2b, starts at I),
//   4. applies them at once, W_P <- W_P J_l (DMMA), and writes the pair back.
// The column rotations of the one-sided method are thereby applied as one orthogonal 2b x 2b
// product per block round, not one plane rotation at a time over the r-long columns: the inner
// rounds touch 2b x 2b numbers instead of r x 2b (the per-round shared-memory traffic that bounds
// k_jacobi_cluster).  Accuracy is the one-sided method's: every decision is taken on
// a Gram formed afresh from the current columns, the rotations are exactly orthogonal
// (cs = rsqrt(1 + t^2), sn = cs t in fp64), and the values are the final column norms; the Gram's
// two-sided updates only steer the angles of one inner sweep (Demmel-Veselic: two-sided Jacobi
// on the Gram of nearly orthogonal columns is relatively accurate).
// 2C-1 block rounds make one outer sweep, in which every column pair of W meets at least once;
// sweeps repeat until no block pair had a pair above tol, or until no pair of the sweep had a
// cosine above 1e-10 (the rotations then leave O(1e-20), as in k_jacobi_small).
// Deterministic: fixed pairing, fixed DMMA and reduction order, independent of timing.
// Outputs as the other Jacobi kernels: sigma_j = |W_j| sorted descending, Ul = W_j / sigma_j,
// Vr = J (want_j: J_l products accumulated in global memory) or Vr = B^T Ul S^-1.
#include <atomic>
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace rsvd {
namespace {

constexpr int kGThreads = 512;   // 16 warps
constexpr int kGWarps = kGThreads / 32;
constexpr int kGMaxC = 512;
constexpr int kGMaxRS = kGMaxC + 8 + 4;
constexpr int kGSmemMax = 225 * 1024;   // dynamic shared memory opt-in (227 KB less the static arrays)

// phase timers (tools/gcl_probe.cu builds this file with RSVD_GCL_TIMING): cycles seen by thread 0
// of cluster rank 0 per phase of the block round
#ifdef RSVD_GCL_TIMING
__device__ unsigned long long gcl_ph[8];
#define GCL_T0() long long gcl_t0 = clock64()
#define GCL_T(i)                                                                 \
  if (tid == 0 && rank == 0) {                                                   \
    const long long gcl_t = clock64();                                           \
    gcl_ph[i] += gcl_t - gcl_t0;                                                 \
    gcl_t0 = gcl_t;                                                              \
  }
#else
#define GCL_T0()
#define GCL_T(i)
#endif

__device__ __forceinline__ void gpair_of(int round, int k, int n, int* p, int* q) {
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

// plane rotation for the pair with Gram entries (a, b, g): w_p' = cs w_p - sn w_q,
// w_q' = sn w_p + cs w_q zeroes g; identity when |g| <= tol sqrt(ab).  Branch-free (a thread forms
// two rotations per round and the two chains interleave); t from the approximate fp64 MUFU ops
// (any t gives an exactly orthogonal rotation), cs = 1/sqrt(1 + t^2) by two Newton steps from the
// MUFU seed (1 + t^2 in [1, 2]: no scaling), sn = cs t.
__device__ __forceinline__ void grot(double a, double b, double g, double tol2, double* cs, double* sn) {
  // zeta = (b - a) / (2g), t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)); no clamps needed: a
  // rotation is only taken for g^2 > tol^2 ab, so |zeta| <= (a + b) / (2 tol sqrt(ab)) stays far
  // inside the fp64 range (the selects discard the non-rotating pairs' inf / NaN)
  const bool rot = (g != 0.0) && (g * g > tol2 * (a * b));
  double rg, rs, rt, y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rg) : "d"(g + g));
  const double z = (b - a) * rg;
  const double s1 = fma(z, z, 1.0);
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rs) : "d"(s1));
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rt) : "d"(fma(s1, rs, fabs(z))));
  const double t = z < 0.0 ? -rt : rt;
  const double x = fma(t, t, 1.0);
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // one third-order step: e = 1 - x y^2, y (1 + e/2 + 3e^2/8) (MUFU seed ~2^-22 -> ~2^-64)
  const double e = fma(-x, y * y, 1.0);
  y = fma(y * e, fma(0.375, e, 0.5), y);
  *cs = rot ? y : 1.0;
  *sn = rot ? y * t : 0.0;
}

// X (rows x B2, column-major, stride RS, in shared memory) <- X * Jl (B2 x B2, Jl(j, n) at
// Jl[n * LJ + j]), in place: warp w owns the 8-row strips w, w + 16, ...; rows8 a multiple of 8
template <int B2, int LJ>
__device__ __forceinline__ void apply_jl(double* X, int RS, int rows8, const double* Jl, int warp, int lane) {
  constexpr int NT = B2 / 8;
  const int g = lane >> 2, t = lane & 3;
  for (int strip = warp; strip < rows8 / 8; strip += kGWarps) {
    const int i0 = strip * 8;
    double acc[NT][2];
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < B2; k0 += 4) {
      const double a = X[(k0 + t) * RS + i0 + g];
#pragma unroll
      for (int n = 0; n < NT; ++n) dmma(acc[n][0], acc[n][1], a, Jl[(n * 8 + g) * LJ + k0 + t]);
    }
    __syncwarp();
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      X[(n * 8 + 2 * t) * RS + i0 + g] = acc[n][0];
      X[(n * 8 + 2 * t + 1) * RS + i0 + g] = acc[n][1];
    }
  }
}

// as apply_jl, the product stored to dst[n] (column n's destination, another buffer: no
// in-place hazard), 8-byte stores through the generic (possibly remote) pointers
template <int B2, int LJ>
__device__ __forceinline__ void apply_jl_to(const double* X, int RS, int rows8, const double* Jl, double* const* dst,
                                            int warp, int lane) {
  constexpr int NT = B2 / 8;
  const int g = lane >> 2, t = lane & 3;
  for (int strip = warp; strip < rows8 / 8; strip += kGWarps) {
    const int i0 = strip * 8;
    double acc[NT][2];
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < B2; k0 += 4) {
      const double a = X[(k0 + t) * RS + i0 + g];
#pragma unroll
      for (int n = 0; n < NT; ++n) dmma(acc[n][0], acc[n][1], a, Jl[(n * 8 + g) * LJ + k0 + t]);
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      dst[n * 8 + 2 * t][i0 + g] = acc[n][0];
      dst[n * 8 + 2 * t + 1][i0 + g] = acc[n][1];
    }
  }
}

// owner of block X in block round br (round-robin on nb = 2C players, m = nb - 1): the CTA k
// whose pair holds X, and the slot (0: first block of the pair, 1: second)
__device__ __forceinline__ void gowner(int br, int X, int nb, int C, int* k, int* slot) {
  const int m = nb - 1;
  if (X == m) { *k = 0; *slot = 1; return; }
  if (X == br) { *k = 0; *slot = 0; return; }
  const int k1 = (X - br + m) % m, k2 = (br - X + m) % m;   // k1 + k2 = m = 2C - 1
  const int kk = k1 < C ? k1 : k2;
  int p, q;
  gpair_of(br, kk, nb, &p, &q);
  *k = kk;
  *slot = (X == p) ? 0 : 1;
}

// DSM: the block pairs move between block rounds through distributed shared memory (two pair
// buffers per CTA; a CTA copies its next pair from the owners' current buffers after the
// cluster barrier); else through W in global memory (r > 256 with 2b = 32: two buffers do not fit)
template <int B2, bool DSM>
__global__ void __launch_bounds__(kGThreads, 1)
    k_jacobi_gcl(const double* __restrict__ M, int64_t ldm, int trans, int r, int c, int nb, int RS,
                 double* __restrict__ Ul, double* __restrict__ Sv, double* __restrict__ Vr, double* __restrict__ W,
                 double* __restrict__ J, double* __restrict__ sval_g, int* __restrict__ flags, double tol,
                 int max_sweeps, int want_j, int once, int flags_mode, int cross, DevStatus* status) {
  constexpr int b = B2 / 2;
  constexpr int NT = B2 / 8;
  constexpr int T = NT * (NT + 1) / 2;             // 8 x 8 Gram tiles on and above the diagonal
  constexpr int S = kGWarps / T > 0 ? kGWarps / T : 1;   // k-slices per tile (one item per warp)
  constexpr int LG = B2 + 1;                       // G row stride
  constexpr int LJ = B2 + 4;                       // J_l column stride
  constexpr int kInner = ((b * b + 31) / 32) * 32; // threads of the inner sweep (named barrier 1)
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  extern __shared__ __align__(16) double gsm[];
  __shared__ double* s_dst[B2];                    // DSM: remote destination of each local column
  __shared__ double s_cs[b], s_sn[b];              // the inner round's rotations (once)
  double* Wbuf = gsm;                              // DSM ? 2 : 1 pair buffers, B2 columns x RS rows
  double* Gb = Wbuf + (DSM ? 2 : 1) * (size_t)B2 * RS;   // two B2 x LG buffers
  double* Jl = Gb + 2 * B2 * LG;                   // B2 x LJ
  double* Gp = Jl + B2 * LJ;                       // S x B2 x B2 Gram partials
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int ncol = nb * b;                         // padded column count (a multiple of 8)
  const int r4 = (r + 3) & ~3, r8 = (r + 7) & ~7;
  // DSM with J: the pair's J columns (ncol rows) travel below its W columns (rows r8..r8+ncol),
  // so J_P <- J_P J_l is part of the same DMMA product and push
  const bool jw = DSM && want_j;
  const int rows8 = r8 + (jw ? ncol : 0);
  const double tol2 = tol * tol;
  // ---- W = B (B = M or M^T), zero-padded; J = I
  for (int64_t e = (int64_t)rank * kGThreads + tid; e < (int64_t)r * ncol; e += (int64_t)C * kGThreads) {
    const int i = (int)(e % r), j = (int)(e / r);
    double v = 0.0;
    if (j < c) v = trans ? M[(int64_t)i * ldm + j] : M[(int64_t)j * ldm + i];
    W[e] = v;
  }
  if (want_j && !DSM)
    for (int64_t e = (int64_t)rank * kGThreads + tid; e < (int64_t)ncol * ncol; e += (int64_t)C * kGThreads) {
      const int i = (int)(e % ncol), j = (int)(e / ncol);
      J[e] = (i == j) ? 1.0 : 0.0;
    }
  if (rank == 0 && tid < 4) flags[tid] = 0;
  __threadfence();
  cluster.sync();

  int sweep = 0, cur = 0;
  bool converged = false, first = true;
  for (; sweep < max_sweeps; ++sweep) {
    int need_any = 0, big_any = 0;
    for (int br = 0; br < nb - 1; ++br) {
      int P, Q;
      gpair_of(br, rank, nb, &P, &Q);
      GCL_T0();
      // 1. block pair -> shared memory (rows r..r8-1 zero), 8 loads in flight per thread; in DSM
      // mode only for the first block round (later pairs are pushed in by the previous owners)
      if (!DSM || first) {
        // 16 threads per column (B2 <= 32), rows sub, sub + 16, ...: no index division
        constexpr int U = 8;
        double* dst = Wbuf + (DSM ? cur : 0) * (size_t)B2 * RS;
        const int lj = tid >> 4, sub = tid & 15;
        if (lj < B2) {
          const int X = lj < b ? P : Q, jb = lj < b ? lj : lj - b;
          const double* srcc = W + (int64_t)(X * b + jb) * r;
          double* dstc = dst + lj * RS;
          for (int i0 = sub; i0 < r8; i0 += 16 * U) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int i = i0 + 16 * u;
              v[u] = (i < r) ? __ldcg(srcc + i) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (i0 + 16 * u < r8) dstc[i0 + 16 * u] = v[u];
          }
          if (jw)   // J = I: the pair's columns of the identity
            for (int i = sub; i < ncol; i += 16) dstc[r8 + i] = (i == X * b + jb) ? 1.0 : 0.0;
        }
      }
      first = false;
      if (DSM && tid < B2) {
        // destination of each local column in the next block round: the next owner's free buffer
        const int nxt = (br + 1) % (nb - 1);
        const int X = tid < b ? P : Q, jb = tid < b ? tid : tid - b;
        int k, slot;
        gowner(nxt, X, nb, C, &k, &slot);
        s_dst[tid] = cluster.map_shared_rank(Wbuf + (size_t)(cur ^ 1) * B2 * RS + (slot * b + jb) * RS, k);
      }
      double* Wp = Wbuf + (DSM ? cur : 0) * (size_t)B2 * RS;
      __syncthreads();
      GCL_T(0);
      // 2. Gram partials on the tensor cores: item = (tile, k-slice)
      for (int item = warp; item < T * S; item += kGWarps) {
        const int tile = item % T, sl = item / T;
        int ti = 0, rem = tile;                    // tile -> (ti <= tj), row-major upper triangle
        while (rem >= NT - ti) { rem -= NT - ti; ++ti; }
        const int I0 = ti * 8, J0 = (ti + rem) * 8;
        // four independent accumulators (the DMMA latency chain), loads of a group issued first
        double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        const double* ca = Wp + (I0 + g8) * RS + t4;
        const double* cb = Wp + (J0 + g8) * RS + t4;
        constexpr int st = 4 * S;
        int k0 = sl * 4;
        for (; k0 + 3 * st < r4; k0 += 4 * st) {
          double a[4], bb[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            a[u] = ca[k0 + u * st];
            bb[u] = cb[k0 + u * st];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) dmma(acc[u][0], acc[u][1], a[u], bb[u]);
        }
        for (; k0 < r4; k0 += st) dmma(acc[0][0], acc[0][1], ca[k0], cb[k0]);
        double* gp = Gp + sl * B2 * B2 + (I0 + g8) * B2 + J0 + 2 * t4;
        gp[0] = (acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]);
        gp[1] = (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]);
      }
      __syncthreads();
      GCL_T(1);
      // symmetric G (upper triangle's partial sums, fixed slice order), J_l = I, and the fresh
      // one-sided test on every pair of the block pair (diagonals summed by the testing thread)
      int need = 0, big = 0;
      // cross-pair rounds (every block round but a sweep's first, `cross` mode) rotate and test only
      // the pairs (p in P, q in Q); the sweep's first block round runs the full 2b-column sweep,
      // which covers every pair inside each block once per sweep
      const bool full = !cross || br == 0;
      for (int e = tid; e < B2 * B2; e += kGThreads) {
        const int i = e / B2, j = e - i * B2;
        const int lo = i < j ? i : j, hi = i < j ? j : i;
        double s = 0.0, gi = 0.0, gj = 0.0;
#pragma unroll
        for (int sl = 0; sl < S; ++sl) {
          s += Gp[sl * B2 * B2 + lo * B2 + hi];
          gi += Gp[sl * B2 * B2 + i * B2 + i];
          gj += Gp[sl * B2 * B2 + j * B2 + j];
        }
        Gb[i * LG + j] = s;
        Jl[j * LJ + i] = (i == j) ? 1.0 : 0.0;
        if (i < j && (full || (i < b && j >= b)) && s != 0.0 && s * s > tol2 * (gi * gj)) {
          need = 1;
          if (s * s > 1e-20 * (gi * gj)) big = 1;
        }
      }
      need = __syncthreads_or(need);
      big = __syncthreads_or(big);
      GCL_T(2);
      need_any |= need;
      big_any |= big;
      if (need) {
        // one cyclic two-sided sweep on G, rotations accumulated into J_l; only the first
        // kInner threads take part (named barrier 1)
        if (tid < kInner) {
          int gc = 0;
          const int nround = full ? B2 - 1 : b;
          for (int ir = 0; ir < nround; ++ir) {
            if (once) {
              // the round's b rotations formed once (fewer fp64 MUFU ops: 8 b^2 -> 4 b)
              if (tid < b) {
                int p, q;
                if (full) gpair_of(ir, tid, B2, &p, &q);
                else { p = tid; q = b + (tid + ir) % b; }
                const double* G = Gb + gc * B2 * LG;
                grot(G[p * LG + p], G[q * LG + q], G[p * LG + q], tol2, &s_cs[tid], &s_sn[tid]);
              }
              asm volatile("bar.sync 1, %0;" ::"r"(kInner) : "memory");
            }
            if (tid < b * b) {
              const int k1 = tid / b, k2 = tid - (tid / b) * b;
              int p1, q1, p2, q2;
              if (full) {
                gpair_of(ir, k1, B2, &p1, &q1);
                gpair_of(ir, k2, B2, &p2, &q2);
              } else {
                p1 = k1; q1 = b + (k1 + ir) % b;
                p2 = k2; q2 = b + (k2 + ir) % b;
              }
              const double* G = Gb + gc * B2 * LG;
              double* Gn = Gb + (gc ^ 1) * B2 * LG;
              double c1, s1, c2, s2;
              if (once) {
                c1 = s_cs[k1];
                s1 = s_sn[k1];
                c2 = s_cs[k2];
                s2 = s_sn[k2];
              } else {
                grot(G[p1 * LG + p1], G[q1 * LG + q1], G[p1 * LG + q1], tol2, &c1, &s1);
                grot(G[p2 * LG + p2], G[q2 * LG + q2], G[p2 * LG + q2], tol2, &c2, &s2);
              }
              const double gpp = G[p1 * LG + p2], gpq = G[p1 * LG + q2];
              const double gqp = G[q1 * LG + p2], gqq = G[q1 * LG + q2];
              // G' = R1^T [g] R2, R = [[cs, sn], [-sn, cs]]
              const double xpp = c2 * gpp - s2 * gpq, xpq = s2 * gpp + c2 * gpq;
              const double xqp = c2 * gqp - s2 * gqq, xqq = s2 * gqp + c2 * gqq;
              Gn[p1 * LG + p2] = c1 * xpp - s1 * xqp;
              Gn[p1 * LG + q2] = c1 * xpq - s1 * xqq;
              Gn[q1 * LG + p2] = s1 * xpp + c1 * xqp;
              Gn[q1 * LG + q2] = s1 * xpq + c1 * xqq;
              // J_l rows {p2, q2}, columns {p1, q1}: J_l <- J_l R1
              const double jpp = Jl[p1 * LJ + p2], jpq = Jl[q1 * LJ + p2];
              const double jqp = Jl[p1 * LJ + q2], jqq = Jl[q1 * LJ + q2];
              Jl[p1 * LJ + p2] = c1 * jpp - s1 * jpq;
              Jl[q1 * LJ + p2] = s1 * jpp + c1 * jpq;
              Jl[p1 * LJ + q2] = c1 * jqp - s1 * jqq;
              Jl[q1 * LJ + q2] = s1 * jqp + c1 * jqq;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(kInner) : "memory");
            gc ^= 1;
          }
        }
        __syncthreads();
        GCL_T(3);
        // 4. W_P <- W_P J_l: DSM into the next owners' buffers, else in place; V columns:
        // J_P <- J_P J_l from global memory, one row per thread
        if (DSM) apply_jl_to<B2, LJ>(Wp, RS, rows8, Jl, s_dst, warp, lane);
        else apply_jl<B2, LJ>(Wp, RS, r8, Jl, warp, lane);
        if (want_j && !DSM) {
          for (int i = tid; i < ncol; i += kGThreads) {
            double x[B2];
#pragma unroll
            for (int lj = 0; lj < B2; ++lj) {
              const int gj = lj < b ? P * b + lj : Q * b + (lj - b);
              x[lj] = __ldcg(J + (int64_t)gj * ncol + i);
            }
#pragma unroll 1
            for (int n = 0; n < B2; ++n) {
              double s = 0.0;
#pragma unroll
              for (int j = 0; j < B2; ++j) s = fma(x[j], Jl[n * LJ + j], s);
              const int gj = n < b ? P * b + n : Q * b + (n - b);
              J[(int64_t)gj * ncol + i] = s;
            }
          }
        }
        if (!DSM) {
          __syncthreads();
          GCL_T(4);
          const int lj = tid >> 4, sub = tid & 15;
          if (lj < B2) {
            const int gj = lj < b ? P * b + lj : Q * b + (lj - b);
            for (int i = sub; i < r; i += 16) W[(int64_t)gj * r + i] = Wp[lj * RS + i];
          }
        }
        GCL_T(5);
      } else if (DSM) {
        // unchanged pair: 16-byte copies into the next owners' buffers
        const int h8 = rows8 >> 1;
        for (int e = tid; e < B2 * h8; e += kGThreads) {
          const int lj = e / h8, i2 = e - lj * h8;
          reinterpret_cast<double2*>(s_dst[lj])[i2] = reinterpret_cast<const double2*>(Wp + lj * RS)[i2];
        }
      }
      if (!DSM) __threadfence();
      cluster.sync();
      if (DSM) cur ^= 1;
      GCL_T(6);
    }
    // convergence: OR over the cluster of (rotated, big) in flags[2 (sweep & 1) + {0, 1}],
    // the next sweep's pair reset one sweep ahead
    if (tid == 0) {
      if (need_any) atomicOr(&flags[2 * (sweep & 1)], 1);
      if (big_any) atomicOr(&flags[2 * (sweep & 1) + 1], 1);
      if (rank == 0) {
        flags[2 * ((sweep + 1) & 1)] = 0;
        flags[2 * ((sweep + 1) & 1) + 1] = 0;
      }
    }
    __threadfence();
    cluster.sync();
    const int any = *((volatile int*)&flags[2 * (sweep & 1)]);
    const int anybig = *((volatile int*)&flags[2 * (sweep & 1) + 1]);
    cluster.sync();   // everyone has read the flags before they are reset next sweep
    if (!any || (!anybig && !(flags_mode & 1))) {
      converged = true;
      ++sweep;
      break;
    }
  }
  if (DSM) {
    // the last block round's pair -> W
    int P, Q;
    gpair_of(0, rank, nb, &P, &Q);   // the pushed pair is round 0's (of the next sweep)
    const double* Wp = Wbuf + (size_t)cur * B2 * RS;
    for (int e = tid; e < B2 * r; e += kGThreads) {
      const int lj = e / r, i = e - lj * r;
      const int gj = lj < b ? P * b + lj : Q * b + (lj - b);
      W[(int64_t)gj * r + i] = Wp[lj * RS + i];
    }
    if (jw)
      for (int e = tid; e < B2 * ncol; e += kGThreads) {
        const int lj = e / ncol, i = e - lj * ncol;
        const int gj = lj < b ? P * b + lj : Q * b + (lj - b);
        J[(int64_t)gj * ncol + i] = Wp[lj * RS + r8 + i];
      }
    __threadfence();
    cluster.sync();
  }
  // ---- singular values (column norms), descending ranks, outputs
  for (int j = rank * kGWarps + warp; j < ncol; j += C * kGWarps) {
    const double* wj = W + (int64_t)j * r;
    double s = 0.0;
    for (int i = lane; i < r; i += 32) s = fma(wj[i], wj[i], s);
    s = warp_sum(s);
    if (lane == 0) sval_g[j] = sqrt(s);
  }
  __threadfence();
  cluster.sync();
  for (int j = rank * kGThreads + tid; j < ncol; j += C * kGThreads) {
    const double sj = sval_g[j];
    int rk = 0;
    for (int i = 0; i < ncol; ++i) {
      const double si = sval_g[i];
      rk += (si > sj) || (si == sj && i < j);
    }
    if (rk < c) {
      Sv[rk] = sj;
      reinterpret_cast<int*>(sval_g + kGMaxC)[rk] = j;  // rank -> column
    }
  }
  __threadfence();
  cluster.sync();
  const int* col_of = reinterpret_cast<const int*>(sval_g + kGMaxC);
  for (int64_t e = (int64_t)rank * kGThreads + tid; e < (int64_t)r * c; e += (int64_t)C * kGThreads) {
    const int i = (int)(e % r), rk = (int)(e / r);
    const int j = col_of[rk];
    const double sj = sval_g[j];
    Ul[(int64_t)rk * r + i] = sj > 0.0 ? W[(int64_t)j * r + i] / sj : 0.0;
  }
  if (want_j) {
    for (int64_t e = (int64_t)rank * kGThreads + tid; e < (int64_t)c * c; e += (int64_t)C * kGThreads) {
      const int i = (int)(e % c), rk = (int)(e / c);
      Vr[(int64_t)rk * c + i] = J[(int64_t)col_of[rk] * ncol + i];
    }
  } else {
    // right vectors from the left ones (B = W J^T, W = U S  ->  J = B^T U S^-1), leading triplets
    for (int64_t e = (int64_t)rank * kGThreads + tid; e < (int64_t)c * c; e += (int64_t)C * kGThreads) {
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

// inner rotations formed once per pair (b threads, one more barrier per round) or by every
// updating thread (no extra barrier, the default: measured faster at every 2b; RSVD_GCL_ONCE=1)
static int gcl_once(int B2) {
  static const int env = [] {
    const char* e = getenv("RSVD_GCL_ONCE");
    return e ? atoi(e) : -1;
  }();
  return env >= 0 ? env : 0;
}

// bit 0: no early exit on small cosines (RSVD_GCL_MODE)
// cross-pair block rounds (RSVD_GCL_CROSS, default 1)
static int gcl_cross() {
  static const int env = [] {
    const char* e = getenv("RSVD_GCL_CROSS");
    return e ? atoi(e) : 1;
  }();
  return env;
}

static int gcl_mode() {
  static const int env = [] {
    const char* e = getenv("RSVD_GCL_MODE");
    return e ? atoi(e) : 0;
  }();
  return env;
}

template <int B2, bool DSM>
size_t gcl_smem(int RS) {
  constexpr int NT = B2 / 8, T = NT * (NT + 1) / 2, S = kGWarps / T > 0 ? kGWarps / T : 1;
  return ((DSM ? 2 : 1) * (size_t)B2 * RS + 2 * B2 * (B2 + 1) + B2 * (B2 + 4) + (size_t)S * B2 * B2) * 8;
}

template <int B2, bool DSM>
int launch_gcl_t(int C, const double* M, int64_t ldm, int trans, int r, int c, double* Ul, double* S, double* Vr,
                 double* W, double* J, double* sval, int* flags, int RS, DevStatus* status, cudaStream_t st,
                 int want_j) {
  const size_t smem = gcl_smem<B2, DSM>(RS);
  static std::atomic<bool> attr{false};  // set once per process (calls may come from several threads)
  if (!attr) {
    cudaFuncSetAttribute(k_jacobi_gcl<B2, DSM>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGSmemMax);
    cudaFuncSetAttribute(k_jacobi_gcl<B2, DSM>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kGThreads);
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
  const int nb = 2 * C;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_jacobi_gcl<B2, DSM>, M, ldm, trans, r, c, nb, RS, Ul, S, Vr, W, J,
                                           sval, flags, tol, 60, want_j, gcl_once(B2), gcl_mode(), gcl_cross(), status);
  return e == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

}  // namespace

// cluster size and block width for a c-column core: b = ceil(c / 2C) rounded up to a multiple
// of 4 (b <= 16); cost model per outer sweep (cycles, B200): (2C - 1) block rounds, each B2 - 1
// inner rounds (~350) plus the two r x B2 x B2 DMMA products, the pair's load / store and the
// cluster barrier
void gcl_plan(int r, int c, int* C_out, int* b_out) {
  double best = 1e300;
  int bc = 16, bb = 16;
  for (int C : {4, 8, 16}) {
    int b = (c + 2 * C - 1) / (2 * C);
    b = (b + 3) & ~3;
    if (b > 16 || b < 4) continue;
    const int B2 = 2 * b;
    const double per_round = (B2 - 1) * 350.0 + 2.0 * r * B2 * B2 / 48.0 + 2.0 * r * B2 * 8 / 48.0 + 1500.0;
    const double cost = (2 * C - 1) * per_round;
    if (cost < best) { best = cost; bc = C; bb = b; }
  }
  *C_out = bc;
  *b_out = bb;
}

int launch_jacobi_gcl(const double* M, int64_t ldm, int trans, int r, int c, double* Ul, double* S, double* Vr,
                      double* scratch, DevStatus* status, cudaStream_t st, int want_j) {
  if (c < 1 || c > kGMaxC || r < c || r > kGMaxC) return RSVD_E_ARG;
  int C, b;
  gcl_plan(r, c, &C, &b);
  if (getenv("RSVD_GCL_C")) {
    C = atoi(getenv("RSVD_GCL_C"));
    b = ((c + 2 * C - 1) / (2 * C) + 3) & ~3;
    if (b > 16 || b < 4 || (C != 4 && C != 8 && C != 16)) return RSVD_E_ARG;
  }
  const int ncol = 2 * C * b;
  double* W = scratch;                              // r x ncol (<= 512 x 512)
  double* J = W + (int64_t)r * kGMaxC;              // ncol x ncol
  double* sval = J + (int64_t)kGMaxC * kGMaxC;      // 2 * kGMaxC
  int* flags = reinterpret_cast<int*>(sval + 2 * kGMaxC);
  // DSM (two pair buffers per CTA, J rows carried when wanted) when it fits in shared memory
  const int r8 = (r + 7) & ~7;
  const int RSd = r8 + (want_j ? ncol : 0) + 4, RSg = r8 + 4;
#define GCL_CASE(B2V)                                                                                             \
  case B2V:                                                                                                       \
    return gcl_smem<B2V, true>(RSd) <= (size_t)kGSmemMax - 4096                                                   \
               ? launch_gcl_t<B2V, true>(C, M, ldm, trans, r, c, Ul, S, Vr, W, J, sval, flags, RSd, status, st,    \
                                         want_j)                                                                  \
               : launch_gcl_t<B2V, false>(C, M, ldm, trans, r, c, Ul, S, Vr, W, J, sval, flags, RSg, status, st,   \
                                          want_j);
  switch (2 * b) {
    GCL_CASE(8)
    GCL_CASE(16)
    GCL_CASE(24)
    GCL_CASE(32)
    default: return RSVD_E_ARG;
  }
#undef GCL_CASE
}

}  // namespace rsvd
