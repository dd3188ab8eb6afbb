// Experimental one-sided Jacobi round variants for r, c <= 64 (values + left vectors, no J).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/jac_small_probe tools/jac_small_probe.cu
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

__device__ unsigned long long g_ph[8];
template <int LPP, int RW, int FAST>
__global__ void __launch_bounds__(256) k_jac(const double* __restrict__ M, int r, int c, double* __restrict__ S,
                                             int* sweeps_out, double tol) {
  unsigned long long ph[7] = {0, 0, 0, 0, 0, 0, 0};
  long long tA = 0;
#ifdef TIMING
#define TS(i) { if (tid == 0) { const long long _t = clock64(); ph[i] += _t - tA; tA = _t; } }
#else
#define TS(i) {}
#endif
  constexpr int RS = LPP * RW + 4;  // padded column stride (bank spread)
  extern __shared__ double W[];     // 128 x RS
  const int tid = threadIdx.x, nt = blockDim.x;
  const int grp = tid / LPP, sl = tid % LPP;
  const unsigned gmask = (LPP == 32 ? 0xffffffffu : ((1u << LPP) - 1u)) << (tid & 31 & ~(LPP - 1));
  const int ce = c + (c & 1);
  const int npairs = ce >> 1, m1 = ce - 1;
  for (int e = tid; e < 128 * RS; e += nt) {
    const int i = e % RS, j = e / RS;
    W[e] = (i < r && j < c) ? M[(int64_t)j * r + i] : 0.0;
  }
  __syncthreads();
  const double tol2 = tol * tol;
  const bool active = grp < npairs;
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < m1; ++round) {
      if (tid == 0) tA = clock64();
      {
        int p, q;
        {
          int pp = round + grp; if (pp >= m1) pp -= m1;
          int qq = round - grp; if (qq < 0) qq += m1;
          p = grp == 0 ? round : min(pp, qq);
          q = grp == 0 ? m1 : max(pp, qq);
          if (!active) p = q = 0;
        }
        double* wp = W + p * RS;
        double* wq = W + q * RS;
        double x[RW], y[RW];
#pragma unroll
        for (int t = 0; t < RW; ++t) { x[t] = wp[sl + LPP * t]; y[t] = wq[sl + LPP * t]; }
        { double sink = x[RW - 1] + y[RW - 1]; asm volatile("" :: "d"(sink)); }
        TS(0);
        constexpr int NA = 2;   // independent accumulators per dot
        double aa[NA], bb[NA], cv[NA];
#pragma unroll
        for (int u = 0; u < NA; ++u) aa[u] = bb[u] = cv[u] = 0.0;
#pragma unroll
        for (int t = 0; t < RW; ++t) {
          aa[t % NA] = fma(x[t], x[t], aa[t % NA]);
          bb[t % NA] = fma(y[t], y[t], bb[t % NA]);
          cv[t % NA] = fma(x[t], y[t], cv[t % NA]);
        }
#pragma unroll
        for (int u = NA / 2; u > 0; u >>= 1)
#pragma unroll
          for (int v = 0; v < u; ++v) { aa[v] += aa[v + u]; bb[v] += bb[v + u]; cv[v] += cv[v + u]; }
        double a = aa[0], b = bb[0], cc = cv[0];
        asm volatile("" :: "d"(a), "d"(b), "d"(cc));
        TS(1);
        __syncwarp();
        if (FAST >= 3) {
          // column norms only steer the test and the angle: reduce them in fp32
          float af = (float)a, bf = (float)b;
#pragma unroll
          for (int o = LPP / 2; o > 0; o >>= 1) {
            af += __shfl_xor_sync(0xffffffffu, af, o, LPP);
            bf += __shfl_xor_sync(0xffffffffu, bf, o, LPP);
            cc += __shfl_xor_sync(0xffffffffu, cc, o, LPP);
          }
          a = af; b = bf;
        } else {
#pragma unroll
          for (int o = LPP / 2; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o, LPP);
            b += __shfl_xor_sync(0xffffffffu, b, o, LPP);
            cc += __shfl_xor_sync(0xffffffffu, cc, o, LPP);
          }
        }
        asm volatile("" :: "d"(a), "d"(b), "d"(cc));
        TS(2);
        if (active && cc * cc > tol2 * (a * b) && cc != 0.0) {
          rotated = 1;
          const double d = b - a, e2 = 2.0 * cc;
          double t;
          if (FAST >= 2) {
            // approximate fp64 MUFU ops: rho = 2c/|d|, t = rho / (1 + sqrt(1 + rho^2))
            double rd, rs, rt;
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(fmax(fabs(d), 1e-300)));
            double rho = fmin(fmax(e2 * rd, -1e100), 1e100);
            const double s1 = fma(rho, rho, 1.0);
            asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rs) : "d"(s1));
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rt) : "d"(1.0 + s1 * rs));
            t = (d < 0.0 ? -rho : rho) * rt;
          } else if (FAST) {
            // any t gives an exactly orthogonal rotation; fp32 fast-math, ratio clamped to fp32 range
            // ratio in fp32: |d| and e2 scaled into range by their common exponent first
            float rf = (float)e2 * __frcp_rn(fmaxf((float)fabs(d), 1e-30f));
            rf = fminf(fmaxf(rf, -1e30f), 1e30f);
            const float s = fmaf(rf, rf, 1.0f);
            const float sq = s * rsqrtf(s);
            t = copysign(1.0, d == 0.0 ? 1.0 : d) * (double)__fdividef(rf, 1.0f + sq);
          } else {
            const double ad = fabs(d);
            const float rf = (float)e2 / (float)ad;
            const float tf = rf / (1.0f + sqrtf(fmaf(rf, rf, 1.0f)));
            t = copysign(1.0, d) * (double)tf;
          }
          const double cs = rsqrt(fma(t, t, 1.0));
          const double sn = cs * t;
          asm volatile("" :: "d"(cs), "d"(sn));
          TS(3);
#pragma unroll
          for (int k = 0; k < RW; ++k) {
            wp[sl + LPP * k] = cs * x[k] - sn * y[k];
            wq[sl + LPP * k] = sn * x[k] + cs * y[k];
          }
          TS(4);
        }
      }
      TS(5);
      __syncthreads();
      TS(6);
    }
    if (!__syncthreads_or(rotated)) { ++sweep; break; }
  }
  for (int j = tid; j < c; j += nt) {
    double s = 0;
    for (int i = 0; i < r; ++i) s = fma(W[j * RS + i], W[j * RS + i], s);
    S[j] = sqrt(s);
  }
  if (tid == 0) {
    *sweeps_out = sweep;
    for (int i = 0; i < 7; ++i) g_ph[i] = ph[i];
  }
}


// Register-resident variant: thread group T keeps the "plus" column of its pair in registers
// across rounds and only the "minus" column moves through shared memory (round-robin positions:
// logical pair g holds plus = r+g, minus = r-g (mod m1), g = 0: (r, fixed)).  Moves per round:
// plus[g] -> plus[g-1] (stays in the thread group, whose logical index is (T - r) mod npairs),
// plus[0] -> minus[1], minus[g] -> minus[g+1], minus[npairs-1] -> plus[npairs-1], minus[0] stays
// at logical 0.  Slots Sp / Sm indexed by the NEW logical index, double-buffered by round parity.
template <int LPP, int RW>
__global__ void __launch_bounds__(256) k_jac_reg(const double* __restrict__ M, int r, int c, double* __restrict__ S,
                                                 int* sweeps_out, double tol) {
  constexpr int RS = LPP * RW + 4;
  extern __shared__ double sm[];
  double* Sm = sm;               // 2 x 32 x RS
  double* Sp = sm + 2 * 32 * RS; // 2 x RS (only logical npairs-1 uses it)
  double* Wf = Sp + 2 * RS;      // 64 x RS final columns
  const int tid = threadIdx.x;
  const int T = tid / LPP, sl = tid % LPP;
  const int ce = c + (c & 1);
  const int npairs = ce >> 1, m1 = ce - 1;
  const bool active = T < npairs;
  double x[RW], y[RW];
  auto colv = [&](int col, int i) -> double { return (i < r && col < c) ? M[(int64_t)col * r + i] : 0.0; };
  {
    const int pc = T, mc = T == 0 ? m1 : m1 - T;
#pragma unroll
    for (int t = 0; t < RW; ++t) {
      x[t] = active ? colv(pc, sl + LPP * t) : 0.0;
      y[t] = active ? colv(mc, sl + LPP * t) : 0.0;
    }
  }
  const double tol2 = tol * tol;
  int sweep = 0, R = 0, h = active ? T : 0;
  for (; sweep < 60; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < m1; ++round, ++R) {
      double a0 = 0.0, b0 = 0.0, c0 = 0.0, a1 = 0.0, b1 = 0.0, c1 = 0.0;
#pragma unroll
      for (int t = 0; t < RW; t += 2) {
        a0 = fma(x[t], x[t], a0); b0 = fma(y[t], y[t], b0); c0 = fma(x[t], y[t], c0);
        if (t + 1 < RW) { a1 = fma(x[t + 1], x[t + 1], a1); b1 = fma(y[t + 1], y[t + 1], b1); c1 = fma(x[t + 1], y[t + 1], c1); }
      }
      double a = a0 + a1, b = b0 + b1, cc = c0 + c1;
      __syncwarp();
#pragma unroll
      for (int o = LPP / 2; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o, LPP);
        b += __shfl_xor_sync(0xffffffffu, b, o, LPP);
        cc += __shfl_xor_sync(0xffffffffu, cc, o, LPP);
      }
      if (active && cc * cc > tol2 * (a * b) && cc != 0.0) {
        rotated = 1;
        const double d = b - a;
        double rd, rs, rt;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(fmax(fabs(d), 1e-300)));
        const double rho = fmin(fmax(2.0 * cc * rd, -1e100), 1e100);
        const double s1 = fma(rho, rho, 1.0);
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rs) : "d"(s1));
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rt) : "d"(1.0 + s1 * rs));
        const double tt = (d < 0.0 ? -rho : rho) * rt;
        const double cs = rsqrt(fma(tt, tt, 1.0));
        const double sn = cs * tt;
#pragma unroll
        for (int k = 0; k < RW; ++k) {
          const double u = x[k], v = y[k];
          x[k] = cs * u - sn * v;
          y[k] = sn * u + cs * v;
        }
      }
      // hand the moving columns to their next owners (slots by NEW logical index); predicated,
      // no divergent branches (a warp reaching the next round's shuffles diverged is very slow)
      double* sm_w = Sm + (R & 1) * 32 * RS;
      double* sp_w = Sp + (R & 1) * RS;
      {
        const bool h0 = h == 0, hl = (h == npairs - 1) && !h0, two = npairs > 1;
        double* ydst = h0 ? sm_w : (hl ? sp_w : sm_w + (h + 1) * RS);
#pragma unroll
        for (int t = 0; t < RW; ++t) {
          if (active) ydst[sl + LPP * t] = y[t];
          if (active && h0 && two) sm_w[RS + sl + LPP * t] = x[t];
        }
        __syncthreads();
        const int hn = h0 ? npairs - 1 : h - 1;
        const double* ysrc = sm_w + hn * RS;
#pragma unroll
        for (int t = 0; t < RW; ++t) {
          const double yn = ysrc[sl + LPP * t];
          y[t] = (active && two) ? yn : y[t];
          if (active && h0 && two) x[t] = sp_w[sl + LPP * t];
        }
        h = active ? hn : 0;
      }
    }
    if (!__syncthreads_or(rotated)) { ++sweep; break; }
  }
  if (active) {
    const int rr = R % m1;
    const int pc = h == 0 ? rr : (rr + h) % m1, mc = h == 0 ? m1 : ((rr - h) % m1 + m1) % m1;
#pragma unroll
    for (int t = 0; t < RW; ++t) { Wf[pc * RS + sl + LPP * t] = x[t]; Wf[mc * RS + sl + LPP * t] = y[t]; }
  }
  __syncthreads();
  for (int j = tid; j < c; j += blockDim.x) {
    double s = 0;
    for (int i = 0; i < r; ++i) s = fma(Wf[j * RS + i], Wf[j * RS + i], s);
    S[j] = sqrt(s);
  }
  if (tid == 0) *sweeps_out = sweep;
}

template <int LPP, int RW>
void run_reg(const char* name, const double* dM, int r, int c, const std::vector<double>& ref) {
  constexpr int RS = LPP * RW + 4;
  const int smem = (2 * 32 + 2 + 64) * RS * 8;
  cudaFuncSetAttribute(k_jac_reg<LPP, RW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  double* dS;
  int* dsw;
  cudaMalloc(&dS, 128 * 8);
  cudaMalloc(&dsw, 4);
  const int ce = c + (c & 1);
  const int threads = ((LPP * (ce / 2)) + 31) / 32 * 32;
  const double tol = 2.220446049250313e-16 * sqrt((double)r);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_jac_reg<LPP, RW><<<1, threads, smem>>>(dM, r, c, dS, dsw, tol);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) k_jac_reg<LPP, RW><<<1, threads, smem>>>(dM, r, c, dS, dsw, tol);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> S(c);
  int sw;
  cudaMemcpy(S.data(), dS, c * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&sw, dsw, 4, cudaMemcpyDeviceToHost);
  std::sort(S.begin(), S.end(), [](double a, double b) { return a > b; });
  double err = 0;
  for (int i = 0; i < c; ++i) err = std::max(err, fabs(S[i] - ref[i]) / ref[0]);
  printf("%-22s r=%d c=%d threads=%d  %8.1f us  sweeps=%d  err=%.2e  (%s)\n", name, r, c, threads, 1000.0 * ms / reps, sw,
         err, cudaGetErrorString(cudaGetLastError()));
  cudaFree(dS);
  cudaFree(dsw);
}

template <int LPP, int RW, int FAST>
void run(const char* name, const double* dM, int r, int c, const std::vector<double>& ref) {
  constexpr int RS = LPP * RW + 4;
  const int smem = 128 * RS * 8;
  cudaFuncSetAttribute(k_jac<LPP, RW, FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  double* dS;
  int* dsw;
  cudaMalloc(&dS, 128 * 8);
  cudaMalloc(&dsw, 4);
  const int ce = c + (c & 1);
  const int threads = ((LPP * (ce / 2)) + 31) / 32 * 32;
  const double tol = 2.220446049250313e-16 * sqrt((double)r);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_jac<LPP, RW, FAST><<<1, threads, smem>>>(dM, r, c, dS, dsw, tol);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) k_jac<LPP, RW, FAST><<<1, threads, smem>>>(dM, r, c, dS, dsw, tol);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> S(c);
  int sw;
  cudaMemcpy(S.data(), dS, c * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&sw, dsw, 4, cudaMemcpyDeviceToHost);
  std::sort(S.begin(), S.end(), [](double a, double b) { return a > b; });
  double err = 0;
  for (int i = 0; i < c; ++i) err = std::max(err, fabs(S[i] - ref[i]) / ref[0]);
  printf("%-22s r=%d c=%d threads=%d  %8.1f us  sweeps=%d  err=%.2e  (%s)\n", name, r, c, threads, 1000.0 * ms / reps, sw,
         err, cudaGetErrorString(cudaGetLastError()));
  unsigned long long ph[8];
  cudaMemcpyFromSymbol(ph, g_ph, sizeof(ph));
  const double rounds = (double)sw * (ce - 1);
  printf("    cycles/round: load %.0f dots %.0f shfl %.0f angle %.0f rot %.0f tail %.0f bar %.0f\n", ph[0] / rounds,
         ph[1] / rounds, ph[2] / rounds, ph[3] / rounds, ph[4] / rounds, ph[5] / rounds, ph[6] / rounds);
  cudaFree(dS);
  cudaFree(dsw);
}

int main(int argc, char** argv) {
  for (int w : {30, 60, 70, 120}) {
    // graded test core: R^T of QR of Yh diag(s) X^T, computed by the reference kernel below
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    const int r = w, c = w;
    std::vector<double> M(r * c);
    for (auto& v : M) v = nd(g);
    // grade the columns and reference singular values from a one-sided Jacobi on the host
    for (int j = 0; j < c; ++j)
      for (int i = 0; i < r; ++i) M[j * r + i] *= exp(-j / 10.0);
    std::vector<double> Wh = M;
    for (int sw = 0; sw < 60; ++sw) {
      bool rot = false;
      for (int p = 0; p < c - 1; ++p)
        for (int q = p + 1; q < c; ++q) {
          double a = 0, b = 0, cc = 0;
          for (int i = 0; i < r; ++i) { a += Wh[p * r + i] * Wh[p * r + i]; b += Wh[q * r + i] * Wh[q * r + i]; cc += Wh[p * r + i] * Wh[q * r + i]; }
          if (fabs(cc) <= 1e-15 * sqrt(a * b)) continue;
          rot = true;
          const double z = (b - a) / (2 * cc);
          const double t = (z >= 0 ? 1 : -1) / (fabs(z) + sqrt(1 + z * z));
          const double cs = 1 / sqrt(1 + t * t), sn = cs * t;
          for (int i = 0; i < r; ++i) {
            const double u = Wh[p * r + i], v = Wh[q * r + i];
            Wh[p * r + i] = cs * u - sn * v;
            Wh[q * r + i] = sn * u + cs * v;
          }
        }
      if (!rot) break;
    }
    std::vector<double> ref(c);
    for (int j = 0; j < c; ++j) {
      double s = 0;
      for (int i = 0; i < r; ++i) s += Wh[j * r + i] * Wh[j * r + i];
      ref[j] = sqrt(s);
    }
    std::sort(ref.begin(), ref.end(), [](double a, double b) { return a > b; });
    double* dM;
    cudaMalloc(&dM, M.size() * 8);
    cudaMemcpy(dM, M.data(), M.size() * 8, cudaMemcpyHostToDevice);
    if (w <= 32) {
      run<8, 4, 0>("lpp8 rw4 ieee", dM, r, c, ref);
      run<8, 4, 2>("lpp8 rw4 mufu64", dM, r, c, ref);
      run_reg<8, 4>("REG lpp8 rw4", dM, r, c, ref);
      run_reg<4, 8>("REG lpp4 rw8", dM, r, c, ref);
      run<8, 4, 3>("lpp8 rw4 mufu64+f32n", dM, r, c, ref);
      run<4, 8, 2>("lpp4 rw8 mufu64", dM, r, c, ref);
      run<4, 8, 3>("lpp4 rw8 mufu64+f32n", dM, r, c, ref);
    } else if (w > 64) {
      run<8, 16, 2>("lpp8 rw16 mufu64", dM, r, c, ref);
      run<4, 32, 2>("lpp4 rw32 mufu64", dM, r, c, ref);
    } else {
      run<8, 8, 0>("lpp8 rw8 ieee", dM, r, c, ref);
      run<8, 8, 3>("lpp8 rw8 mufu64+f32n", dM, r, c, ref);
      run<4, 16, 0>("lpp4 rw16 ieee", dM, r, c, ref);
      run<4, 16, 2>("lpp4 rw16 mufu64", dM, r, c, ref);
      run_reg<4, 16>("REG lpp4 rw16", dM, r, c, ref);
      run_reg<8, 8>("REG lpp8 rw8", dM, r, c, ref);
      run<4, 16, 3>("lpp4 rw16 mufu64+f32n", dM, r, c, ref);
    }
    cudaFree(dM);
  }
  return 0;
}
