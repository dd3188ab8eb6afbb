// Latency of the Jacobi angle computation and of dependent shared-memory loads on B200 (one warp,
// dependent chain of N steps, clock64).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void angle_f64(double a, double b, double cc, double* cs, double* sn) {
  const double d = b - a;
  double rd, rsq, rt;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(fmax(fabs(d), 1e-300)));
  const double rho = fmin(fmax(2.0 * cc * rd, -1e100), 1e100);
  const double s1 = fma(rho, rho, 1.0);
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rsq) : "d"(s1));
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rt) : "d"(fma(s1, rsq, 1.0)));
  const double t = (d < 0.0 ? -rho : rho) * rt;
  *cs = rsqrt(fma(t, t, 1.0));
  *sn = *cs * t;
}
__device__ __forceinline__ void angle_f32(double a, double b, double cc, double* cs, double* sn) {
  const double d = b - a;
  double rd;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(fmax(fabs(d), 1e-300)));
  const float rho = (float)fmin(fmax(2.0 * cc * rd, -1e30), 1e30);
  const float tf = __fdividef(rho, 1.0f + sqrtf(fmaf(rho, rho, 1.0f)));
  const double t = (d < 0.0 ? -(double)tf : (double)tf);
  *cs = rsqrt(fma(t, t, 1.0));
  *sn = *cs * t;
}
template <int MODE>
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-3;
  __syncthreads();
  double a = 1.0 + threadIdx.x * 1e-3, b = 2.0, c = 0.3;
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (MODE == 0) { double cs, sn; angle_f64(a, b, c, &cs, &sn); a = 1.0 + cs * 1e-3; c = 0.3 + sn * 1e-3; }
    if (MODE == 1) { double cs, sn; angle_f32(a, b, c, &cs, &sn); a = 1.0 + cs * 1e-3; c = 0.3 + sn * 1e-3; }
    if (MODE == 2) { double v = sm[idx & 1023]; idx = (int)v + (idx & 7); a += v; }         // dependent LDS
    if (MODE == 3) { a = fma(a, 1.0000001, 1e-9); }                                        // dependent DFMA
    if (MODE == 4) { a = rsqrt(a + 1.0); }                                                 // full rsqrt
    if (MODE == 5) { __syncthreads(); a += 1.0; }                                          // barrier
  }
  long long t1 = clock64();
  out[threadIdx.x] = a + b + c;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8);
  const char* nm[] = {"angle fp64", "angle fp32-t", "dependent LDS", "dependent DFMA", "rsqrt fp64", "syncthreads(256)"};
  for (int m = 0; m < 6; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      const int n = 2000, th = (m == 5) ? 256 : 32;
      if (m == 0) k<0><<<1, th>>>(o, c, n);
      if (m == 1) k<1><<<1, th>>>(o, c, n);
      if (m == 2) k<2><<<1, th>>>(o, c, n);
      if (m == 3) k<3><<<1, th>>>(o, c, n);
      if (m == 4) k<4><<<1, th>>>(o, c, n);
      if (m == 5) k<5><<<1, th>>>(o, c, n);
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      if (rep) printf("%-18s %.1f cycles/step\n", nm[m], (double)h / n);
    }
  }
  return 0;
}
