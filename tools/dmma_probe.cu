// DMMA (mma.sync m8n8k4 f64) latency / issue probe on one SM: dependent chain vs N independent
// chains per warp, 1 or 8 warps.
#include <cstdio>
#include <cuda_runtime.h>
__device__ double sinkd;
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NCH>
__global__ void k(int n, long long* out) {
  double acc[NCH][2];
  for (int c = 0; c < NCH; ++c) acc[c][0] = acc[c][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-3;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) dmma(acc[c][0], acc[c][1], a, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  double s = 0; for (int c = 0; c < NCH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.0) sinkd = s;
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  auto run = [&](auto kern, int threads, const char* nm, int nch) {
    long long h = 0; const int n = 2000;
    kern<<<1, threads>>>(10, d); cudaDeviceSynchronize();
    kern<<<1, threads>>>(n, d); cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-26s %7.1f clk/iter  %6.2f clk/DMMA per warp  (%d threads)\n", nm, (double)h / n, (double)h / n / nch, threads);
  };
  run(k<1>, 32, "chain x1", 1); run(k<2>, 32, "chains x2", 2); run(k<4>, 32, "chains x4", 4);
  run(k<8>, 32, "chains x8", 8); run(k<16>, 32, "chains x16", 16);
  run(k<1>, 256, "chain x1, 8 warps", 1); run(k<4>, 256, "chains x4, 8 warps", 4); run(k<8>, 256, "chains x8, 8 warps", 8);
  run(k<8>, 512, "chains x8, 16 warps", 8); run(k<8>, 1024, "chains x8, 32 warps", 8);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
