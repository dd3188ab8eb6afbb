// Where does a 16-CTA "load 250x30 doubles per CTA + Gram" kernel spend its time?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ unsigned long long g_t[8];
__global__ void empty_k() {}
// MODE 0: cp.async 8B column-major gather into row-major smem; 1: LDG coalesced + STS; 2: mode 1 + ldg only timing
template <int MODE>
__global__ void __launch_bounds__(256) load_k(const double* __restrict__ Y, int ldy, int rows_per, int w, double* out) {
  extern __shared__ double T[];
  const int ld = 36;
  long long c0 = clock64();
  const double* base = Y + (size_t)blockIdx.x * rows_per;
  if (MODE == 0) {
    for (int c = 0; c < 32; ++c)
      for (int i = threadIdx.x; i < rows_per; i += 256)
        if (c < w) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa(T + i * ld + c)), "l"(base + (size_t)c * ldy + i) : "memory");
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  } else {
    for (int c = 0; c < w; ++c)
      for (int i = threadIdx.x; i < rows_per; i += 256) T[i * ld + c] = base[(size_t)c * ldy + i];
  }
  __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { g_t[0] = c1 - c0; }
  if (threadIdx.x == 0 && T[0] == 12345.0) out[0] = T[1];
}
int main() {
  const int rows = 4000, w = 30, G = 16, rp = rows / G;
  double *Y, *o; cudaMalloc(&Y, rows * 32 * 8); cudaMalloc(&o, 8); cudaMemset(Y, 0, rows * 32 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  cudaFuncSetAttribute(load_k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(load_k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); for (int i = 0; i < 100; ++i) empty_k<<<G, 256>>>(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("empty kernel x100: %.2f us each\n", ms * 10);
    unsigned long long t;
    cudaEventRecord(e0); for (int i = 0; i < 100; ++i) load_k<0><<<G, 256, rp * 36 * 8>>>(Y, rows, rp, w, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); cudaMemcpyFromSymbol(&t, g_t, 8); printf("cp.async gather: %.2f us each, in-kernel %llu cyc\n", ms * 10, t);
    cudaEventRecord(e0); for (int i = 0; i < 100; ++i) load_k<1><<<G, 256, rp * 36 * 8>>>(Y, rows, rp, w, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); cudaMemcpyFromSymbol(&t, g_t, 8); printf("ldg+sts: %.2f us each, in-kernel %llu cyc\n", ms * 10, t);
  }
  // graph of 10 empty kernels
  cudaStream_t s; cudaStreamCreate(&s); cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 20; ++i) empty_k<<<G, 256, 0, s>>>();
  cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
  cudaEventRecord(e0, s); for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("graph of 20 empty kernels: %.2f us per kernel node\n", ms * 1e3 / 200);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
