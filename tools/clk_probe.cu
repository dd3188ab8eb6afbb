// Is a lone CTA running at full SM clock?  Compare clock64 cycles with %globaltimer ns.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(long long cycles, unsigned long long* out) {
  unsigned long long g0, g1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g0));
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
  long long t1 = clock64();
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = g1 - g0; }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16); unsigned long long h[2];
  for (int blocks : {1, 148}) {
    for (long long cyc : {20000LL, 200000LL, 2000000LL, 20000000LL}) {
      spin<<<blocks, 32>>>(cyc, d); cudaDeviceSynchronize();
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("blocks %3d  %9llu cycles in %9llu ns  -> %.0f MHz\n", blocks, h[0], h[1], h[0] * 1e3 / (double)h[1]);
    }
  }
  return 0;
}
