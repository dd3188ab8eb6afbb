// Phase timing of k_orth_cluster (clock64 stamps of CTA 0, thread 0) on a random rows x w block.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRSVD_ORTH_TIMING -o tools/orth_probe tools/orth_probe.cu
#include "../paper_1804_07531_b200/csrc/orth_cluster.cu"
#include <cstdio>
#include <vector>
using namespace rsvd;
int chol_alone_main();
int gram_alone_main();
int main(int argc, char** argv) {
  if (argc > 4) return gram_alone_main();
  if (argc > 3) return chol_alone_main();
  const int rows = argc > 1 ? atoi(argv[1]) : 4000, w = argc > 2 ? atoi(argv[2]) : 30;
  const int ld = (rows + 31) / 32 * 32;
  std::vector<double> h((size_t)ld * w);
  unsigned s = 1;
  for (auto& x : h) { s = s * 1664525u + 1013904223u; x = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
  double *Y, *R, *Rw; DevStatus* st;
  cudaMalloc(&Y, h.size() * 8); cudaMalloc(&R, w * w * 8); cudaMalloc(&Rw, 2 * w * w * 8); cudaMalloc(&st, sizeof(DevStatus));
  cudaMemset(st, 0, sizeof(DevStatus));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(Y, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    int rc = launch_orth_cluster(Y, ld, rows, w, 0, 0.0, R, Rw, st, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long t[32]; cudaMemcpyFromSymbol(t, g_orth_t, sizeof(t));
    printf("rc %d err %s  total %.1f us | load %lld gram0 %lld sync %lld reduce0 %lld chol0 %lld sync %lld | "
           "apply+gram1 %lld sync %lld reduce1 %lld chol1 %lld sync %lld | final %lld sync %lld (cycles) || gram-dmma %lld gram-add %lld mirror %lld || chol-entry %lld pivot0 %lld pivots %lld inverse %lld\n",
           rc, cudaGetErrorString(cudaGetLastError()), ms * 1e3, t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3],
           t[5] - t[4], t[6] - t[5], t[8] - t[6], t[9] - t[8], t[10] - t[9], t[11] - t[10], t[12] - t[11],
           t[21] - t[20], t[22] - t[21], t[23] - t[1], t[24] - t[23], t[2] - t[24], t[15] - t[4], t[16] - t[15], t[13] - t[16], t[14] - t[13]);
    printf("   final split: apply %lld, sync %lld, stage %lld, product %lld\n", t[28] - t[20], t[29] - t[28], t[30] - t[29], t[21] - t[30]);
#ifdef RSVD_ORTH_GRAM_TWICE
    printf("   gram0 again (warm i-cache): %lld\n", t[31] - t[2]);
#endif
  }
}
// ---- standalone timing of the factorisation (single CTA, no cluster)
namespace rsvd { namespace {
template <int W>
__global__ void k_chol_alone(const double* Gin, int w, double* R, long long* t) {
  __shared__ double G[W * W], Ri[W * 64], bc[256];
  for (int e = threadIdx.x; e < W * W; e += blockDim.x) G[e] = Gin[e];
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x < 32 * chol_warps<W>()) chol_inv_cols<W>(G, w, 0.0, 1e-12, R, Ri, oc_ld(W), bc);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) t[0] = t1 - t0;
}
} }
int chol_alone_main() {
  const int W = 32;
  std::vector<double> h(W * W);
  for (int i = 0; i < W; ++i) for (int j = 0; j < W; ++j) h[j * W + i] = (i == j ? W : 0.0) + 1.0 / (1 + i + j);
  double *G, *R; long long* t; cudaMalloc(&G, W * W * 8); cudaMalloc(&R, W * W * 8); cudaMalloc(&t, 8);
  cudaMemcpy(G, h.data(), W * W * 8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    k_chol_alone<32><<<1, 256>>>(G, 30, R, t); long long ht; cudaMemcpy(&ht, t, 8, cudaMemcpyDeviceToHost);
    long long tt[32]; cudaMemcpyFromSymbol(tt, g_orth_t, sizeof(tt));
    printf("standalone chol+inv W=32: %lld cycles (pivots %lld, R out %lld, inverse %lld)\n", ht, tt[26]-tt[25], 0LL, tt[27]-tt[26]);
  }
  return 0;
}
namespace rsvd { namespace {
template <int W>
__global__ void k_gram_alone(int rpc, long long* t, double* out, double* gout, int64_t ldo) {
  extern __shared__ double sm[];
  double* G = sm;
  double* Yc = sm + W * W;
  constexpr int ld = oc_ld(W);
  for (int e = threadIdx.x; e < rpc * ld; e += blockDim.x) Yc[e] = 1e-3 * (e % 97);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long t0 = clock64();
  gram_tiles<W>(Yc, rpc, G, warp, lane >> 2, lane & 3);
  long long t1 = clock64();
  apply_rinv<W>(Yc, G, rpc, warp, lane >> 2, lane & 3, nullptr, 0, 0, 0);
  __syncthreads();
  long long t2 = clock64();
  apply_rinv<W>(Yc, G, rpc, warp, lane >> 2, lane & 3, gout, ldo, rpc, W);
  __syncthreads();
  long long t3 = clock64();
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; out[0] = G[5] + Yc[7]; }
}
} }
template <int W>
void gram_alone_w() {
  long long* t; double* o; double* go; cudaMalloc(&t, 24); cudaMalloc(&o, 8); cudaMalloc(&go, 4032 * 64 * 8);
  const int rpc = 256;
  size_t smem = (W * W + rpc * oc_ld(W)) * 8;
  cudaFuncSetAttribute(k_gram_alone<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for (int rep = 0; rep < 3; ++rep) {
    k_gram_alone<W><<<1, 256, smem>>>(rpc, t, o, go, 4032); long long ht[3]; cudaMemcpy(ht, t, 24, cudaMemcpyDeviceToHost);
    printf("standalone W=%d rpc=256: gram %lld cycles, apply %lld cycles, apply->global %lld cycles (%s)\n", W, ht[0], ht[1], ht[2], cudaGetErrorString(cudaGetLastError()));
  }
}
int gram_alone_main() {
  gram_alone_w<32>();
  gram_alone_w<64>();
  return 0;
}
