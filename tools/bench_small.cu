// Microbenchmark of the small kernels (phase timing with %globaltimer). Built with
//   nvcc -DRSVD_PHASE_TIMING ... tools/bench_small.cu paper_1804_07531_b200/csrc/small_kernels.cu
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_1804_07531_b200/csrc/internal.h"
namespace rsvd {
int launch_cholqr_pass(const double*, int64_t, double*, int64_t, int64_t, int, const double*, double*, unsigned*, double, double, int, double*, double*, DevStatus*, cudaStream_t);
int cholqr_pass_ctas(int64_t rows);
void read_phases(unsigned long long* out);
void reset_phases();
int launch_jacobi_t(const double* M, int64_t ldm, int trans, int r, int c, double* Ul, double* S, double* Vr, double* scratch, DevStatus* status, cudaStream_t st, int want_j);
}
using namespace rsvd;
int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 4000;
  const int w = argc > 2 ? atoi(argv[2]) : 30;
  std::vector<double> h(rows * w);
  std::mt19937_64 g(1); std::normal_distribution<double> nd;
  for (auto& x : h) x = nd(g);
  double *Y, *T, *slots, *R, *Ri, *R2, *R2i; unsigned* cnt; DevStatus* st;
  cudaMalloc(&Y, rows * w * 8); cudaMalloc(&T, rows * w * 8); cudaMalloc(&slots, 148 * 64 * 64 * 8);
  cudaMalloc(&R, 64 * 64 * 8); cudaMalloc(&Ri, 64 * 64 * 8); cudaMalloc(&R2, 64 * 64 * 8); cudaMalloc(&R2i, 64 * 64 * 8);
  cudaMalloc(&cnt, 256); cudaMemset(cnt, 0, 256); cudaMalloc(&st, sizeof(DevStatus)); cudaMemset(st, 0, sizeof(DevStatus));
  cudaMemcpy(Y, h.data(), rows * w * 8, cudaMemcpyHostToDevice);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int variant = 0; variant < 2; ++variant) {
    const double* Rin = variant ? Ri : nullptr;
    for (int it = 0; it < 3; ++it) launch_cholqr_pass(Y, rows, T, rows, rows, w, Rin, slots, cnt, 1e-12, 0.0, 0, variant ? R2 : R, variant ? R2i : Ri, st, s);
    cudaStreamSynchronize(s);
    reset_phases();
    cudaEventRecord(e0, s);
    launch_cholqr_pass(Y, rows, T, rows, rows, w, Rin, slots, cnt, 1e-12, 0.0, 0, variant ? R2 : R, variant ? R2i : Ri, st, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long ph[16]; read_phases(ph);
    printf("cholqr_pass rows=%lld w=%d apply=%d G=%d: event %.1f us | main %.1f us, finisher reduce %.1f us, chol+inv %.1f us (after last main %.1f)\n",
           (long long)rows, w, variant, cholqr_pass_ctas(rows), ms * 1e3, (ph[1] - ph[0]) / 1e3, (ph[3] - ph[2]) / 1e3, (ph[4] - ph[3]) / 1e3, (ph[2] - ph[1]) / 1e3);
    // graph-free back-to-back timing of 20 launches
    cudaEventRecord(e0, s);
    for (int it = 0; it < 20; ++it) launch_cholqr_pass(Y, rows, T, rows, rows, w, Rin, slots, cnt, 1e-12, 0.0, 0, variant ? R2 : R, variant ? R2i : Ri, st, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("   back-to-back avg %.1f us\n", ms * 1e3 / 20);
    printf("   cycles: chol loop %llu, scale %llu, inverse %llu\n", ph[9] - ph[8], ph[10] - ph[9], ph[11] - ph[10]);
  }
  // jacobi on an upper-triangular w x w
  std::vector<double> m(w * w, 0.0);
  for (int j = 0; j < w; ++j) for (int i = 0; i <= j; ++i) m[j * w + i] = nd(g) * (i == j ? 3.0 : 1.0) * pow(0.8, j);
  double *M, *U, *S, *V, *scr; cudaMalloc(&M, w * w * 8); cudaMalloc(&U, w * w * 8); cudaMalloc(&S, w * 8); cudaMalloc(&V, w * w * 8); cudaMalloc(&scr, 2 * 256 * 256 * 8);
  cudaMemcpy(M, m.data(), w * w * 8, cudaMemcpyHostToDevice);
  for (int t = 0; t < 2; ++t) {
    for (int it = 0; it < 2; ++it) launch_jacobi_t(M, w, t, w, w, U, S, V, scr, st, s, 0);
    cudaEventRecord(e0, s);
    for (int it = 0; it < 10; ++it) launch_jacobi_t(M, w, t, w, w, U, S, V, scr, st, s, 0);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    DevStatus hs; cudaMemcpy(&hs, st, sizeof hs, cudaMemcpyDeviceToHost);
    printf("jacobi w=%d trans=%d: %.1f us, sweeps %d\n", w, t, ms * 1e3 / 10, hs.jacobi_sweeps);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
