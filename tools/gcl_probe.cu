// Phase timing of the Gram-block cluster Jacobi (k_jacobi_gcl) per block round.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRSVD_GCL_TIMING \
//      -I paper_1804_07531_b200/csrc -o tools/gcl_probe tools/gcl_probe.cu
#include "../paper_1804_07531_b200/csrc/jacobi_gcl.cu"

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

int main(int argc, char** argv) {
  std::vector<int> widths;
  for (int i = 1; i < argc; ++i) widths.push_back(atoi(argv[i]));
  if (widths.empty()) widths = {60, 120, 140, 250, 500};
  double *dM, *dU, *dS, *dV, *dscr;
  rsvd::DevStatus* dst;
  cudaMalloc(&dM, 512 * 512 * 8);
  cudaMalloc(&dU, 512 * 512 * 8);
  cudaMalloc(&dS, 512 * 8);
  cudaMalloc(&dV, 512 * 512 * 8);
  cudaMalloc(&dscr, (2 * 512 * 512 + 4096) * 8);
  cudaMalloc(&dst, sizeof(rsvd::DevStatus));
  for (int w : widths) {
    std::mt19937_64 g(7);
    std::normal_distribution<double> nd;
    std::vector<double> M((size_t)w * w);
    for (int j = 0; j < w; ++j)
      for (int i = 0; i < w; ++i) M[(size_t)j * w + i] = nd(g) * (exp(-j / (w / 2.5)) + 1e-6);
    cudaMemcpy(dM, M.data(), M.size() * 8, cudaMemcpyHostToDevice);
    for (int want_j = 0; want_j < 2; ++want_j) {
      for (int it = 0; it < 2; ++it)
        rsvd::launch_jacobi_gcl(dM, w, 0, w, w, dU, dS, dV, dscr, dst, 0, want_j);
      unsigned long long z[8] = {};
      cudaMemcpyToSymbol(rsvd::gcl_ph, z, sizeof(z));
      cudaMemset(dst, 0, sizeof(rsvd::DevStatus));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      const int rc = rsvd::launch_jacobi_gcl(dM, w, 0, w, w, dU, dS, dV, dscr, dst, 0, want_j);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long ph[8];
      cudaMemcpyFromSymbol(ph, rsvd::gcl_ph, sizeof(ph));
      rsvd::DevStatus st;
      cudaMemcpy(&st, dst, sizeof(st), cudaMemcpyDeviceToHost);
      int C, b;
      rsvd::gcl_plan(w, w, &C, &b);
      if (getenv("RSVD_GCL_C")) {
        C = atoi(getenv("RSVD_GCL_C"));
        b = ((w + 2 * C - 1) / (2 * C) + 3) & ~3;
      }
      const double nbr = (double)st.jacobi_sweeps * (2 * C - 1);
      printf("w=%d J=%d rc=%d %s  %.3f ms  C=%d b=%d sweeps=%d  cycles/block round: load %.0f gram %.0f test %.0f "
             "inner %.0f apply %.0f store %.0f sync %.0f\n",
             w, want_j, rc, cudaGetErrorString(cudaGetLastError()), ms, C, b, st.jacobi_sweeps, ph[0] / nbr,
             ph[1] / nbr, ph[2] / nbr, ph[3] / nbr, ph[4] / nbr, ph[5] / nbr, ph[6] / nbr);
    }
  }
  return 0;
}
