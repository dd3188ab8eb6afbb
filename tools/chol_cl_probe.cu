// Phase timing of the cluster Cholesky + inverse (k_chol_cl) per cluster rank.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRSVD_CHOL_TIMING \
//      -I paper_1804_07531_b200/csrc -o tools/chol_cl_probe tools/chol_cl_probe.cu
#include "../paper_1804_07531_b200/csrc/chol_big.cu"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

int main(int argc, char** argv) {
  std::vector<int> widths;
  for (int i = 1; i < argc; ++i) widths.push_back(atoi(argv[i]));
  if (widths.empty()) widths = {70, 140, 250, 500};
  double *dG, *dR, *dRi;
  rsvd::DevStatus* dst;
  cudaMalloc(&dG, 512 * 512 * 8);
  cudaMalloc(&dR, 512 * 512 * 8);
  cudaMalloc(&dRi, 512 * 512 * 8);
  cudaMalloc(&dst, sizeof(rsvd::DevStatus));
  for (int w : widths) {
    // G = Y^T Y of a graded Gaussian Y (rows = 2w)
    std::mt19937_64 gen(5);
    std::normal_distribution<double> nd;
    const int rows = 2 * w;
    std::vector<double> Y((size_t)rows * w), G((size_t)w * w, 0.0);
    for (int j = 0; j < w; ++j)
      for (int i = 0; i < rows; ++i) Y[(size_t)j * rows + i] = nd(gen) * pow(10.0, -3.0 * j / w);
    for (int a = 0; a < w; ++a)
      for (int b = 0; b < w; ++b) {
        double s = 0;
        for (int i = 0; i < rows; ++i) s += Y[(size_t)a * rows + i] * Y[(size_t)b * rows + i];
        G[(size_t)b * w + a] = s;
      }
    cudaMemcpy(dG, G.data(), G.size() * 8, cudaMemcpyHostToDevice);
    cudaStream_t st = 0;
    for (int rep = 0; rep < 3; ++rep) rsvd::launch_chol_cl(dG, nullptr, w, 1e-12, dR, dRi, dst, st, 0.0);
    cudaDeviceSynchronize();
    unsigned long long z[128] = {};
    cudaMemcpyToSymbol(rsvd::chol_ph, z, sizeof z);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 10;
    cudaEventRecord(e0);
    for (int rep = 0; rep < reps; ++rep) rsvd::launch_chol_cl(dG, nullptr, w, 1e-12, dR, dRi, dst, st, 0.0);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long ph[128];
    cudaMemcpyFromSymbol(ph, rsvd::chol_ph, sizeof ph);
    // check: |R^T R - G| / |G| and |R Rinv - I|
    std::vector<double> R((size_t)w * w), Ri((size_t)w * w);
    cudaMemcpy(R.data(), dR, R.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(Ri.data(), dRi, Ri.size() * 8, cudaMemcpyDeviceToHost);
    double eg = 0, ng = 0, ei = 0;
    for (int a = 0; a < w; ++a)
      for (int b = 0; b < w; ++b) {
        double s = 0, t = 0;
        for (int k = 0; k < w; ++k) {
          s += R[(size_t)a * w + k] * R[(size_t)b * w + k];
          t += R[(size_t)k * w + a] * Ri[(size_t)b * w + k];
        }
        eg += (s - G[(size_t)b * w + a]) * (s - G[(size_t)b * w + a]);
        ng += G[(size_t)b * w + a] * G[(size_t)b * w + a];
        ei = fmax(ei, fabs(t - (a == b)));
      }
    // the one-CTA kernel on the same G for reference
    std::vector<double> R2((size_t)w * w);
    rsvd::launch_chol_big(dG, nullptr, w, 1e-12, dR, dRi, dst, st, 0.0);
    cudaMemcpy(R2.data(), dR, R2.size() * 8, cudaMemcpyDeviceToHost);
    double dmax = 0;
    int da = -1, db = -1;
    for (int a = 0; a < w; ++a)
      for (int b = 0; b < w; ++b)
        if (fabs(R[(size_t)b * w + a] - R2[(size_t)b * w + a]) > dmax) {
          dmax = fabs(R[(size_t)b * w + a] - R2[(size_t)b * w + a]);
          da = a;
          db = b;
        }
    printf("  max |R_cl - R_big| = %.3e at (%d, %d): %.6e vs %.6e\n", dmax, da, db, da >= 0 ? R[(size_t)db * w + da] : 0.0,
           da >= 0 ? R2[(size_t)db * w + da] : 0.0);
    const int nb = (w + 31) / 32;
    printf("w=%d nb=%d: %.1f us per launch; |R^T R - G|/|G| = %.2e, max|R Rinv - I| = %.2e\n", w, nb,
           1000.0 * ms / reps, sqrt(eg / ng), ei);
    const char* nm[7] = {"prologue", "factor", "wait_X", "panel", "wait_R", "update", "inverse"};
    for (int r : {0, nb / 2, nb - 1}) {
      printf("  rank %2d:", r);
      for (int p = 0; p < 7; ++p) printf(" %s %.0f", nm[p], (double)ph[r * 8 + p] / reps);
      printf("\n");
    }
  }
  return 0;
}
