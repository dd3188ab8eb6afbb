// Per-CTA timeline of k_view_ax (%globaltimer stamps, -DRSVD_VIEW_TIMING): start skew, time to the
// first consumed stage, per-unit durations and the spread of CTA end times, for one m x n x w view.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRSVD_VIEW_TIMING \
//          -o tools/view_timeline tools/view_timeline.cu -lcuda
// run:   tools/view_timeline [m n w [gap]]   ("gap": event time of R back-to-back launches, plain /
//        interleaved with a 1-CTA kernel / with programmatic dependent launch / in a CUDA graph)
#include "../paper_1804_07531_b200/csrc/view_kernels.cu"
#include <algorithm>
#include <cstdio>
#include <functional>
#include <vector>
using namespace rsvd;
__global__ void k_tiny(double* p) { if (threadIdx.x == 0) p[0] += 1.0; }
static float timed(cudaEvent_t e0, cudaEvent_t e1, cudaStream_t st, const std::function<void()>& f) {
  cudaEventRecord(e0, st);
  f();
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f;
}
int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atol(argv[1]) : 4000, n = argc > 2 ? atol(argv[2]) : 4000;
  const int w = argc > 3 ? atoi(argv[3]) : 30;
  double *A, *X, *out;
  cudaMalloc(&A, m * n * 8);
  cudaMalloc(&X, (size_t)w * n * 8);
  std::vector<double> h((size_t)w * n);
  unsigned s = 1;
  for (auto& x : h) { s = s * 1664525u + 1013904223u; x = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
  cudaMemcpy(X, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(A, 0, m * n * 8);
  ViewArgs a;
  a.A = A; a.rows = m; a.n = n; a.lda = n; a.X = X; a.ldx = n; a.w = w; a.grid_cap = 148;
  plan_view(VIEW_AX, m, n, w, 148, &a.S, &a.KTS);
  cudaMalloc(&out, (size_t)a.S * m * w * 8);
  a.out = out; a.ldo = m; a.slot_stride = m * w;
  double* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double ideal_us = 2.0 * m * n * ((w + 7) / 8 * 8) / 37.05e12 * 1e6;
  printf("m %ld n %ld w %d  S %d KTS %d  padded-DMMA ideal %.1f us\n", (long)m, (long)n, w, a.S, a.KTS, ideal_us);
  if (argc > 4) {  // launch-gap experiment
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    double* tiny;
    cudaMalloc(&tiny, 8);
    using C = AxCfg<4>;
    CUtensorMap tmA, tmX;
    make_map(&tmA, a.A, a.n, a.rows, a.lda, C::BM);
    make_map(&tmX, a.X, a.n, a.w, a.ldx, C::WP);
    cudaFuncSetAttribute(k_view_ax<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    const int RB = (int)((m + C::BM - 1) / C::BM), KT = (int)((n + kBK - 1) / kBK);
    const int grid = std::min(RB * a.S, 148);
    auto plain = [&]() {
      k_view_ax<4><<<grid, kThreads, C::SMEM, st>>>(tmA, tmX, a.out, a.ldo, a.slot_stride, (int)m, w, RB, a.S, KT, a.KTS, 0);
    };
    auto pdl = [&]() {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid; cfg.blockDim = kThreads; cfg.dynamicSmemBytes = C::SMEM; cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_view_ax<4>, tmA, tmX, a.out, a.ldo, a.slot_stride, (int)m, w, RB, a.S, KT, a.KTS, 0);
    };
    for (int R : {1, 2, 8}) {
      float t[6] = {};
      for (int rep = 0; rep < 4; ++rep) {
        cudaMemsetAsync(flush, rep, 256 << 20, st);
        t[0] = timed(e0, e1, st, [&] { for (int i = 0; i < R; ++i) plain(); });
        cudaMemsetAsync(flush, rep, 256 << 20, st);
        t[1] = timed(e0, e1, st, [&] { for (int i = 0; i < R; ++i) { k_tiny<<<1, 32, 0, st>>>(tiny); plain(); } });
        cudaMemsetAsync(flush, rep, 256 << 20, st);
        t[2] = timed(e0, e1, st, [&] { for (int i = 0; i < R; ++i) pdl(); });
        cudaMemsetAsync(flush, rep, 256 << 20, st);
        t[3] = timed(e0, e1, st, [&] { for (int i = 0; i < R; ++i) { k_tiny<<<1, 32, 0, st>>>(tiny); pdl(); } });
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < R; ++i) { k_tiny<<<1, 32, 0, st>>>(tiny); pdl(); }
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaMemsetAsync(flush, rep, 256 << 20, st);
        t[4] = timed(e0, e1, st, [&] { cudaGraphLaunch(ge, st); });
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < R; ++i) { k_tiny<<<1, 32, 0, st>>>(tiny); plain(); }
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaMemsetAsync(flush, rep, 256 << 20, st);
        t[5] = timed(e0, e1, st, [&] { cudaGraphLaunch(ge, st); });
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
      }
      printf("R %d  per launch (us): plain %.1f | tiny+plain %.1f | pdl %.1f | tiny+pdl %.1f | graph(tiny+pdl) %.1f | graph(tiny+plain) %.1f  %s\n", R,
             t[0] / R, t[1] / R, t[2] / R, t[3] / R, t[4] / R, t[5] / R, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
  }
  for (int rep = 0; rep < 6; ++rep) {
    cudaMemset(flush, rep, 256 << 20);
    unsigned long long z[160][9] = {};
    cudaMemcpyToSymbol(g_view_t, z, sizeof(z));
    cudaEventRecord(e0);
    int rc = launch_view_ax(a, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long t[160][9];
    cudaMemcpyFromSymbol(t, g_view_t, sizeof(t));
    const int G = std::min(148, a.S * (int)((m + 127) / 128));
    unsigned long long t0 = ~0ull, tend = 0;
    for (int b = 0; b < G; ++b) { t0 = std::min(t0, t[b][0]); tend = std::max(tend, t[b][8]); }
    std::vector<double> st, first, ends, u0, u1;
    for (int b = 0; b < G; ++b) {
      st.push_back((t[b][0] - t0) * 1e-3);
      first.push_back((t[b][1] - t[b][0]) * 1e-3);
      ends.push_back((t[b][8] - t0) * 1e-3);
      u0.push_back((t[b][2] - t[b][1]) * 1e-3);
      if (t[b][3]) u1.push_back((t[b][3] - t[b][2]) * 1e-3);
    }
    auto q = [](std::vector<double> v, double f) { std::sort(v.begin(), v.end()); return v.empty() ? 0.0 : v[(size_t)(f * (v.size() - 1))]; };
    printf("rc %d %s event %.1f us | span %.1f us | start skew max %.2f | first-stage wait min/med/max %.2f/%.2f/%.2f | "
           "unit0 (from first stage) min/med/max %.2f/%.2f/%.2f | unit1 min/med/max %.2f/%.2f/%.2f | end min/med/max %.1f/%.1f/%.1f\n",
           rc, cudaGetErrorString(cudaGetLastError()), ms * 1e3, (tend - t0) * 1e-3, q(st, 1.0), q(first, 0), q(first, 0.5),
           q(first, 1.0), q(u0, 0), q(u0, 0.5), q(u0, 1.0), q(u1, 0), q(u1, 0.5), q(u1, 1.0), q(ends, 0), q(ends, 0.5), q(ends, 1.0));
  }
  return 0;
}
