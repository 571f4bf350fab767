// Microbenchmark of the fused panel kernel (panel.cuh) on one synthetic chunk:
// phase clocks of CTA 0 + event time of the launch.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DGMRF_PANEL_CLOCKS \
//        -I paper_2503_08343_b200/csrc tools/panel_bench.cu -o tools/panel_bench
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "panel.cuh"

using namespace gmrf;

int main(int argc, char** argv) {
  const int nbelow = argc > 1 ? atoi(argv[1]) : 2000;
  const int w = 64, rows = w + nbelow;
  std::vector<double> h(static_cast<size_t>(rows) * w);
  for (int j = 0; j < w; ++j)
    for (int i = 0; i < rows; ++i)
      h[i + static_cast<size_t>(j) * rows] = (i == j) ? 100.0 : 0.01 * ((i * 7 + j * 13) % 17 - 8);
  double *d, *diag;
  int* status;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&diag, 64 * 8);
  cudaMalloc(&status, 4);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  std::vector<PanelTask> tasks;
  for (int t = 0; t == 0 || t * kTrsmRows < nbelow; ++t) tasks.push_back({d, rows, w, nbelow, t, 0});
  PanelTask* dt;
  cudaMalloc(&dt, tasks.size() * sizeof(PanelTask));
  cudaMemcpy(dt, tasks.data(), tasks.size() * sizeof(PanelTask), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_potrf_trsm<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       panel_smem_bytes<64>());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_potrf_trsm<64><<<static_cast<unsigned>(tasks.size()), 128, panel_smem_bytes<64>()>>>(
        dt, status, diag);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long clk[8];
    cudaMemcpyFromSymbol(clk, g_panel_clk, sizeof(clk));
    printf("rep %d: %.1f us | load %lld  chol %lld [a0 %lld b0 %lld rest %lld] publish %lld  trsm %lld  store %lld cycles\n",
           rep, ms * 1e3, clk[1] - clk[0], clk[2] - clk[1], clk[6] - clk[1], clk[7] - clk[6], clk[2] - clk[7], clk[3] - clk[2], clk[4] - clk[3],
           clk[5] - clk[4]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
