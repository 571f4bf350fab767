// Microbenchmark of the panel kernels (panel.cuh) on one synthetic chunk:
// k_potrf_trsm (blocked, smem) vs k_panel_rows (row per thread), event time per
// launch and the max difference of their outputs.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DGMRF_PANEL_CLOCKS \
//        -I paper_2503_08343_b200/csrc tools/panel_bench.cu -o tools/panel_bench
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "panel.cuh"

using namespace gmrf;

int main(int argc, char** argv) {
  const int nbelow = argc > 1 ? atoi(argv[1]) : 2000;
  const int w = argc > 2 ? atoi(argv[2]) : 64, rows = w + nbelow;
  std::vector<double> h(static_cast<size_t>(rows) * w);
  for (int j = 0; j < w; ++j)
    for (int i = 0; i < rows; ++i)
      h[i + static_cast<size_t>(j) * rows] = (i == j) ? 100.0 : 0.01 * ((i * 7 + j * 13) % 17 - 8);
  double *d, *diag;
  int* status;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&diag, 64 * 8);
  cudaMalloc(&status, 4);
  const int sr = argc > 3 ? atoi(argv[3]) : 128;
  std::vector<PanelTask> tasks, tasks_r;
  for (int t = 0; t == 0 || t * kTrsmRows < nbelow; ++t) tasks.push_back({d, rows, w, nbelow, t, 0});
  for (int t = 0; t == 0 || t * sr < nbelow; ++t) tasks_r.push_back({d, rows, w, nbelow, t, 0});
  PanelTask *dt, *dtr;
  cudaMalloc(&dt, tasks.size() * sizeof(PanelTask));
  cudaMemcpy(dt, tasks.data(), tasks.size() * sizeof(PanelTask), cudaMemcpyHostToDevice);
  cudaMalloc(&dtr, tasks_r.size() * sizeof(PanelTask));
  cudaMemcpy(dtr, tasks_r.data(), tasks_r.size() * sizeof(PanelTask), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_potrf_trsm<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       panel_smem_bytes<64>());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<double> out[2];
  for (int kind = 0; kind < 2; ++kind) {
    for (int rep = 0; rep < 6; ++rep) {
      cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
      cudaEventRecord(e0);
      if (kind == 0)
        k_potrf_trsm<64><<<static_cast<unsigned>(tasks.size()), 128, panel_smem_bytes<64>()>>>(
            dt, status, diag);
      else
      {
        const unsigned g = static_cast<unsigned>(tasks_r.size());
        if (sr == 32)
          k_panel_rows<64, 32><<<g, nbelow == 0 ? 64 : panel_rows_threads<64, 32>()>>>(dtr, status, diag);
        else if (sr == 64)
          k_panel_rows<64, 64><<<g, nbelow == 0 ? 64 : panel_rows_threads<64, 64>()>>>(dtr, status, diag);
        else
          k_panel_rows<64, 128><<<g, nbelow == 0 ? 64 : panel_rows_threads<64, 128>()>>>(dtr, status, diag);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      long long clk[8];
      cudaMemcpyFromSymbol(clk, g_panel_clk, sizeof(clk));
      if (rep > 0 && kind == 1)
        printf("rows  rep %d: %.1f us (%zu CTAs) load %lld sweep %lld store %lld cycles\n", rep,
               ms * 1e3, tasks_r.size(), clk[1] - clk[0], clk[2] - clk[1], clk[3] - clk[2]);
      else if (rep > 0)
        printf("potrf rep %d: %.1f us (%zu CTAs)\n", rep, ms * 1e3, tasks.size());
    }
    out[kind].resize(h.size());
    cudaMemcpy(out[kind].data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  }
  {
    long long col[64];
    cudaMemcpyFromSymbol(col, g_panel_col, sizeof(col));
    printf("per-column cycles:");
    for (int j = 1; j < 64; ++j) printf(" %lld", col[j] - col[j - 1]);
    printf("\n");
  }
  double md = 0, mx = 0;
  for (size_t i = 0; i < h.size(); ++i) {
    md = fmax(md, fabs(out[0][i] - out[1][i]));
    mx = fmax(mx, fabs(out[0][i]));
  }
  printf("max |potrf - rows| = %.3e (max |x| %.3e)\nerr: %s\n", md, mx,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
