// Microbenchmark of the DMMA tile GEMM (kernels.cu) on synthetic task lists
// shaped like the factorization's launches:
//   update64 : 64x64 tiles, K=64, lower trapezoid of a 2048-wide trailing block
//   small    : 18k tiles 48x48, K=32 (bottom-of-tree SYRKs)
//   syrk1k   : 64x64 tiles, K=1024, lower triangle of a 1024x1024 update
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2503_08343_b200/csrc tools/gemm_bench.cu -o tools/gemm_bench
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../tools/gemm_variants.cuh"

using namespace gmrf;

typedef void (*KFn)(const GemmTask*);
struct Var {
  const char* name;
  KFn fn;
  int threads;
  int smem = 0;
};
static std::vector<Var> g_vars;

static void run(const char* name, std::vector<GemmTask>& tasks, double flops) {
  GemmTask* dt;
  cudaMalloc(&dt, tasks.size() * sizeof(GemmTask));
  cudaMemcpy(dt, tasks.data(), tasks.size() * sizeof(GemmTask), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (const Var& v : g_vars) {
    float best = 1e9f;
    for (int rep = 0; rep < 8; ++rep) {
      cudaEventRecord(e0);
      v.fn<<<static_cast<unsigned>(tasks.size()), v.threads, v.smem>>>(dt);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("%-9s %-14s %6zu tiles  %8.1f us  %6.2f TF/s  (%s)\n", name, v.name, tasks.size(),
           best * 1e3, flops / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  cudaFree(dt);
}

int main() {
  g_vars = {{"base", k_gemm_tiles, 128},
            {"var_ref", k_gemm_var<2, 2, 16, false, 4, false, 0>, 128},
            {"nomul", k_gemm_var<2, 2, 16, false, 4, false, 3>, 128},
            {"nomul_nv", k_gemm_var<2, 2, 16, false, 4, true, 3>, 128},
            {"nomul_w2x4", k_gemm_var<2, 4, 16, false, 3, true, 3>, 256},
            {"ld16", k_gemm_var<2, 2, 16, false, 4, false, 4>, 128}
            };
  cudaFuncSetAttribute(k_gemm_ms<3, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_ms_smem<3>());
  cudaFuncSetAttribute(k_gemm_ms<4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_ms_smem<4>());
  cudaFuncSetAttribute(k_gemm_ms<5, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_ms_smem<5>());
  cudaFuncSetAttribute(k_gemm_ms<5, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_ms_smem<5>());
  const int64_t N = 4096;
  double* buf;
  cudaMalloc(&buf, N * N * sizeof(double) * 3);
  cudaMemset(buf, 0, N * N * sizeof(double) * 3);
  double* A = buf;
  double* C = buf + N * N;
  {  // update64: trailing block 2048 wide, rows 2048, K = 64 (A panel = 2048 x 64)
    std::vector<GemmTask> t;
    double fl = 0;
    const int w = 2048;
    for (int jb = 0; jb < w; jb += 64)
      for (int ib = jb; ib < w; ib += 64) {
        GemmTask g{};
        g.c = C + ib + static_cast<int64_t>(jb) * w;
        g.ldc = w;
        g.m = 64;
        g.n = 64;
        g.a[0] = A + ib;
        g.lda[0] = w;
        g.b[0] = A + jb;
        g.ldb[0] = w;
        g.k[0] = 64;
        g.flags = 2;
        g.alpha = -1.0;
        g.beta = 1.0;
        t.push_back(g);
        fl += 2.0 * 64 * 64 * 64;
      }
    run("update64", t, fl);
    t.resize(500);
    run("upd64x500", t, 2.0 * 64 * 64 * 64 * 500);
  }
  {  // small: 18k independent 48x48 K=32 tiles spread over the buffer
    std::vector<GemmTask> t;
    double fl = 0;
    for (int q = 0; q < 18000; ++q) {
      GemmTask g{};
      const int64_t off = (static_cast<int64_t>(q) * 4099) % (N * N - 64 * 200);
      g.c = C + off;
      g.ldc = 97;
      g.m = 48;
      g.n = 48;
      g.a[0] = A + off;
      g.lda[0] = 97;
      g.b[0] = A + off + 50;
      g.ldb[0] = 97;
      g.k[0] = 32;
      g.flags = 2;
      g.alpha = -1.0;
      g.beta = 1.0;
      t.push_back(g);
      fl += 2.0 * 48 * 48 * 32;
    }
    run("small", t, fl);
  }
  {  // syrk1k: U (1024 x 1024 lower) -= L_R L_Rᵀ, K = 1024
    std::vector<GemmTask> t;
    double fl = 0;
    const int r = 1024;
    for (int jb = 0; jb < r; jb += 64)
      for (int ib = jb; ib < r; ib += 64) {
        GemmTask g{};
        g.c = C + ib + static_cast<int64_t>(jb) * r;
        g.ldc = r;
        g.m = 64;
        g.n = 64;
        g.a[0] = A + ib;
        g.lda[0] = 2048;
        g.b[0] = A + jb;
        g.ldb[0] = 2048;
        g.k[0] = 1024;
        g.flags = 2;
        g.alpha = -1.0;
        g.beta = 1.0;
        t.push_back(g);
        fl += 2.0 * 64 * 64 * 1024;
      }
    run("syrk1k", t, fl);
    std::vector<GemmTask> t4;
    for (int c = 0; c < 4; ++c)
      for (GemmTask g : t) {
        g.c += static_cast<int64_t>(c) * 1024 * 1024 * 2;
        t4.push_back(g);
      }
    run("syrk1k_x4", t4, 4 * fl);
    std::vector<GemmTask> t2(t4.begin(), t4.end());
    for (GemmTask& g : t2) g.k[0] = 256;
    run("syrk256_x4", t2, fl);
  }
  {  // wide tiles 64x128 over the same syrk/update shapes (K = 64 / 256 / 1024)
    auto wide = [&](const char* name, int K, int rmax, int reps) {
      std::vector<GemmTask> t;
      double fl = 0;
      for (int rep = 0; rep < reps; ++rep)
        for (int jb = 0; jb < rmax; jb += 128)
          for (int ib = jb; ib < rmax; ib += 64) {
            GemmTask g{};
            g.c = C + ib + static_cast<int64_t>(jb) * 2048 + rep * 2048 * 2048;
            g.ldc = 2048; g.m = 64; g.n = 128;
            g.a[0] = A + ib; g.lda[0] = 2048;
            g.b[0] = A + jb; g.ldb[0] = 2048;
            g.k[0] = K; g.flags = 2; g.alpha = -1.0; g.beta = 1.0;
            t.push_back(g);
            fl += 2.0 * 64 * 128 * K;
          }
      GemmTask* dt;
      cudaMalloc(&dt, t.size() * sizeof(GemmTask));
      cudaMemcpy(dt, t.data(), t.size() * sizeof(GemmTask), cudaMemcpyHostToDevice);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      auto timeit = [&](auto fn, int smem, const char* v) {
        float best = 1e9f;
        for (int r = 0; r < 8; ++r) {
          cudaEventRecord(e0);
          fn<<<static_cast<unsigned>(t.size()), 128, smem>>>(dt);
          cudaEventRecord(e1); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          if (r > 0 && ms < best) best = ms;
        }
        printf("%-10s %-12s %6zu tiles  %8.1f us  %6.2f TF/s  (%s)\n", name, v, t.size(), best * 1e3,
               fl / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
      };
      cudaFuncSetAttribute(k_gemm_big<128, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_big_smem<128, 3>());
      cudaFuncSetAttribute(k_gemm_big<128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_big_smem<128, 4>());
      cudaFuncSetAttribute(k_gemm_big<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_big_smem<128, 2>());
      timeit(k_gemm_big<128, 2>, gemm_big_smem<128, 2>(), "w128_s2");
      timeit(k_gemm_big<128, 3>, gemm_big_smem<128, 3>(), "w128_s3");
      timeit(k_gemm_big<128, 4>, gemm_big_smem<128, 4>(), "w128_s4");
      cudaFree(dt);
    };
    wide("wupd64", 64, 2048, 1);
    wide("wsyrk256x4", 256, 1024, 4);
    wide("wsyrk1kx4", 1024, 1024, 4);
  }
  return 0;
}
