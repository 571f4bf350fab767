// Benchmark of the tile GEMMs on launch shapes of the throughput-bound part of
// the factorization (operands larger than L2, odd leading dimensions, odd row
// offsets), 64x64 k_gemm_tiles against the 128x128 TMA-staged k_gemm_wide, with a
// bit-for-bit comparison of the two results.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -I paper_2503_08343_b200/csrc tools/gemm_big_bench.cu -o tools/gemm_big_bench
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kernels.cu"
#include "gemm_wide.cuh"
#include "../tools/gemm_wide_tn.cuh"

using namespace gmrf;

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__global__ void k_fill(double* p, int64_t n, unsigned seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long x = (i + 1) * 0x9E3779B97F4A7C15ull + seed;
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    p[i] = (double)(x & 0xFFFFFF) / 16777216.0 - 0.5;
  }
}
__global__ void k_diff(const double* a, const double* b, int64_t n, unsigned long long* cnt) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += a[i] != b[i];
  if (c) atomicAdd(cnt, c);
}

// lower-trapezoid SYRK-like update: C (rows x cols, ldc) -= A (rows x K) * B (cols x K)^T, tiles with
// row block >= column block when sym
static void tasks_for(int T, double* C, int64_t ldc, const double* A, int lda, const double* B, int ldb,
                      int rows, int cols, int K, bool sym, std::vector<GemmTask>& out, double& flops) {
  for (int jb = 0; jb < cols; jb += T)
    for (int ib = sym ? jb : 0; ib < rows; ib += T) {
      GemmTask g{};
      g.c = C + ib + (int64_t)jb * ldc;
      g.ldc = (int32_t)ldc;
      g.m = std::min(T, rows - ib);
      g.n = std::min(T, cols - jb);
      g.a[0] = A + ib; g.lda[0] = lda;
      g.b[0] = B + jb; g.ldb[0] = ldb;
      g.k[0] = K; g.flags = 2; g.alpha = -1.0; g.beta = 1.0;
      out.push_back(g);
      flops += 2.0 * g.m * g.n * K;
    }
}

static float time_launch(void (*fn)(const GemmTask*), const GemmTask* dt, size_t n, int threads, int smem, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    fn<<<(unsigned)n, threads, smem>>>(dt);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
    if (getenv("GEMM_TRACE_REPS") && (r % 8 == 0 || r == reps - 1)) printf("    rep %d: %.2f ms\n", r, ms);
  }
  CK(cudaGetLastError());
  return best;
}

struct Shape { const char* name; int fronts, rows, cols, K, lda, off; bool sym; };

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 4;
  CK(cudaFuncSetAttribute(k_gemm_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_wide_smem_bytes()));
  std::vector<Shape> shapes = {
      {"c5_137", 5, 8450, 8450, 1860, 10310, 1860, true},
      {"syrk8k_K4096", 1, 8192, 8192, 4096, 12417, 4225, true},
      {"syrk8k_K4225", 1, 8191, 8191, 4225, 12417, 4225, true},
      {"syrk2k_K512x16", 16, 2048, 2048, 512, 2561, 513, true},
      {"syrk1k_K256x64", 64, 1000, 1000, 250, 1251, 250, true},
      {"defer_K256", 1, 8000, 3968, 256, 12417, 300, true},
      {"upd_K64", 1, 8000, 3968, 64, 12417, 300, true},
  };
  for (const Shape& s : shapes) {
    const int64_t asz = (int64_t)s.lda * s.K + 4096, csz = (int64_t)s.rows * s.cols + 4096;
    double *A, *C0, *C1;
    CK(cudaMalloc(&A, asz * s.fronts * 8));
    CK(cudaMalloc(&C0, csz * s.fronts * 8));
    CK(cudaMalloc(&C1, csz * s.fronts * 8));
    k_fill<<<1024, 256>>>(A, asz * s.fronts, 1);
    k_fill<<<1024, 256>>>(C0, csz * s.fronts, 2);
    CK(cudaMemcpy(C1, C0, csz * s.fronts * 8, cudaMemcpyDeviceToDevice));
    std::vector<GemmTask> t64, t128, t128b;
    double f64 = 0, f128 = 0, fb = 0;
    for (int f = 0; f < s.fronts; ++f) {
      const double* Af = A + f * asz + s.off;  // L21: rows below the supernode's w columns
      tasks_for(64, C0 + f * csz, s.rows, Af, s.lda, Af, s.lda, s.rows, s.cols, s.K, s.sym, t64, f64);
      tasks_for(128, C1 + f * csz, s.rows, Af, s.lda, Af, s.lda, s.rows, s.cols, s.K, s.sym, t128, f128);
    }
    GemmTask *d64, *d128;
    CK(cudaMalloc(&d64, t64.size() * sizeof(GemmTask)));
    CK(cudaMalloc(&d128, t128.size() * sizeof(GemmTask)));
    CK(cudaMemcpy(d64, t64.data(), t64.size() * sizeof(GemmTask), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d128, t128.data(), t128.size() * sizeof(GemmTask), cudaMemcpyHostToDevice));
    // correctness: one application each from identical C
    k_gemm_tiles<<<(unsigned)t64.size(), 128>>>(d64);
    k_gemm_wide<<<(unsigned)t128.size(), kWThreads, gemm_wide_smem_bytes()>>>(d128);
    CK(cudaDeviceSynchronize());
    unsigned long long* cnt;
    CK(cudaMalloc(&cnt, 8)); CK(cudaMemset(cnt, 0, 8));
    k_diff<<<1024, 256>>>(C0, C1, csz * s.fronts, cnt);
    unsigned long long h = 0;
    CK(cudaMemcpy(&h, cnt, 8, cudaMemcpyDeviceToHost));
    const float m64 = time_launch(k_gemm_tiles, d64, t64.size(), 128, 0, reps);
    const float m128 = time_launch(k_gemm_wide, d128, t128.size(), kWThreads, gemm_wide_smem_bytes(), reps);
    // algorithmic flops (lower trapezoid only needs its lower part: both kernels compute whole tiles)
    printf("%-16s base64 %6zu tiles %9.1f us %6.2f TF/s | wide128 %6zu tiles %9.1f us %6.2f TF/s | mismatches %llu\n",
           s.name, t64.size(), m64 * 1e3, f64 / (m64 * 1e-3) / 1e12, t128.size(), m128 * 1e3,
           f64 / (m128 * 1e-3) / 1e12, h);
    fflush(stdout);
    cudaFree(A); cudaFree(C0); cudaFree(C1); cudaFree(d64); cudaFree(d128); cudaFree(cnt);
  }
  // K-contiguous operands (selected inversion: Y_R = Sigma_RR * L_RJ): C (r x w) = S (r x r, symmetric,
  // read transposed) * L (r x w block of a panel with ld rows), 64x64 k_gemm_tiles vs k_gemm_wide_tn
  CK(cudaFuncSetAttribute(k_gemm_wide_tn, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_wide_tn_smem_bytes()));
  struct TN { const char* name; int r, w, rows; };
  for (const TN& s : {TN{"tn_r8450_w3900", 8450, 3900, 12350}, TN{"tn_r4225_w4160", 4225, 4160, 8385},
                      TN{"tn_r1996_w1000", 1996, 1000, 2996}}) {
    const int64_t ssz = (int64_t)s.r * s.r + 4096, lsz = (int64_t)s.rows * s.w + 4096, csz = (int64_t)s.r * s.w + 4096;
    double *S, *L, *C0, *C1;
    CK(cudaMalloc(&S, ssz * 8)); CK(cudaMalloc(&L, lsz * 8)); CK(cudaMalloc(&C0, csz * 8)); CK(cudaMalloc(&C1, csz * 8));
    k_fill<<<1024, 256>>>(S, ssz, 3);
    k_fill<<<1024, 256>>>(L, lsz, 4);
    CK(cudaMemset(C0, 0, csz * 8)); CK(cudaMemset(C1, 0, csz * 8));
    auto mk = [&](int T, double* C, std::vector<GemmTask>& out, double& fl) {
      for (int jb = 0; jb < s.w; jb += T)
        for (int ib = 0; ib < s.r; ib += T) {
          GemmTask g{};
          g.c = C + ib + (int64_t)jb * s.r; g.ldc = s.r;
          g.m = std::min(T, s.r - ib); g.n = std::min(T, s.w - jb);
          g.a[0] = S + (int64_t)ib * s.r; g.lda[0] = s.r;
          g.b[0] = L + (s.rows - s.r) + (int64_t)jb * s.rows; g.ldb[0] = s.rows;
          g.k[0] = s.r; g.flags = 1; g.alpha = 1.0; g.beta = 0.0;
          out.push_back(g); fl += 2.0 * g.m * g.n * s.r;
        }
    };
    std::vector<GemmTask> t64, t128; double f64 = 0, f128 = 0;
    mk(64, C0, t64, f64); mk(128, C1, t128, f128);
    GemmTask *d64, *d128;
    CK(cudaMalloc(&d64, t64.size() * sizeof(GemmTask))); CK(cudaMalloc(&d128, t128.size() * sizeof(GemmTask)));
    CK(cudaMemcpy(d64, t64.data(), t64.size() * sizeof(GemmTask), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d128, t128.data(), t128.size() * sizeof(GemmTask), cudaMemcpyHostToDevice));
    const float m64 = time_launch(k_gemm_tiles, d64, t64.size(), 128, 0, reps);
    const float m128 = time_launch(k_gemm_wide_tn, d128, t128.size(), kWThreads, gemm_wide_tn_smem_bytes(), reps);
    unsigned long long* cnt; CK(cudaMalloc(&cnt, 8)); CK(cudaMemset(cnt, 0, 8));
    k_diff<<<1024, 256>>>(C0, C1, (int64_t)s.r * s.w, cnt);
    unsigned long long h = 0; CK(cudaMemcpy(&h, cnt, 8, cudaMemcpyDeviceToHost));
    printf("%-16s base64 %6zu tiles %9.1f us %6.2f TF/s | wide_tn %6zu tiles %9.1f us %6.2f TF/s | mismatches %llu\n",
           s.name, t64.size(), m64 * 1e3, f64 / (m64 * 1e-3) / 1e12, t128.size(), m128 * 1e3,
           f64 / (m128 * 1e-3) / 1e12, h);
    fflush(stdout);
    cudaFree(S); cudaFree(L); cudaFree(C0); cudaFree(C1); cudaFree(d64); cudaFree(d128); cudaFree(cnt);
  }
  return 0;
}
