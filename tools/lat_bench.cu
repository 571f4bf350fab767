// Latency microbenchmark for the pivot chain of the panel kernels (clock64 in
// one thread / one CTA): dependent DFMA, MUFU rsqrt/rcp f64, pivot_rn,
// div_rn, shared store->load round trip, bar.sync with 64 and 192 threads.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2503_08343_b200/csrc tools/lat_bench.cu -o tools/lat_bench
#include <cuda_runtime.h>

#include <cstdio>

#include "panel.cuh"

using namespace gmrf;

constexpr int N = 4096;

__global__ void k_lat(long long* out, double* sink, double seed) {
  __shared__ double sh[64];
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0, t1;
  // 0: dependent DFMA
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-300);
  t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  // 1: dependent DMUL
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x * y;
  t1 = clock64();
  if (threadIdx.x == 0) out[1] = t1 - t0;
  // 2: dependent rsqrt.approx.f64
  double z = 1.5 + x * 1e-300;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(z));
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = t1 - t0;
  // 3: dependent pivot_rn
  double p = 2.0 + z * 1e-300, rp = 0.5;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) {
    pivot_rn(p + 1.0, p, rp);
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = t1 - t0;
  // 4: dependent div_rn
  double a = 3.0 + rp * 1e-300;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = div_rn(a, 1.0000001, 0.9999999);
  t1 = clock64();
  if (threadIdx.x == 0) out[4] = t1 - t0;
  // 5: shared store -> load round trip (one thread)
  double v = a;
  __syncthreads();
  t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < N; ++i) {
      sh[i & 63] = v;
      v = sh[(i & 63)] + 1e-300;
    }
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = t1 - t0;
  // 6: bar.sync loop
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < N; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) out[6] = t1 - t0;
  // 7: shared publish + barrier + read by all (the per-column handoff)
  double q = v;
  t0 = clock64();
  for (int i = 0; i < N; ++i) {
    if (threadIdx.x == (i & 31)) sh[i & 1] = q + 1.0;
    __syncthreads();
    q = sh[i & 1];
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[7] = t1 - t0;
  // 8: shfl-based handoff within a warp (dependent)
  double s = q;
  t0 = clock64();
  for (int i = 0; i < N; ++i) s = __shfl_sync(0xffffffffu, s, i & 31) + 1e-300;
  t1 = clock64();
  if (threadIdx.x == 0) out[8] = t1 - t0;
  // 9: dependent FP32 FMA (reference)
  float f = static_cast<float>(s), g = 1.0000001f;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) f = fmaf(f, g, 1e-30f);
  t1 = clock64();
  if (threadIdx.x == 0) out[9] = t1 - t0;
  sink[threadIdx.x] = x + z + p + rp + a + v + q + s + f;
}

int main() {
  long long* d_out;
  double* sink;
  cudaMalloc(&d_out, 16 * sizeof(long long));
  cudaMalloc(&sink, 1024 * sizeof(double));
  const char* names[] = {"dfma", "dmul", "rsqrt.f64", "pivot_rn", "div_rn", "sts->lds",
                         "bar.sync", "publish+bar+lds", "shfl dep", "ffma"};
  for (int threads : {32, 64, 192}) {
    for (int rep = 0; rep < 2; ++rep) {
      k_lat<<<1, threads>>>(d_out, sink, 1.0);
      cudaDeviceSynchronize();
    }
    long long h[16];
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads=%d\n", threads);
    for (int i = 0; i < 10; ++i) printf("  %-18s %7.1f cycles/iter\n", names[i], double(h[i]) / N);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
