// Wide-tile DMMA GEMM for the throughput-bound launches (U SYRKs and deferred
// trailing updates of large fronts, selected-inversion products): one 128×128
// output tile per CTA, operands staged by the TMA engine.
//
//   * producer warp: one lane issues cp.async.bulk (global → shared, 1-D bulk
//     copies, one per operand column of the K stage) into a kWStages-deep ring;
//     completion is signalled on an mbarrier per stage (complete_tx bytes), the
//     consumers hand a stage back through a second mbarrier — no per-thread
//     cp.async address arithmetic, no block-wide barrier in the K loop.
//   * 8 consumer warps (2 × 4), each a 64×32 sub-tile = 8×4 m8n8k4 DMMA
//     fragments: 12 fragment loads per 32 DMMAs (the 64×64 kernel: 8 per 16),
//     and half the L2 → SM operand traffic per flop of the 64×64 tile.
//   * bulk copies need 16-byte aligned sources: a column that starts 8 bytes
//     into a 16-byte chunk is copied from the chunk's start and read one element
//     later (the same per-column phase as load_operand in kernels.cu).
//
// Same GemmTask as k_gemm_tiles (one K segment, A not transposed, B transposed:
// C = beta·C + alpha·A·Bᵀ with A = a[0] (m×K, ld lda), B = b[0] (n×K, ld ldb));
// per output entry the K accumulation order is the 64×64 kernel's (4 at a time,
// ascending), so the two kernels agree bit for bit.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace gmrf {

constexpr int kWTile = 128;                 // output tile (rows = cols)
constexpr int kWKC = 16;                    // K per stage
constexpr int kWStages = 4;                 // ring depth
constexpr int kWPitch = kWTile + 4;         // smem column pitch (doubles): ≡ 4 mod 16 → the 4 k-rows of a
                                            // fragment load fall in disjoint bank groups
constexpr int kWConsumers = 8;              // consumer warps (+ 1 producer warp: 3 warps on one SM
                                            // sub-partition, so ptxas caps the kernel at 168 registers)
constexpr int kWThreads = 32 * (kWConsumers + 1);
constexpr int kWColBytes = (kWTile + 2) * 8;  // bytes per bulk copy (one element of alignment slack)

constexpr int gemm_wide_smem_bytes() {
  return kWStages * 2 * kWKC * kWPitch * 8 + 2 * kWStages * 8 + 16;
}

namespace wide_detail {
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global → shared (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes,
                                         unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
}  // namespace wide_detail

__global__ void __launch_bounds__(kWThreads, 1) k_gemm_wide(const GemmTask* __restrict__ tasks) {
  using namespace wide_detail;
  extern __shared__ __align__(16) unsigned char wsm[];
  double* As = reinterpret_cast<double*>(wsm);           // [stage][kWKC][kWPitch]
  double* Bs = As + kWStages * kWKC * kWPitch;           // [stage][kWKC][kWPitch]
  uint64_t* bars = reinterpret_cast<uint64_t*>(Bs + kWStages * kWKC * kWPitch);
  const unsigned full0 = smem_u32(bars), empty0 = smem_u32(bars + kWStages);
  const GemmTask& t = tasks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = t.k[0];
  const double* A = t.a[0];
  const double* B = t.b[0];
  const int lda = t.lda[0], ldb = t.ldb[0];
  const int nk = (K + kWKC - 1) / kWKC;
  if (tid == 0) {
    for (int s = 0; s < kWStages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kWConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kWConsumers) {
    // ---- producer: lane kk issues the stage's A and B copies of column kk
    if (lane < kWKC) {
      const int pa = static_cast<int>((reinterpret_cast<uintptr_t>(A) >> 3) & 1);
      const int pb = static_cast<int>((reinterpret_cast<uintptr_t>(B) >> 3) & 1);
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % kWStages;
        if (kc >= kWStages) mbar_wait(empty0 + 8 * s, ((kc / kWStages) - 1) & 1);
        const int k = kc * kWKC + lane;
        const int live = min(kWKC, K - kc * kWKC);
        if (lane == 0) mbar_expect_tx(full0 + 8 * s, 2u * kWColBytes * live);
        __syncwarp();
        if (k < K) {
          const double* ca = A + static_cast<int64_t>(k) * lda;
          const double* cb = B + static_cast<int64_t>(k) * ldb;
          // aligned-down start: phase of column k = p0 ^ (k & ld & 1)
          ca -= pa ^ (k & lda & 1);
          cb -= pb ^ (k & ldb & 1);
          bulk_g2s(smem_u32(As + (s * kWKC + lane) * kWPitch), ca, kWColBytes, full0 + 8 * s);
          bulk_g2s(smem_u32(Bs + (s * kWKC + lane) * kWPitch), cb, kWColBytes, full0 + 8 * s);
        }
      }
    }
    return;
  }

  // ---- consumers: warp (wm, wn) owns rows [64·wm, +64) × cols [32·wn, +32)
  const int wm = warp & 1, wn = warp >> 1;
  const int m = t.m, n = t.n;
  const double alpha = t.alpha, beta = t.beta;
  double* C = t.c;
  const int64_t ldc = t.ldc;
  double acc[8][4][2];
  // alpha = ±1 in every plan: folded into the accumulator's sign (exact), so the
  // K loop has no multiply:  C = alpha·(alpha·beta·C + A·Bᵀ)
  const double b0 = alpha * beta;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = wm * 64 + i * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * 32 + j * 8 + (lane & 3) * 2 + e;
        acc[i][j][e] = (beta != 0.0 && row < m && col < n) ? b0 * C[row + col * ldc] : 0.0;
      }
  }
  const int pa0 = static_cast<int>((reinterpret_cast<uintptr_t>(A) >> 3) & 1), la = lda & 1;
  const int pb0 = static_cast<int>((reinterpret_cast<uintptr_t>(B) >> 3) & 1), lb = ldb & 1;
  const int arow = wm * 64 + (lane >> 2), brow = wn * 32 + (lane >> 2);
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc % kWStages;
    mbar_wait(full0 + 8 * s, (kc / kWStages) & 1);
    const double* a = As + s * kWKC * kWPitch;
    const double* b = Bs + s * kWKC * kWPitch;
    const int krem = K - kc * kWKC;  // live columns of this stage
    if (krem >= kWKC) {
#pragma unroll
      for (int kk = 0; kk < kWKC; kk += 4) {
        const int kr = kk + (lane & 3);
        const int kg = kc * kWKC + kr;
        const double* ap = a + kr * kWPitch + arow + (pa0 ^ (kg & la));
        const double* bp = b + kr * kWPitch + brow + (pb0 ^ (kg & lb));
        double af[8], bf[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) af[i] = ap[i * 8];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = bp[j * 8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    } else {
      // last, partial stage: columns past K were not copied (stale shared memory): zero
      for (int kk = 0; kk < krem; kk += 4) {
        const int kr = kk + (lane & 3);
        const int kg = kc * kWKC + kr;
        const bool ok = kr < krem;
        const double* ap = a + kr * kWPitch + arow + (pa0 ^ (kg & la));
        const double* bp = b + kr * kWPitch + brow + (pb0 ^ (kg & lb));
        double af[8], bf[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) af[i] = ok ? ap[i * 8] : 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = ok ? bp[j * 8] : 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = wm * 64 + i * 8 + (lane >> 2);
    if (row >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * 32 + j * 8 + (lane & 3) * 2 + e;
        if (col < n) C[row + col * ldc] = alpha * acc[i][j][e];
      }
  }
}


}  // namespace gmrf
