// K-contiguous variant of k_gemm_wide (paper_2503_08343_b200/csrc/gemm_wide.cuh), bench only
// (tools/gemm_big_bench.cu). Measured and not kept: with the contraction index contiguous in
// both operands a TMA stage is 256 short (272-byte) bulk copies per 128x128 tile, and bulk
// copies issue at about one per 60 cycles per SM whatever their size, so the ring starves the
// DMMA pipe: 19.5 TFLOP/s against 28.4 for the 64x64 cp.async kernel on the selected
// inversion's Y = Sigma_RR * L_RJ shapes (profiles/r02_gemm_big_bench.txt).
#pragma once

#include "gemm_wide.cuh"

namespace gmrf {

// ---------------------------------------------------------------------------
// K-contiguous operands (the selected inversion's Y = Σ_RR · L_RJ): both operands
// are stored with the contraction index contiguous,
//   A(i, l) = a[l + i·lda]   (GemmTask "A transposed"; Σ_RR is symmetric),
//   B(l, j) = b[l + j·ldb]   (GemmTask "B not transposed": L's rows below the supernode),
// so a K stage is one short bulk copy per tile row / column (kWtKC doubles of
// each of the 128 + 128 operand columns), 8 copies per producer lane. Fragments
// read k along the shared-memory row; the alignment phase is per operand column.
// ---------------------------------------------------------------------------
constexpr int kWtKC = 32;                   // K per stage
constexpr int kWtStages = 3;
constexpr int kWtPitch = kWtKC + 4;         // ≡ 4 mod 16 doubles: conflict-free fragment loads
constexpr int kWtRowBytes = (kWtKC + 2) * 8;  // bytes per bulk copy (alignment slack)

constexpr int gemm_wide_tn_smem_bytes() {
  return kWtStages * 2 * kWTile * kWtPitch * 8 + 2 * kWtStages * 8 + 16;
}

__global__ void __launch_bounds__(kWThreads, 1) k_gemm_wide_tn(const GemmTask* __restrict__ tasks) {
  using namespace wide_detail;
  extern __shared__ __align__(16) unsigned char wsm[];
  double* As = reinterpret_cast<double*>(wsm);            // [stage][kWTile][kWtPitch]
  double* Bs = As + kWtStages * kWTile * kWtPitch;        // [stage][kWTile][kWtPitch]
  uint64_t* bars = reinterpret_cast<uint64_t*>(Bs + kWtStages * kWTile * kWtPitch);
  const unsigned full0 = smem_u32(bars), empty0 = smem_u32(bars + kWtStages);
  const GemmTask& t = tasks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = t.k[0];
  const double* A = t.a[0];
  const double* B = t.b[0];
  const int lda = t.lda[0], ldb = t.ldb[0];
  const int nk = (K + kWtKC - 1) / kWtKC;
  const int pa0 = static_cast<int>((reinterpret_cast<uintptr_t>(A) >> 3) & 1), la = lda & 1;
  const int pb0 = static_cast<int>((reinterpret_cast<uintptr_t>(B) >> 3) & 1), lb = ldb & 1;
  if (tid == 0) {
    for (int s = 0; s < kWtStages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kWConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kWConsumers) {
    // ---- producer: lane q copies operand columns q, q+32, q+64, q+96 of A and of B
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % kWtStages;
      if (kc >= kWtStages) mbar_wait(empty0 + 8 * s, ((kc / kWtStages) - 1) & 1);
      if (lane == 0) mbar_expect_tx(full0 + 8 * s, 2u * kWTile * kWtRowBytes);
      __syncwarp();
      const int k0 = kc * kWtKC;  // even: the column's phase does not depend on the stage
#pragma unroll
      for (int q = 0; q < kWTile / 32; ++q) {
        const int c = lane + 32 * q;
        // operand columns past the tile's m / n repeat the last valid one (their
        // outputs are never stored; the source stays inside the operand)
        const int cm = min(c, t.m - 1), cn = min(c, t.n - 1);
        const double* ca = A + static_cast<int64_t>(cm) * lda + k0;
        const double* cb = B + static_cast<int64_t>(cn) * ldb + k0;
        ca -= pa0 ^ (cm & la);
        cb -= pb0 ^ (cn & lb);
        bulk_g2s(smem_u32(As + (s * kWTile + c) * kWtPitch), ca, kWtRowBytes, full0 + 8 * s);
        bulk_g2s(smem_u32(Bs + (s * kWTile + c) * kWtPitch), cb, kWtRowBytes, full0 + 8 * s);
      }
    }
    return;
  }

  const int wm = warp & 1, wn = warp >> 1;
  const int m = t.m, n = t.n;
  const double alpha = t.alpha, beta = t.beta;
  double* C = t.c;
  const int64_t ldc = t.ldc;
  double acc[8][4][2];
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
  const int arow = wm * 64 + (lane >> 2), brow = wn * 32 + (lane >> 2);
  // operand column c = arow + 8i: its phase only depends on the lane (8i is even)
  const int aoff = arow * kWtPitch + (lane & 3) + (pa0 ^ (arow & la));
  const int boff = brow * kWtPitch + (lane & 3) + (pb0 ^ (brow & lb));
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc % kWtStages;
    mbar_wait(full0 + 8 * s, (kc / kWtStages) & 1);
    const double* a = As + s * kWTile * kWtPitch + aoff;
    const double* b = Bs + s * kWTile * kWtPitch + boff;
    const int krem = K - kc * kWtKC;
    if (krem >= kWtKC) {
#pragma unroll
      for (int kk = 0; kk < kWtKC; kk += 4) {
        double af[8], bf[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) af[i] = a[i * 8 * kWtPitch + kk];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = b[j * 8 * kWtPitch + kk];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    } else {
      // last, partial stage: entries past K belong to other columns (or are stale): zero
      for (int kk = 0; kk < krem; kk += 4) {
        const bool ok = kk + (lane & 3) < krem;
        double af[8], bf[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) af[i] = ok ? a[i * 8 * kWtPitch + kk] : 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = ok ? b[j * 8 * kWtPitch + kk] : 0.0;
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
