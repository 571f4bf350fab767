// Experimental variants of k_gemm_tiles (kernels.cu) for tools/gemm_bench.cu:
// warp layout (WM x WN warps over the 64x64 tile), K stage depth KC, and the
// DMMA shape (m8n8k4 or m16n8k4).
#pragma once
#include "kernels.cu"

namespace gmrf {

__device__ __forceinline__ void dmma1684(double (&c)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

__device__ __forceinline__ void dmma884nv(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

template <int NT, int KC>
__device__ __forceinline__ void load_op_v(double (*dst)[kPad], const double* src, int ld,
                                          bool kcontig, int mn_lim, int k0, int k_lim, int tid) {
  if (!kcontig) {
#pragma unroll
    for (int it = 0; it < (KC * kTile) / NT; ++it) {
      int idx = tid + it * NT;
      int kk = idx >> 6, mm = idx & 63;
      bool ok = mm < mn_lim && (k0 + kk) < k_lim;
      const double* p = ok ? src + mm + static_cast<int64_t>(k0 + kk) * ld : src;
      cp_async8(&dst[kk][mm], p, ok);
    }
  } else {
#pragma unroll
    for (int it = 0; it < (KC * kTile) / NT; ++it) {
      int idx = tid + it * NT;
      int mm = idx / KC, kk = idx % KC;
      bool ok = mm < mn_lim && (k0 + kk) < k_lim;
      const double* p = ok ? src + (k0 + kk) + static_cast<int64_t>(mm) * ld : src;
      cp_async8(&dst[kk][mm], p, ok);
    }
  }
}

// 16-byte cp.async for mm-contiguous operands (requires 16-B aligned columns:
// even ld and even row offset); falls back to 8-byte copies otherwise
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
template <int NT, int KC>
__device__ __forceinline__ void load_op16(double (*dst)[kPad], const double* src, int ld,
                                          bool kcontig, int mn_lim, int k0, int k_lim, int tid) {
  const bool al = !kcontig && ((reinterpret_cast<uintptr_t>(src) | (static_cast<uintptr_t>(ld) * 8)) & 15) == 0 &&
                  mn_lim == 64 && k0 + KC <= k_lim;
  if (!al) {
    load_op_v<NT, KC>(dst, src, ld, kcontig, mn_lim, k0, k_lim, tid);
    return;
  }
#pragma unroll
  for (int it = 0; it < (KC * kTile) / (2 * NT); ++it) {
    int idx = tid + it * NT;
    int kk = idx >> 5, mm = (idx & 31) * 2;
    cp_async16(&dst[kk][mm], src + mm + static_cast<int64_t>(k0 + kk) * ld);
  }
}

template <int WM, int WN, int KC, bool M16, int MINB, bool NV = false, int MODE = 0>
__global__ void __launch_bounds__(32 * WM * WN, MINB) k_gemm_var(const GemmTask* __restrict__ tasks) {
  constexpr int NT = 32 * WM * WN;
  constexpr int TM = 64 / WM, TN = 64 / WN;          // warp tile
  constexpr int FM = M16 ? TM / 16 : TM / 8, FN = TN / 8;
  constexpr int CE = M16 ? 4 : 2;                    // accumulator regs per fragment
  __shared__ __align__(16) double As[2][KC][kPad];
  __shared__ __align__(16) double Bs[2][KC][kPad];
  const GemmTask& t = tasks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WM, wn = warp / WM;
  const int m = t.m, n = t.n;
  const double alpha = t.alpha, beta = t.beta;
  double* C = t.c;
  const int64_t ldc = t.ldc;
  double acc[FM][FN][CE];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int e = 0; e < CE; ++e) {
        const int row = wm * TM + (M16 ? i * 16 : i * 8) + (lane >> 2) + (e >= 2 ? 8 : 0);
        const int col = wn * TN + j * 8 + (lane & 3) * 2 + (e & 1);
        const double bs = (MODE == 3 && alpha < 0.0) ? -beta : beta;
        acc[i][j][e] = (MODE != 2 && beta != 0.0 && row < m && col < n) ? bs * C[row + col * ldc] : 0.0;
      }
  for (int seg = 0; seg < 2; ++seg) {
    const int K = t.k[seg];
    if (K <= 0) continue;
    const double* A = t.a[seg];
    const double* B = t.b[seg];
    const int lda = t.lda[seg], ldb = t.ldb[seg];
    const bool a_kc = (t.flags >> (2 * seg)) & 1;
    const bool b_kc = !((t.flags >> (2 * seg + 1)) & 1);
    const int nk = (K + KC - 1) / KC;
    if constexpr (MODE == 4) {
      load_op16<NT, KC>(As[0], A, lda, a_kc, m, 0, K, tid);
      load_op16<NT, KC>(Bs[0], B, ldb, b_kc, n, 0, K, tid);
    } else {
      load_op_v<NT, KC>(As[0], A, lda, a_kc, m, 0, K, tid);
      load_op_v<NT, KC>(Bs[0], B, ldb, b_kc, n, 0, K, tid);
    }
    cp_async_commit();
    for (int kc = 0; kc < nk; ++kc) {
      const int buf = kc & 1;
      if (kc + 1 < nk) {
        if constexpr (MODE == 4) {
          load_op16<NT, KC>(As[buf ^ 1], A, lda, a_kc, m, (kc + 1) * KC, K, tid);
          load_op16<NT, KC>(Bs[buf ^ 1], B, ldb, b_kc, n, (kc + 1) * KC, K, tid);
        } else {
        load_op_v<NT, KC>(As[buf ^ 1], A, lda, a_kc, m, (kc + 1) * KC, K, tid);
        load_op_v<NT, KC>(Bs[buf ^ 1], B, ldb, b_kc, n, (kc + 1) * KC, K, tid);
        }
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < (MODE == 1 ? 0 : KC); kk += 4) {
        double bf[FN];
#pragma unroll
        for (int j = 0; j < FN; ++j) bf[j] = Bs[buf][kk + (lane & 3)][wn * TN + j * 8 + (lane >> 2)];
        if constexpr (M16) {
          double a0[FM], a1[FM];
#pragma unroll
          for (int i = 0; i < FM; ++i) {
            a0[i] = alpha * As[buf][kk + (lane & 3)][wm * TM + i * 16 + (lane >> 2)];
            a1[i] = alpha * As[buf][kk + (lane & 3)][wm * TM + i * 16 + 8 + (lane >> 2)];
          }
#pragma unroll
          for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j) dmma1684(acc[i][j], a0[i], a1[i], bf[j]);
        } else {
          double af[FM];
#pragma unroll
          for (int i = 0; i < FM; ++i)
            af[i] = (MODE == 3 ? 1.0 : alpha) * As[buf][kk + (lane & 3)][wm * TM + i * 8 + (lane >> 2)];
#pragma unroll
          for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j) {
              if constexpr (NV) dmma884nv(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
              else dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
        }
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int e = 0; e < CE; ++e) {
        const int row = wm * TM + (M16 ? i * 16 : i * 8) + (lane >> 2) + (e >= 2 ? 8 : 0);
        const int col = wn * TN + j * 8 + (lane & 3) * 2 + (e & 1);
        if (row < m && col < n && (MODE != 2 || acc[i][j][e] == 12345.0))
          C[row + col * ldc] = (MODE == 3 && alpha < 0.0) ? -acc[i][j][e] : acc[i][j][e];
      }
}

}  // namespace gmrf

namespace gmrf {
// Multistage variant: NS K-stages of 16 in flight (dynamic shared memory), so a
// K ≤ 16·(NS−1) tile issues all its operand loads at once (one memory round
// trip instead of one per stage).
template <int NS, int MINB>
__global__ void __launch_bounds__(128, MINB) k_gemm_ms(const GemmTask* __restrict__ tasks) {
  extern __shared__ __align__(16) double smem_ms[];
  typedef double Stage[kKC][kPad];
  Stage* As = reinterpret_cast<Stage*>(smem_ms);
  Stage* Bs = As + NS;
  const GemmTask& t = tasks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int m = t.m, n = t.n;
  const double alpha = t.alpha, beta = t.beta;
  double* C = t.c;
  const int64_t ldc = t.ldc;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = wm * 32 + i * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * 32 + j * 8 + (lane & 3) * 2 + e;
        acc[i][j][e] = (beta != 0.0 && row < m && col < n) ? beta * C[row + col * ldc] : 0.0;
      }
  }
  for (int seg = 0; seg < 2; ++seg) {
    const int K = t.k[seg];
    if (K <= 0) continue;
    const double* A = t.a[seg];
    const double* B = t.b[seg];
    const int lda = t.lda[seg], ldb = t.ldb[seg];
    const bool a_kc = (t.flags >> (2 * seg)) & 1;
    const bool b_kc = !((t.flags >> (2 * seg + 1)) & 1);
    const int nk = (K + kKC - 1) / kKC;
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) {
      if (s < nk) {
        load_operand(As[s], A, lda, a_kc, m, s * kKC, K, tid);
        load_operand(Bs[s], B, ldb, b_kc, n, s * kKC, K, tid);
      }
      cp_async_commit();
    }
    for (int kc = 0; kc < nk; ++kc) {
      const int nx = kc + NS - 1;
      if (nx < nk) {
        load_operand(As[nx % NS], A, lda, a_kc, m, nx * kKC, K, tid);
        load_operand(Bs[nx % NS], B, ldb, b_kc, n, nx * kKC, K, tid);
      }
      cp_async_commit();
      cp_async_wait<NS - 1>();
      __syncthreads();
      const int buf = kc % NS;
#pragma unroll
      for (int kk = 0; kk < kKC; kk += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          af[i] = alpha * As[buf][kk + (lane & 3)][wm * 32 + i * 8 + (lane >> 2)];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][kk + (lane & 3)][wn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = wm * 32 + i * 8 + (lane >> 2);
    if (row >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * 32 + j * 8 + (lane & 3) * 2 + e;
        if (col < n) C[row + col * ldc] = acc[i][j][e];
      }
  }
}
template <int NS>
constexpr int gemm_ms_smem() {
  return 2 * NS * kKC * kPad * static_cast<int>(sizeof(double));
}
}  // namespace gmrf

namespace gmrf {
// Wide-tile variant: CTA tile 64 x TN (TN = 128), 4 warps 2x2 of 32 x TN/2, so a
// warp issues 4 A + TN/16 B fragment loads per 4*TN/16... DMMAs (better DMMA:LDS
// ratio than 32x32 warp tiles); NS-stage cp.async pipeline in dynamic shared
// memory, 16-byte copies (operands 16-B aligned, mm contiguous: bench only).
template <int TN, int NS>
constexpr int gemm_big_smem() {
  return NS * 16 * ((64 + 8) + (TN + 8)) * static_cast<int>(sizeof(double));
}
template <int TN, int NS>
__global__ void __launch_bounds__(128, 2) k_gemm_big(const GemmTask* __restrict__ tasks) {
  constexpr int KC = 16, PA = 64 + 8, PB = TN + 8, FM = 4, FN = TN / 16;
  extern __shared__ __align__(16) double smb[];
  double* As = smb;                 // [NS][KC][PA]
  double* Bs = smb + NS * KC * PA;  // [NS][KC][PB]
  const GemmTask& t = tasks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int m = t.m, n = t.n;
  const double alpha = t.alpha, beta = t.beta;
  double* C = t.c;
  const int64_t ldc = t.ldc;
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = wm * 32 + i * 8 + (lane >> 2);
        const int col = wn * (TN / 2) + j * 8 + (lane & 3) * 2 + e;
        acc[i][j][e] = (beta != 0.0 && row < m && col < n) ? beta * C[row + col * ldc] : 0.0;
      }
  const int K = t.k[0];
  const double* A = t.a[0];
  const double* B = t.b[0];
  const int lda = t.lda[0], ldb = t.ldb[0];
  const int nk = (K + KC - 1) / KC;
  auto load = [&](int st, int k0) {
    double* a = As + st * KC * PA;
    double* b = Bs + st * KC * PB;
#pragma unroll
    for (int it = 0; it < (KC * 64) / (2 * 128); ++it) {
      const int idx = tid + it * 128, kk = idx >> 5, mm = (idx & 31) * 2;
      cp_async16(a + kk * PA + mm, A + mm + static_cast<int64_t>(k0 + kk) * lda);
    }
#pragma unroll
    for (int it = 0; it < (KC * TN) / (2 * 128); ++it) {
      const int idx = tid + it * 128, kk = idx / (TN / 2), mm = (idx % (TN / 2)) * 2;
      cp_async16(b + kk * PB + mm, B + mm + static_cast<int64_t>(k0 + kk) * ldb);
    }
  };
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nk) load(s, s * KC);
    cp_async_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<NS - 2>();
    __syncthreads();
    if (kc + NS - 1 < nk) load((kc + NS - 1) % NS, (kc + NS - 1) * KC);
    cp_async_commit();
    const double* a = As + (kc % NS) * KC * PA;
    const double* b = Bs + (kc % NS) * KC * PB;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      const int kr = kk + (lane & 3);
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = alpha * a[kr * PA + wm * 32 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = b[kr * PB + wn * (TN / 2) + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
#pragma unroll
  for (int i = 0; i < FM; ++i) {
    const int row = wm * 32 + i * 8 + (lane >> 2);
    if (row >= m) continue;
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * (TN / 2) + j * 8 + (lane & 3) * 2 + e;
        if (col < n) C[row + col * ldc] = acc[i][j][e];
      }
  }
}
}  // namespace gmrf
