// sm_100a kernels for the supernodal multifrontal Cholesky, the supernodal
// triangular solves and the supernodal selected inversion (FP64).
//
// FP64 tensor math on Blackwell is DMMA (mma.sync ... .f64); tcgen05 has no
// f64 kind. The GEMM tile kernel stages operands through shared
// memory with cp.async double buffering and issues m8n8k4 DMMA.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace gmrf {

// ---------------------------------------------------------------------------
// DMMA primitive: D(8x8) += A(8x4, row) * B(4x8, col), one f64 per lane for A
// and B, two for C/D. Fragment layout (PTX ISA, mma.m8n8k4 .f64):
//   A: row = lane>>2, col = lane&3;  B: row = lane&3, col = lane>>2;
//   C: row = lane>>2, col = 2*(lane&3) + i.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------------------
// Batched tile GEMM: one 64x64 output tile per CTA, 4 warps (2x2), each warp a
// 32x32 sub-tile = 4x4 DMMA m8n8 fragments. K staged in chunks of 16.
// ---------------------------------------------------------------------------
constexpr int kKC = 16;
constexpr int kPad = 68;  // smem row pitch (doubles), ≡ 4 mod 16: the four k-rows of a fragment load
                          // (LDS.64, 16 lanes per wavefront) fall in disjoint bank groups (72 gave 2-way
                          // conflicts on every load: ncu l1tex__data_bank_conflicts, r02_ncu_summary.txt)

// 16-byte copy, zero-filled when !pred
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

// Parity (in doubles) of an operand column's start address: a column-major
// panel with an odd leading dimension alternates between 16-byte-aligned and
// 8-byte-offset columns.
__device__ __forceinline__ int col_phase(const double* p) {
  return static_cast<int>((reinterpret_cast<uintptr_t>(p) >> 3) & 1);
}

__device__ __forceinline__ void load_operand(double (*dst)[kPad], const double* src, int ld,
                                             bool kcontig, int mn_lim, int k0, int k_lim,
                                             int tid) {
  if (!kcontig) {
    // element (mm, kk) at src[mm + kk*ld]: mm contiguous. Column kk is copied in
    // 16-byte chunks from its 16-byte-aligned start (one element early when the
    // column starts 8 bytes into a chunk): dst[kk][mm + ph(kk)] = element (mm, kk),
    // ph(kk) = the column's phase. Elements past mn_lim are copied too (they only
    // reach output rows/columns that are never stored); columns past k_lim are zero.
    // Allocations carry slack (DevBuf) for the last tile of a buffer.
    constexpr int CH = kTile / 2 + 1;  // chunks per column
#pragma unroll
    for (int it = 0; it < (kKC * CH + 127) / 128; ++it) {
      const int idx = tid + it * 128;
      if (idx < kKC * CH) {
        const int kk = idx / CH, ch = idx - kk * CH;
        const bool ok = (k0 + kk) < k_lim;
        const double* col = src + static_cast<int64_t>(k0 + kk) * ld;
        const double* p = ok ? col - col_phase(col) + 2 * ch : src - col_phase(src);
        cp_async16(&dst[kk][2 * ch], p, ok);
      }
    }
    (void)mn_lim;
  } else {
    // element (mm, kk) at src[kk + mm*ld]: kk contiguous
#pragma unroll
    for (int it = 0; it < (kKC * kTile) / 128; ++it) {
      int idx = tid + it * 128;
      int mm = idx >> 4, kk = idx & 15;
      bool ok = mm < mn_lim && (k0 + kk) < k_lim;
      const double* p = ok ? src + (k0 + kk) + static_cast<int64_t>(mm) * ld : src;
      cp_async8(&dst[kk][mm], p, ok);
    }
  }
}

// The accumulator starts from beta*C (issued with the first operand loads, so
// the C round trip overlaps them instead of trailing the MMA loop) and alpha is
// folded into the A fragments (alpha = ±1 in every plan: exact).
__global__ void __launch_bounds__(128, 5) k_gemm_tiles(const GemmTask* __restrict__ tasks) {
  __shared__ __align__(16) double As[2][kKC][kPad];
  __shared__ __align__(16) double Bs[2][kKC][kPad];
  const GemmTask& t = tasks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int m = t.m, n = t.n;
  const double alpha = t.alpha, beta = t.beta;
  double* C = t.c;
  const int64_t ldc = t.ldc;
  double acc[4][4][2];
  if (beta == 0.0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = wm * 32 + i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = wn * 32 + j * 8 + (lane & 3) * 2 + e;
          acc[i][j][e] = (row < m && col < n) ? beta * C[row + col * ldc] : 0.0;
        }
    }
  }

  for (int seg = 0; seg < 2; ++seg) {
    const int K = t.k[seg];
    if (K <= 0) continue;
    const double* A = t.a[seg];
    const double* B = t.b[seg];
    const int lda = t.lda[seg], ldb = t.ldb[seg];
    // A: N → mm contiguous; T → kk contiguous. B: N → kk contiguous; T → nn contiguous.
    const bool a_kc = (t.flags >> (2 * seg)) & 1;
    const bool b_kc = !((t.flags >> (2 * seg + 1)) & 1);
    const int nk = (K + kKC - 1) / kKC;
    // smem column shift of an mm-contiguous operand (load_operand): the phase of
    // column kk is ph0 ^ (kk & ld) — stage offsets k0 are even
    const int pa0 = a_kc ? 0 : col_phase(A), la = a_kc ? 0 : (lda & 1);
    const int pb0 = b_kc ? 0 : col_phase(B), lb = b_kc ? 0 : (ldb & 1);
    load_operand(As[0], A, lda, a_kc, m, 0, K, tid);
    load_operand(Bs[0], B, ldb, b_kc, n, 0, K, tid);
    cp_async_commit();
    for (int kc = 0; kc < nk; ++kc) {
      const int buf = kc & 1;
      if (kc + 1 < nk) {
        load_operand(As[buf ^ 1], A, lda, a_kc, m, (kc + 1) * kKC, K, tid);
        load_operand(Bs[buf ^ 1], B, ldb, b_kc, n, (kc + 1) * kKC, K, tid);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kKC; kk += 4) {
        double af[4], bf[4];
        const int kr = kk + (lane & 3);
        const int sa = pa0 ^ (kr & la), sb = pb0 ^ (kr & lb);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          af[i] = alpha * As[buf][kr][wm * 32 + i * 8 + (lane >> 2) + sa];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][kr][wn * 32 + j * 8 + (lane >> 2) + sb];
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

// ---------------------------------------------------------------------------
// Chain GEMM of the one-wave levels at the top of the tree: the update of a
// chunk's NEXT column block (K ≤ 64, a few dozen 64×64 tiles) sits on the
// factorization's critical path between two panel steps, where a 64×64 tile per
// CTA is four dependent K-stage round trips plus 256 DMMAs per warp (~8 µs for
// 0.5 MFLOP). Here a CTA owns a 32×32 tile (four times the CTAs, still under
// one wave), issues ALL its operand copies at once (K ≤ 64: one memory round
// trip) and each warp runs 2×2 fragments. Same K order per output entry as
// k_gemm_tiles (4 at a time, ascending): bit-identical. One segment, A not
// transposed, B transposed (the trailing-update form).
// ---------------------------------------------------------------------------
constexpr int kNTile = 32;            // output tile
constexpr int kNKMax = 64;            // K handled in one shot
constexpr int kNPad = kNTile + 4;     // ≡ 4 mod 16 doubles: conflict-free fragment loads
__global__ void __launch_bounds__(128) k_gemm_next(const GemmTask* __restrict__ tasks) {
  __shared__ __align__(16) double As[kNKMax][kNPad];
  __shared__ __align__(16) double Bs[kNKMax][kNPad];
  const GemmTask& t = tasks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int m = t.m, n = t.n, K = t.k[0];
  const double* A = t.a[0];
  const double* B = t.b[0];
  const int lda = t.lda[0], ldb = t.ldb[0];
  {
    // column kk of each operand in 16-byte chunks from its aligned start (phase
    // shift as in load_operand); columns past K are zero filled
    constexpr int CH = kNTile / 2 + 1;
    for (int idx = tid; idx < kNKMax * CH; idx += 128) {
      const int kk = idx / CH, ch = idx - kk * CH;
      const bool ok = kk < K;
      const double* ca = A + static_cast<int64_t>(kk) * lda;
      const double* cb = B + static_cast<int64_t>(kk) * ldb;
      cp_async16(&As[kk][2 * ch], ok ? ca - col_phase(ca) + 2 * ch : A - col_phase(A), ok);
      cp_async16(&Bs[kk][2 * ch], ok ? cb - col_phase(cb) + 2 * ch : B - col_phase(B), ok);
    }
    cp_async_commit();
  }
  const double alpha = t.alpha, beta = t.beta;
  double* C = t.c;
  const int64_t ldc = t.ldc;
  double acc[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = wm * 16 + i * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * 16 + j * 8 + (lane & 3) * 2 + e;
        acc[i][j][e] = (beta != 0.0 && row < m && col < n) ? beta * C[row + col * ldc] : 0.0;
      }
  }
  const int pa0 = col_phase(A), la = lda & 1;
  const int pb0 = col_phase(B), lb = ldb & 1;
  cp_async_wait<0>();
  __syncthreads();
  // as many 4-wide K steps as k_gemm_tiles runs (whole 16-column stages; the
  // columns past K are zero), so even signed zeros come out the same
  const int nks = ((K + kKC - 1) / kKC) * (kKC / 4);
  for (int ks = 0; ks < nks; ++ks) {
    const int kr = 4 * ks + (lane & 3);
    const int sa = pa0 ^ (kr & la), sb = pb0 ^ (kr & lb);
    double af[2], bf[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) af[i] = alpha * As[kr][wm * 16 + i * 8 + (lane >> 2) + sa];
#pragma unroll
    for (int j = 0; j < 2; ++j) bf[j] = Bs[kr][wn * 16 + j * 8 + (lane >> 2) + sb];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = wm * 16 + i * 8 + (lane >> 2);
    if (row >= m) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * 16 + j * 8 + (lane & 3) * 2 + e;
        if (col < n) C[row + col * ldc] = acc[i][j][e];
      }
  }
}

// ---------------------------------------------------------------------------
// (panel step: panel.cuh)
// ---------------------------------------------------------------------------
// Extend-add (multifrontal assembly), gather form: one warp per (front, front
// column) that some child updates, and per column of the front's update block
// (zeroed here first, so no per-factorization memset of the update matrices);
// the plan lists the contributing children
// and the row where each child's update column starts (no searching on the
// device). Children are visited in ascending order, so every target entry
// receives its contributions in a fixed order (deterministic, no atomics).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int find_sorted(const int32_t* a, int len, int key) {
  int lo = 0, hi = len;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return (lo < len && a[lo] == key) ? lo : -1;
}

__global__ void k_extend_add(const EaTask* __restrict__ tasks, int ntasks,
                             const int2* __restrict__ pairs, SymDev sd, double* __restrict__ L,
                             double* __restrict__ U) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= ntasks) return;
  const EaTask t = tasks[warp];
  const int s = t.sn, b = t.col;
  const int w = sd.sn_first[s + 1] - sd.sn_first[s];
  const int rows = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]);
  const int r = rows - w;
  double* Ls = L + sd.lptr[s];
  double* Us = U + sd.uptr[s];
  double* dst = b < w ? Ls + static_cast<int64_t>(b) * rows : Us + static_cast<int64_t>(b - w) * r - w;
  if (b >= w) {  // update-block column: starts from zero (lower part, rows b..rows-1)
    for (int a = b + lane; a < rows; a += 32) dst[a] = 0.0;
    __syncwarp();
  }
  for (int p = t.p0; p < t.p0 + t.np; ++p) {
    const int2 cp = pairs[p];
    const int c = cp.x, ib = cp.y;
    const int wc = sd.sn_first[c + 1] - sd.sn_first[c];
    const int rc = static_cast<int>(sd.sn_rptr[c + 1] - sd.sn_rptr[c]) - wc;
    const int32_t* rel = sd.relmap + sd.sn_rptr[c] + wc;
    const double* Uc = U + sd.uptr[c] + static_cast<int64_t>(ib) * rc;
    // 4 independent gathers in flight per lane (memory-level parallelism)
    int ia = ib + lane;
    for (; ia + 96 < rc; ia += 128) {
      int t0 = rel[ia], t1 = rel[ia + 32], t2 = rel[ia + 64], t3 = rel[ia + 96];
      double u0 = Uc[ia], u1 = Uc[ia + 32], u2 = Uc[ia + 64], u3 = Uc[ia + 96];
      double d0 = dst[t0], d1 = dst[t1], d2 = dst[t2], d3 = dst[t3];
      dst[t0] = d0 + u0;
      dst[t1] = d1 + u1;
      dst[t2] = d2 + u2;
      dst[t3] = d3 + u3;
    }
    for (; ia < rc; ia += 32) dst[rel[ia]] += Uc[ia];
    __syncwarp();
  }
}

// Same assembly with one CTA per (front, front column): the levels at the top of
// the tree have few but long columns (a few thousand rows, two large children),
// where one warp per column is a chain of dependent gather rounds. The threads
// of the CTA split each child's rows; children stay in ascending order (a
// barrier between them), so every entry sums in the same order as k_extend_add.
constexpr int kEaCtaThreads = 256;
__global__ void __launch_bounds__(kEaCtaThreads) k_extend_add_cta(
    const EaTask* __restrict__ tasks, const int2* __restrict__ pairs, SymDev sd,
    double* __restrict__ L, double* __restrict__ U) {
  const int tid = threadIdx.x;
  const EaTask t = tasks[blockIdx.x];
  const int s = t.sn, b = t.col;
  const int w = sd.sn_first[s + 1] - sd.sn_first[s];
  const int rows = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]);
  const int r = rows - w;
  double* Ls = L + sd.lptr[s];
  double* Us = U + sd.uptr[s];
  double* dst = b < w ? Ls + static_cast<int64_t>(b) * rows : Us + static_cast<int64_t>(b - w) * r - w;
  if (b >= w) {
    for (int a = b + tid; a < rows; a += kEaCtaThreads) dst[a] = 0.0;
    __syncthreads();
  }
  for (int p = t.p0; p < t.p0 + t.np; ++p) {
    const int2 cp = pairs[p];
    const int c = cp.x, ib = cp.y;
    const int wc = sd.sn_first[c + 1] - sd.sn_first[c];
    const int rc = static_cast<int>(sd.sn_rptr[c + 1] - sd.sn_rptr[c]) - wc;
    const int32_t* rel = sd.relmap + sd.sn_rptr[c] + wc;
    const double* Uc = U + sd.uptr[c] + static_cast<int64_t>(ib) * rc;
    int ia = ib + tid;
    for (; ia + 3 * kEaCtaThreads < rc; ia += 4 * kEaCtaThreads) {
      int t0 = rel[ia], t1 = rel[ia + kEaCtaThreads], t2 = rel[ia + 2 * kEaCtaThreads],
          t3 = rel[ia + 3 * kEaCtaThreads];
      double u0 = Uc[ia], u1 = Uc[ia + kEaCtaThreads], u2 = Uc[ia + 2 * kEaCtaThreads],
             u3 = Uc[ia + 3 * kEaCtaThreads];
      double d0 = dst[t0], d1 = dst[t1], d2 = dst[t2], d3 = dst[t3];
      dst[t0] = d0 + u0;
      dst[t1] = d1 + u1;
      dst[t2] = d2 + u2;
      dst[t3] = d3 + u3;
    }
    for (; ia < rc; ia += kEaCtaThreads) dst[rel[ia]] += Uc[ia];
    __syncthreads();
  }
}

// Q values → L panels through the precomputed offset map.
__global__ void k_scatter_q(const double* __restrict__ q, const int64_t* __restrict__ qmap,
                            int64_t nnz, double* __restrict__ L) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t o = qmap[p];
    if (o >= 0) L[o] = q[p];
  }
}

constexpr int kMaxRhs = 16;

// out[i + r*n] = in[perm[i] + r*n]  (gather: P b)
__global__ void k_permute_gather(const double* __restrict__ in, const int32_t* __restrict__ perm,
                                 int n, int nrhs, double* __restrict__ out) {
  int64_t tot = static_cast<int64_t>(n) * nrhs;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < tot;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r = idx / n, i = idx % n;
    out[idx] = in[perm[i] + r * n];
  }
}
// out[perm[i] + r*n] = in[i + r*n]  (scatter: Pᵀ y)
__global__ void k_permute_scatter(const double* __restrict__ in, const int32_t* __restrict__ perm,
                                  int n, int nrhs, double* __restrict__ out) {
  int64_t tot = static_cast<int64_t>(n) * nrhs;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < tot;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r = idx / n, i = idx % n;
    out[perm[i] + r * n] = in[idx];
  }
}

// ---------------------------------------------------------------------------
// Selected inversion (supernodal Takahashi, top-down).
// ---------------------------------------------------------------------------
// Σ_RR(s) (full r×r, stored in the U buffer) gathered from the parent's Σ front.
__global__ void k_sel_gather(const ColTask* __restrict__ tasks, int ntasks, SymDev sd,
                             const int32_t* __restrict__ sn_parent, const double* __restrict__ Sig,
                             double* __restrict__ U) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= ntasks) return;
  const int s = tasks[warp].sn, b = tasks[warp].col;  // b: column of Σ_RR(s), 0..r-1
  const int w = sd.sn_first[s + 1] - sd.sn_first[s];
  const int r = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]) - w;
  const int p = sn_parent[s];
  const int wp = sd.sn_first[p + 1] - sd.sn_first[p];
  const int rowsp = static_cast<int>(sd.sn_rptr[p + 1] - sd.sn_rptr[p]);
  const int rp = rowsp - wp;
  const int32_t* rel = sd.relmap + sd.sn_rptr[s] + w;
  const double* Sp = Sig + sd.lptr[p];
  const double* Up = U + sd.uptr[p];
  double* dst = U + sd.uptr[s] + static_cast<int64_t>(b) * r;
  const int y = rel[b];
  for (int a = lane; a < r; a += 32) {
    const int x = rel[a];
    double v;
    if (y < wp)
      v = Sp[x + static_cast<int64_t>(y) * rowsp];       // panel column y (full in diag block)
    else if (x < wp)
      v = Sp[y + static_cast<int64_t>(x) * rowsp];       // mirror of panel column x
    else
      v = Up[(x - wp) + static_cast<int64_t>(y - wp) * rp];
    dst[a] = v;
  }
}

// (selected-inversion chunk kernels: selinv.cuh)

// var[perm[j]] = Σ_jj (a partitioned factor writes 0 for columns it does not
// own; the all-reduce over ranks then completes the vector exactly)
__global__ void k_extract_diag(SymDev sd, const int32_t* __restrict__ col2sn,
                               const int32_t* __restrict__ perm, const double* __restrict__ Sig,
                               const char* __restrict__ colmine, double* __restrict__ out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < sd.n; j += gridDim.x * blockDim.x) {
    if (colmine && !colmine[j]) {
      out[perm[j]] = 0.0;
      continue;
    }
    const int s = col2sn[j];
    const int f0 = sd.sn_first[s];
    const int64_t rows = sd.sn_rptr[s + 1] - sd.sn_rptr[s];
    const int a = j - f0;
    out[perm[j]] = Sig[sd.lptr[s] + a + a * rows];
  }
}

// ---------------------------------------------------------------------------
// Partitioned factor (partition.hpp): backward-solve row exchange and result masking.
// ---------------------------------------------------------------------------
// kPack: buf[off*nr + rr*cnt + i] = x[rows[i] + rr*n]; else the reverse.
template <bool kPack>
__global__ void __launch_bounds__(256) k_rows_xfer(const RowXfer* __restrict__ tasks,
                                                   double* __restrict__ x, int n, int nr,
                                                   double* __restrict__ buf) {
  const RowXfer t = tasks[blockIdx.x];
  double* b = buf + t.off * nr;
  for (int idx = threadIdx.x; idx < t.cnt * nr; idx += blockDim.x) {
    const int i = idx % t.cnt, rr = idx / t.cnt;
    double* xv = x + t.rows[i] + static_cast<int64_t>(rr) * n;
    if (kPack) b[idx] = *xv;
    else *xv = b[idx];
  }
}

// y[i + r*n] = 0 for the columns this rank does not own (before the all-reduce).
__global__ void k_mask_cols(double* __restrict__ y, const char* __restrict__ colmine, int n,
                            int nrhs) {
  const int64_t tot = static_cast<int64_t>(n) * nrhs;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < tot;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (!colmine[idx % n]) y[idx] = 0.0;
}

// ---------------------------------------------------------------------------
// Sampling and RBMC variances (gmrf.hpp:173-240).
// ---------------------------------------------------------------------------
// u[:, b] = mean + x[:, b] (vec_add, gmrf.hpp:179)
__global__ void k_add_mean(const double* __restrict__ mean, int n, int nb,
                           double* __restrict__ u) {
  const int64_t tot = static_cast<int64_t>(n) * nb;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < tot;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x)
    u[idx] = __dadd_rn(mean[idx % n], u[idx]);
}

// y[i, b] = Σ_j Q_ij c_j with c = u[:, b] − mean (vec_sub), Q symmetric: column i
// of the full CSC in ascending j — the accumulation order of matvec(Q, c)
// (sparse.hpp:130-147) for row i.
__global__ void k_rbmc_spmv(const int64_t* __restrict__ cp, const int32_t* __restrict__ ri,
                            const double* __restrict__ qv, const double* __restrict__ mean,
                            const double* __restrict__ u, int n, int nb,
                            double* __restrict__ y) {
  const int64_t tot = static_cast<int64_t>(n) * nb;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < tot;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(idx % n);
    const double* ub = u + (idx / n) * n;
    double s = 0.0;
    for (int64_t p = cp[i]; p < cp[i + 1]; ++p) {
      const int j = ri[p];
      s = __dadd_rn(s, __dmul_rn(qv[p], __dadd_rn(ub[j], -mean[j])));
    }
    y[idx] = s;
  }
}

// Welford update per coordinate over the batch's samples in draw order
// (gmrf.hpp:226-235): m = μ + c − (Qc)_i / Q_ii.
__global__ void k_rbmc_welford(const double* __restrict__ mean, const double* __restrict__ u,
                               const double* __restrict__ qc, const double* __restrict__ qdiag,
                               int n, int nb, int s0, double* __restrict__ mm,
                               double* __restrict__ m2) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double a = mm[i], b = m2[i];
    const double mu = mean[i], qd = qdiag[i];
    for (int k = 0; k < nb; ++k) {
      const double c = __dadd_rn(u[i + static_cast<int64_t>(k) * n], -mu);
      const double m = __dadd_rn(__dadd_rn(mu, c), -__ddiv_rn(qc[i + static_cast<int64_t>(k) * n], qd));
      const double delta = __dadd_rn(m, -a);
      a = __dadd_rn(a, __ddiv_rn(delta, static_cast<double>(s0 + k + 1)));
      b = __dadd_rn(b, __dmul_rn(delta, __dadd_rn(m, -a)));
    }
    mm[i] = a;
    m2[i] = b;
  }
}

__global__ void k_rbmc_final(const double* __restrict__ qdiag, const double* __restrict__ m2,
                             int n, int ns, double* __restrict__ var) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    var[i] = __dadd_rn(__ddiv_rn(1.0, qdiag[i]), __ddiv_rn(m2[i], static_cast<double>(ns - 1)));
}

// Q_ii from the full CSC (csc_diag); 0 if the diagonal is not stored
__global__ void k_csc_diag(const int64_t* __restrict__ cp, const int32_t* __restrict__ ri,
                           const double* __restrict__ qv, int n, double* __restrict__ d) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t p = cp[i]; p < cp[i + 1]; ++p)
      if (ri[p] == i) v = qv[p];
    d[i] = v;
  }
}

// ---------------------------------------------------------------------------
// Microbenchmarks for the FP64 roofline denominator (DMMA vs DFMA issue rate).
// ---------------------------------------------------------------------------
__global__ void k_bench_dmma(double* out, int iters) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma884(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_bench_dfma(double* out, int iters) {
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = i;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

}  // namespace gmrf
