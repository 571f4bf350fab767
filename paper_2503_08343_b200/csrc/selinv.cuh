// Per-chunk dense steps of the supernodal selected inversion (takahashi.hpp
// recurrences, supernodal form), register resident and barrier free:
//   k_sel_trsm<W>: dst = −src · L_JJ⁻¹ for one 128-row slab, one row per
//                  thread (x·L = b, right-looking over the columns, j descending):
//                  Σ_{R,J} from Y, and Z = −W L_JJ⁻¹ from W = L_{R,J}ᵀ Y;
//   k_sel_diag<W>: Σ_JJ = L_JJ⁻ᵀ (L_JJ⁻¹ − Z), one column per thread:
//                  forward solve L x = e_c, subtract z_c, backward solve Lᵀ s = x.
// W is the chunk width bucket (16/32/64, identity padded). L_JJ is staged once
// in shared memory and read by broadcast; divisions are correctly rounded
// (div_rn with the correctly rounded 1/L_jj of the factorization).
#pragma once

#include "kernels.cuh"
#include "panel.cuh"

namespace gmrf {

template <int W>
constexpr int sel_diag_smem_bytes() {
  return (2 * W * (W + 1) + W) * static_cast<int>(sizeof(double));
}

template <int W>
__global__ void __launch_bounds__(kTrsmRows) k_sel_trsm_w(const SelChunk* __restrict__ tasks) {
  constexpr int LP = W + 2;  // even pitch: rows stay 16-byte aligned for the double2 reads
  __shared__ __align__(16) double Lr[W * LP];  // Lr[j*LP + k] = L_jk (row j of L_JJ, k < j)
  __shared__ double dg[W], rd[W];
  const SelChunk& t = tasks[blockIdx.x];
  const int w = t.w, ld = t.ld, tid = threadIdx.x;
  const double* Lk = t.l + t.c0 + static_cast<int64_t>(t.c0) * ld;
  // fully unrolled (compile-time trip count): every thread's loads are in flight
  // together instead of one memory round trip per element; consecutive threads
  // read consecutive rows of a column (coalesced), the transpose happens in the
  // shared-memory write
#pragma unroll
  for (int idx = tid; idx < W * W; idx += kTrsmRows) {
    const int j = idx % W, k = idx / W;
    Lr[j * LP + k] = (k < j && j < w) ? Lk[j + static_cast<int64_t>(k) * ld] : 0.0;
  }
  if (tid < W) {
    dg[tid] = tid < w ? Lk[tid + static_cast<int64_t>(tid) * ld] : 1.0;
    rd[tid] = tid < w ? t.rd[tid] : 1.0;
  }
  const int r0 = t.tile * kTrsmRows;
  const int nr = min(kTrsmRows, t.nrows - r0);
  const double* B = t.src + r0 + tid;
  double* D = t.dst + r0 + tid;
  const bool act = tid < nr;
  double b[W];
#pragma unroll
  for (int j = 0; j < W; ++j) b[j] = (act && j < w) ? -B[static_cast<int64_t>(j) * t.lds] : 0.0;
  __syncthreads();
#pragma unroll
  for (int j = W - 1; j >= 0; --j) {
    const double x = div_rn(b[j], dg[j], rd[j]);
    b[j] = x;
    const double* lj = Lr + j * LP;
#pragma unroll
    for (int k = 0; k + 1 < j; k += 2) {
      const double2 v = *reinterpret_cast<const double2*>(lj + k);
      b[k] = fma(-x, v.x, b[k]);
      b[k + 1] = fma(-x, v.y, b[k + 1]);
    }
    if (j & 1) b[j - 1] = fma(-x, lj[j - 1], b[j - 1]);
  }
  if (act) {
#pragma unroll
    for (int j = 0; j < W; ++j)
      if (j < w) D[static_cast<int64_t>(j) * t.ldd] = b[j];
  }
  (void)ld;
}

template <int W>
__global__ void __launch_bounds__(W < 32 ? 32 : W) k_sel_diag_w(const SelChunk* __restrict__ tasks) {
  extern __shared__ __align__(16) double sm[];
  constexpr int P = W + 1;
  double* Lc = sm;          // Lc[i*P + k] = L_ki (column i), k > i
  double* Lt = sm + W * P;  // Lt[i*P + k] = L_ik (row i),    k < i
  double* rd = sm + 2 * W * P;
  const SelChunk& t = tasks[blockIdx.x];
  const int w = t.w, ld = t.ld, tid = threadIdx.x;
  const double* Lk = t.l + t.c0 + static_cast<int64_t>(t.c0) * ld;
  double* Sk = t.sig + t.c0 + static_cast<int64_t>(t.c0) * ld;
  // L_JJ read once, coalesced (consecutive threads: consecutive rows k of column
  // i), all of a thread's loads in flight together; the row copy Lt is the
  // shared-memory transpose
  constexpr int NT = W < 32 ? 32 : W;
#pragma unroll 16
  for (int idx = tid; idx < W * W; idx += NT) {
    const int i = idx / W, k = idx % W;
    const bool in = i < w && k < w;
    Lc[i * P + k] = (in && k >= i) ? Lk[k + static_cast<int64_t>(i) * ld] : (k == i ? 1.0 : 0.0);
  }
  if (tid < W) rd[tid] = tid < w ? t.rd[tid] : 1.0;
  __syncthreads();
  for (int idx = tid; idx < W * W; idx += NT) {
    const int i = idx / W, k = idx % W;
    Lt[i * P + k] = k <= i ? Lc[k * P + i] : 0.0;  // L_ik = column k's entry i (1 on the padding)
  }
  const int c = tid;
  const bool act = c < w;
  double x[W];
#pragma unroll
  for (int k = 0; k < W; ++k) x[k] = (k == c) ? 1.0 : 0.0;
  __syncthreads();
  // L x = e_c
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const double xi = div_rn(x[i], Lc[i * P + i], rd[i]);
    x[i] = xi;
#pragma unroll
    for (int k = i + 1; k < W; ++k) x[k] = fma(-xi, Lc[i * P + k], x[k]);
  }
  // x − z_c  (Z = L_{R,J}ᵀ Σ_{R,J}, staged by the plan in its own w × w slot)
  if (act) {
    const double* zc = t.z + static_cast<int64_t>(c) * t.ldz;
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k < w) x[k] -= zc[k];
  }
  // Lᵀ s = x
#pragma unroll
  for (int i = W - 1; i >= 0; --i) {
    const double si = div_rn(x[i], Lt[i * P + i], rd[i]);
    x[i] = si;
#pragma unroll
    for (int k = 0; k < i; ++k) x[k] = fma(-si, Lt[i * P + k], x[k]);
  }
  __syncthreads();  // every thread has read L_JJ before Σ_JJ overwrites it (in place)
  if (act) {
#pragma unroll
    for (int i = 0; i < W; ++i)
      if (i >= c && i < w) {
        Sk[i + static_cast<int64_t>(c) * ld] = x[i];
        Sk[c + static_cast<int64_t>(i) * ld] = x[i];
      }
  }
}

// Mirror Σ_{P,J} → Σ_{J,P} (P = the supernode's later columns) for one 64-row
// tile of P, transposed through shared memory so reads and writes coalesce.
__global__ void __launch_bounds__(256) k_sel_mirror(const SelChunk* __restrict__ tasks) {
  __shared__ double T[64][65];
  const SelChunk& t = tasks[blockIdx.x];
  const int w = t.w, ld = t.ld, tid = threadIdx.x;
  const int p = t.wsn - t.c0 - w;
  const int p0 = t.tile * 64, np = min(64, p - p0);
  double* Sk = t.sig + t.c0 + static_cast<int64_t>(t.c0) * ld;
  for (int idx = tid; idx < 64 * w; idx += blockDim.x) {  // read: rows of P contiguous
    const int i = idx & 63, j = idx >> 6;
    if (i < np) T[j][i] = Sk[(w + p0 + i) + static_cast<int64_t>(j) * ld];
  }
  __syncthreads();
  for (int idx = tid; idx < 64 * w; idx += blockDim.x) {  // write: chunk columns contiguous
    const int j = idx % w, i = idx / w;
    if (i < np) Sk[j + static_cast<int64_t>(w + p0 + i) * ld] = T[j][i];
  }
}

// ---------------------------------------------------------------------------
// Blocked selected inversion of a multi-chunk supernode (factor.cu,
// build_selinv_plan): instead of a chain of 64-column chunk steps, the whole
// supernode J (w columns, rows R below) is done with a few batched GEMM stages:
//   W  = L_JJ⁻¹                     (k_tri_inv64 on the diagonal blocks, then
//                                    log2(chunks) merge steps  X = −C⁻¹ B A⁻¹)
//   Gn = −L_RJ W,  Σ_RJ = Σ_RR Gn,  Σ_JJ = Wᵀ W + Gnᵀ Σ_RJ
// (takahashi.hpp:43-60 in supernodal form, e.g. Lin et al., SelInv).
//
// k_tri_inv64: dst (w × w block of the W workspace, zeros above the diagonal)
// = inverse of the chunk's lower-triangular diagonal block; one column per
// thread, forward substitution L x = e_c with L_JJ staged in shared memory.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(64) k_tri_inv64(const SelChunk* __restrict__ tasks) {
  constexpr int W = 64, P = W + 1;
  __shared__ double Lc[W * P];  // Lc[i*P + k] = L_ki (column i), k >= i
  __shared__ double rd[W];
  const SelChunk& t = tasks[blockIdx.x];
  const int w = t.w, ld = t.ld, tid = threadIdx.x;
  const double* Lk = t.l + t.c0 + static_cast<int64_t>(t.c0) * ld;
#pragma unroll 16
  for (int idx = tid; idx < W * W; idx += W) {
    const int i = idx / W, k = idx % W;
    const bool in = i < w && k < w;
    Lc[i * P + k] = (in && k >= i) ? Lk[k + static_cast<int64_t>(i) * ld] : (k == i ? 1.0 : 0.0);
  }
  rd[tid] = tid < w ? t.rd[tid] : 1.0;
  const int c = tid;
  double x[W];
#pragma unroll
  for (int k = 0; k < W; ++k) x[k] = (k == c) ? 1.0 : 0.0;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const double xi = div_rn(x[i], Lc[i * P + i], rd[i]);
    x[i] = xi;
#pragma unroll
    for (int k = i + 1; k < W; ++k) x[k] = fma(-xi, Lc[i * P + k], x[k]);
  }
  if (c < w) {
    double* D = t.dst + static_cast<int64_t>(c) * t.ldd;
#pragma unroll
    for (int i = 0; i < W; ++i)
      if (i < w) D[i] = i >= c ? x[i] : 0.0;
  }
}

// Σ_JJ tile (rows c0.., columns tile.., w × wsn entries, c0 >= tile) mirrored
// into the upper triangle: Σ[j, i] = Σ[i, j] for i > j, through shared memory.
__global__ void __launch_bounds__(256) k_sel_mirror_blk(const SelChunk* __restrict__ tasks) {
  __shared__ double T[64][65];
  const SelChunk& t = tasks[blockIdx.x];
  const int m = t.w, n = t.wsn, i0 = t.c0, j0 = t.tile, tid = threadIdx.x;
  const int64_t ld = t.ld;
  double* S = t.sig;
  for (int idx = tid; idx < 64 * n; idx += blockDim.x) {
    const int i = idx & 63, j = idx >> 6;
    if (i < m) T[j][i] = S[(i0 + i) + (j0 + j) * ld];
  }
  __syncthreads();
  for (int idx = tid; idx < 64 * m; idx += blockDim.x) {
    const int j = idx & 63, i = idx >> 6;
    if (j < n && i0 + i > j0 + j) S[(j0 + j) + (i0 + i) * ld] = T[j][i];
  }
}

}  // namespace gmrf
