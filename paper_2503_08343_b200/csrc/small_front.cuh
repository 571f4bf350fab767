// Fused multifrontal step for small supernodes (rows ≤ RB ≤ 96), one CTA per
// front: the whole front (L panel columns + update block) lives in shared
// memory; the CTA extend-adds its children, factors the w pivot columns
// right-looking (pivot via rsqrt, column scale, rank-1 trailing update over the
// full front), then writes the L panel and the update matrix U. The bottom
// tree levels hold tens of thousands of such fronts; this replaces their
// extend-add, panel and GEMM launches and keeps U round trips in shared memory.
// Children are visited in order and each entry is owned by one thread per
// child, so the summation order is fixed (deterministic).
#pragma once

#include "kernels.cuh"
#include "panel.cuh"

namespace gmrf {

template <int RB>
constexpr int small_front_smem_bytes() {
  return RB * (RB + 1) * static_cast<int>(sizeof(double));
}

template <int RB>
__global__ void __launch_bounds__(256) k_small_front(const int32_t* __restrict__ sns, SymDev sd,
                                                     double* __restrict__ L,
                                                     double* __restrict__ U,
                                                     int32_t* __restrict__ status,
                                                     double* __restrict__ rdiag) {
  extern __shared__ double F[];  // F[j*FP + i], front rows × rows, column-major
  constexpr int FP = RB + 1;
  __shared__ double sh_rs, sh_rp;
  const int s = sns[blockIdx.x];
  const int f0 = sd.sn_first[s];
  const int w = sd.sn_first[s + 1] - f0;
  const int rows = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]);
  const int r = rows - w;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Ls = L + sd.lptr[s];
  double* Us = U + sd.uptr[s];
  // 1. front = [L panel (A values) | 0]
  for (int j = warp; j < rows; j += 8)
    for (int i = lane; i < rows; i += 32) {
      if (j < w) cpasync8(&F[j * FP + i], Ls + i + static_cast<int64_t>(j) * rows);
      else F[j * FP + i] = 0.0;
    }
  cpasync_wait_all();
  __syncthreads();
  // 2. extend-add the children's update matrices (lower triangles)
  for (int q = sd.ch_ptr[s]; q < sd.ch_ptr[s + 1]; ++q) {
    const int c = sd.ch_list[q];
    const int wc = sd.sn_first[c + 1] - sd.sn_first[c];
    const int rc = static_cast<int>(sd.sn_rptr[c + 1] - sd.sn_rptr[c]) - wc;
    const int32_t* rel = sd.relmap + sd.sn_rptr[c] + wc;
    const double* Uc = U + sd.uptr[c];
    for (int jb = warp; jb < rc; jb += 8) {
      const int b = rel[jb];
      const double* col = Uc + static_cast<int64_t>(jb) * rc;
      for (int ia = jb + lane; ia < rc; ia += 32) F[b * FP + rel[ia]] += col[ia];
    }
    __syncthreads();
  }
  // 3. right-looking partial Cholesky of the w pivot columns
  for (int j = 0; j < w; ++j) {
    if (tid == 0) {
      // correctly rounded pivot and division, as cholesky.hpp:143,158
      const double d = F[j * FP + j];
      if (!(d > 0.0)) atomicMin(status, f0 + j);
      const double p = sqrt_rn_pos(d);
      const double rp = recip_nr(p);
      F[j * FP + j] = p;
      sh_rs = p;
      sh_rp = rp;
      rdiag[f0 + j] = div_rn(1.0, p, rp);
    }
    __syncthreads();
    const double p = sh_rs, rp = sh_rp;
    for (int i = j + 1 + tid; i < rows; i += blockDim.x) F[j * FP + i] = div_rn(F[j * FP + i], p, rp);
    __syncthreads();
    for (int k = j + 1 + warp; k < rows; k += 8) {
      const double lk = F[j * FP + k];
      for (int i = k + lane; i < rows; i += 32) F[k * FP + i] -= F[j * FP + i] * lk;
    }
    __syncthreads();
  }
  // 4. write the L panel (lower part) and the update matrix
  for (int j = warp; j < w; j += 8)
    for (int i = j + lane; i < rows; i += 32) Ls[i + static_cast<int64_t>(j) * rows] = F[j * FP + i];
  for (int jb = warp; jb < r; jb += 8)
    for (int ia = jb + lane; ia < r; ia += 32)
      Us[ia + static_cast<int64_t>(jb) * r] = F[(w + jb) * FP + (w + ia)];
}

// Row-sweep variant for the largest small fronts (64 < rows ≤ 96), bucketed by
// pivot count w ≤ W. Assembly as above (front in shared memory, children in
// order); then the w pivot columns are factored by the register-resident
// right-looking column sweep of the panel kernels (panel.cuh diag_sweep: thread
// per front row, one barrier per column, correctly rounded pivots/divisions,
// cholesky.hpp:143,158) instead of three barriers and a shared-memory rank-1
// update of the whole front per column; the update block then takes ONE
// symmetric rank-w update U = F22 − L21 L21ᵀ from shared memory in 4×4
// register tiles, the k terms in pivot order (the same order of operations as
// the rank-1 sequence).
template <int W>
__host__ __device__ constexpr int small_rows_slab() {
  return W == 64 ? 64 : 96;  // rows below the pivots: ≤ 96 − w
}
template <int W>
__host__ __device__ constexpr int small_rows_threads() {
  return panel_rows_diag<W>() + small_rows_slab<W>();
}

// W <= 32: three CTAs per SM (the 96×97 front in shared memory allows three; the
// default register allocation of 255 only two)
template <int W>
__global__ void __launch_bounds__(small_rows_threads<W>(), W <= 32 ? 3 : 1)
    k_small_front_rows(const int32_t* __restrict__ sns, SymDev sd, double* __restrict__ L,
                       double* __restrict__ U, int32_t* __restrict__ status,
                       double* __restrict__ rdiag) {
  constexpr int RB = 96, FP = RB + 1, DT = panel_rows_diag<W>(), NT = small_rows_threads<W>();
  extern __shared__ double F[];  // F[j*FP + i], front rows × rows, column-major
  __shared__ __align__(16) double s_l[2][DT + 2];
  __shared__ __align__(16) double s_p[2][2];
  const int s = sns[blockIdx.x];
  const int f0 = sd.sn_first[s];
  const int w = sd.sn_first[s + 1] - f0;
  const int rows = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]);
  const int r = rows - w;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  double* Ls = L + sd.lptr[s];
  double* Us = U + sd.uptr[s];
  // 1. front = [L panel (A values) | 0], then the children's update matrices
  for (int j = warp; j < rows; j += NW)
    for (int i = lane; i < rows; i += 32) {
      if (j < w) cpasync8(&F[j * FP + i], Ls + i + static_cast<int64_t>(j) * rows);
      else F[j * FP + i] = 0.0;
    }
  cpasync_wait_all();
  __syncthreads();
  for (int q = sd.ch_ptr[s]; q < sd.ch_ptr[s + 1]; ++q) {
    const int c = sd.ch_list[q];
    const int wc = sd.sn_first[c + 1] - sd.sn_first[c];
    const int rc = static_cast<int>(sd.sn_rptr[c + 1] - sd.sn_rptr[c]) - wc;
    const int32_t* rel = sd.relmap + sd.sn_rptr[c] + wc;
    const double* Uc = U + sd.uptr[c];
    for (int jb = warp; jb < rc; jb += NW) {
      const int b = rel[jb];
      const double* col = Uc + static_cast<int64_t>(jb) * rc;
      for (int ia = jb + lane; ia < rc; ia += 32) F[b * FP + rel[ia]] += col[ia];
    }
    __syncthreads();
  }
  // 2. pivot rows (tid < DT, identity-padded beyond w) and rows below
  const bool is_diag = tid < DT;
  const int a = is_diag ? tid : w + (tid - DT);  // front row of this thread
  const bool live = is_diag ? tid < w : a < rows;
  double rg[W];
#pragma unroll
  for (int k = 0; k < W; ++k)
    rg[k] = is_diag ? ((tid < w && k <= tid) ? F[k * FP + tid] : (k == tid ? 1.0 : 0.0))
                    : ((live && k < w) ? F[k * FP + a] : 0.0);
  int bad = INT_MAX;
  if (tid == 0) {
    double p0, rp0;
    pivot_rn(rg[0], p0, rp0);
    s_p[0][0] = p0;
    s_p[0][1] = rp0;
    if (w > 0 && !(rg[0] > 0.0)) bad = 0;
  }
  double mypiv = 1.0, lp = 0.0;
  __syncthreads();
  diag_sweep<W, 0>(rg, lp, mypiv, bad, is_diag ? tid : (1 << 20), w, s_l, s_p, is_diag ? tid : DT);
  if (bad != INT_MAX) atomicMin(status, f0 + bad);
  // 3. L panel out; L21 into its front slots for the update
  if (is_diag && live) {
    double* dst = Ls + tid;
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k <= tid) dst[static_cast<int64_t>(k) * rows] = k == tid ? mypiv : rg[k];
    rdiag[f0 + tid] = 1.0 / mypiv;
  } else if (!is_diag && live) {
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k < w) {
        Ls[a + static_cast<int64_t>(k) * rows] = rg[k];
        F[k * FP + a] = rg[k];
      }
  }
  __syncthreads();
  // 4. U = F22 − L21 L21ᵀ, 4×4 tiles of the lower triangle, k in pivot order
  const int nb = (r + 3) / 4;
  for (int t = tid; t < nb * (nb + 1) / 2; t += NT) {
    int bi = static_cast<int>((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);  // t = bi(bi+1)/2 + bj
    while (bi * (bi + 1) / 2 > t) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    const int bj = t - bi * (bi + 1) / 2;
    const int i0 = w + 4 * bi, j0 = w + 4 * bj;
    double acc[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y)
        acc[x][y] = (i0 + x < rows && j0 + y < rows) ? F[(j0 + y) * FP + i0 + x] : 0.0;
    for (int k = 0; k < w; ++k) {
      double li[4], lj[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        li[x] = F[k * FP + min(i0 + x, RB - 1)];
        lj[x] = F[k * FP + min(j0 + x, RB - 1)];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fma(-li[x], lj[y], acc[x][y]);
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int ia = i0 + x - w, jb = j0 + y - w;
        if (ia < r && jb < r && ia >= jb) Us[ia + static_cast<int64_t>(jb) * r] = acc[x][y];
      }
  }
}

}  // namespace gmrf
