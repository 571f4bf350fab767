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

}  // namespace gmrf
