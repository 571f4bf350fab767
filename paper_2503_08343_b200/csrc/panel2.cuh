// Two-phase panel step (all chunk levels): the chunk's diagonal block is
// factored ONCE, then every row below it is solved by its own thread.
//
//   k_panel_diag<W>  one CTA per chunk: the W diagonal-block rows run the
//                    right-looking column sweep of panel.cuh (diag_sweep: one
//                    barrier per column, correctly rounded pivots and
//                    divisions, cholesky.hpp:143,158). Publishes the block into
//                    the strict upper triangle + diag[] (k_diag_writeback moves
//                    it into place after the last level), 1/L_jj into rdiag[],
//                    and a dense column-major copy Lt[j*W + k] = L_kj with the
//                    pivots into the level's staging slot.
//   k_panel_trsm<W>  one CTA per 64-row slab below the block, one row per
//                    thread in registers, no barriers after staging: for each
//                    column j, l = a_ij / L_jj (correctly rounded: Markstein
//                    with RN(1/L_jj)), then a_ik -= l · L_kj for k > j — the
//                    same right-looking order as the diagonal rows.
//
// The previous fused kernels (panel.cuh) re-factored the diagonal block in
// every 128-row slab and serialized the slab rows on the same barriers; here
// the slab work is barrier-free and its CTAs are small enough to co-reside
// several per SM, so multi-wave levels no longer pay one 64-step chain per slab.
#pragma once

#include "panel.cuh"

namespace gmrf {

constexpr int kTrsm2Rows = 64;                  // rows per k_panel_trsm CTA
constexpr int kL11Slot = kNB * kNB + 2 * kNB;   // doubles per staging slot

template <int W>
__global__ void __launch_bounds__(panel_rows_diag<W>()) k_panel_diag(
    const PanelTask* __restrict__ tasks, int32_t* __restrict__ status, double* __restrict__ diag,
    double* __restrict__ rdiag, double* __restrict__ stage) {
  constexpr int DT = panel_rows_diag<W>();
  __shared__ __align__(16) double s_l[2][DT + 2];
  __shared__ __align__(16) double s_p[2][2];
  const PanelTask& t = tasks[blockIdx.x];
  const int w = t.w, ld = t.ld, tid = threadIdx.x;
  double r[W];
  {
    const double* src = t.d + tid;
#pragma unroll
    for (int k = 0; k < W; ++k)
      r[k] = (tid < w && k <= tid) ? src[static_cast<int64_t>(k) * ld] : (k == tid ? 1.0 : 0.0);
  }
  int bad = INT_MAX;
  if (tid == 0) {
    double p0, rp0;
    pivot_rn(r[0], p0, rp0);
    s_p[0][0] = p0;
    s_p[0][1] = rp0;
    if (w > 0 && !(r[0] > 0.0)) bad = 0;
  }
  double mypiv = 1.0, lp = 0.0;
  __syncthreads();
  diag_sweep<W, 0>(r, lp, mypiv, bad, tid, w, s_l, s_p, tid);
  if (bad != INT_MAX) atomicMin(status, t.gcol + bad);
  double* Lt = stage + static_cast<int64_t>(t.slot) * kL11Slot;
  double* pv = Lt + W * W;
  if (tid < W) {
    // column tid of the dense copy: Lt[j*W + tid] = L_{tid, j} (j < tid), else 0
#pragma unroll
    for (int j = 0; j < W; ++j) Lt[j * W + tid] = (j < tid && tid < w) ? r[j] : 0.0;
    const bool live = tid < w;
    const double rp = live ? 1.0 / mypiv : 1.0;  // RN(1/L_jj): exact Markstein division
    pv[2 * tid] = live ? mypiv : 1.0;
    pv[2 * tid + 1] = rp;
    if (live) {
      double* dst = t.d + static_cast<int64_t>(tid) * ld;  // row tid, transposed (upper)
#pragma unroll
      for (int k = 0; k < W; ++k)
        if (k < tid) dst[k] = r[k];
      diag[t.gcol + tid] = mypiv;
      rdiag[t.gcol + tid] = rp;
    }
  }
}

// r[k] -= l · lt[k] for k in [K0, W): shared loads two at a time, issued in
// groups of 8 (an empty asm with a memory clobber keeps the compiler from
// hoisting every load of the column ahead of the FMAs, which spills r[])
template <int W, int K0>
__device__ __forceinline__ void col_update(double (&r)[W], double l, const double* lt) {
  if constexpr (K0 < W) {
    if constexpr (K0 & 1) {
      r[K0] = fma(-l, lt[K0], r[K0]);
      col_update<W, K0 + 1>(r, l, lt);
    } else {
#pragma unroll
      for (int k = K0; k + 1 < W; k += 2) {
        if (((k - K0) & 15) == 0) asm volatile("" ::: "memory");
        const double2 v = *reinterpret_cast<const double2*>(lt + k);
        r[k] = fma(-l, v.x, r[k]);
        r[k + 1] = fma(-l, v.y, r[k + 1]);
      }
    }
  }
}

template <int W, int J>
__device__ __forceinline__ void trsm_sweep(double (&r)[W], const double* Lt, const double* pv) {
  if constexpr (J < W) {
    const double2 pr = *reinterpret_cast<const double2*>(pv + 2 * J);
    const double l = div_rn(r[J], pr.x, pr.y);
    r[J] = l;
    col_update<W, J + 1>(r, l, Lt + J * W);
    trsm_sweep<W, J + 1>(r, Lt, pv);
  }
}

template <int W>
__global__ void __launch_bounds__(kTrsm2Rows, 1) k_panel_trsm(const PanelTask* __restrict__ tasks,
                                                           const double* __restrict__ stage) {
  __shared__ __align__(16) double sm[W * W + 2 * W];
  const PanelTask& t = tasks[blockIdx.x];
  const int w = t.w, ld = t.ld, tid = threadIdx.x;
  const double* Lt = stage + static_cast<int64_t>(t.slot) * kL11Slot;
  for (int q = tid; q < (W * W + 2 * W) / 2; q += kTrsm2Rows) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm + 2 * q));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(Lt + 2 * q));
  }
  const int r0 = t.tile * kTrsm2Rows;
  const int nr = min(kTrsm2Rows, t.nbelow - r0);
  double r[W];
  double* B = t.d + w + r0 + tid;
  const bool act = tid < nr;
#pragma unroll
  for (int k = 0; k < W; ++k) r[k] = (act && k < w) ? B[static_cast<int64_t>(k) * ld] : 0.0;
  cpasync_wait_all();
  __syncthreads();
  trsm_sweep<W, 0>(r, sm, sm + W * W);
  if (act) {
    // opaque copy of B: the store addresses are recomputed here instead of
    // being kept live (64 address registers) across the sweep
    double* Bs;
    asm("mov.b64 %0, %1;" : "=l"(Bs) : "l"(B));
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k < w) Bs[static_cast<int64_t>(k) * ld] = r[k];
  }
}

}  // namespace gmrf
