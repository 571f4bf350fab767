// Supernodal triangular solves (cholesky.hpp:179-222 semantics), level by
// level over the supernodal tree. Per level and sweep, two launches:
//   *_diag : one CTA per supernode — the dense w×w triangle L_JJ, blocked by
//            64-column chunks whose diagonal blocks are staged in shared memory
//            and solved by one warp;
//   *_off  : many CTAs per supernode — the rectangular L_RJ part, 128-row tiles,
//            streaming L once with coalesced column reads.
// Supernodes with at most kSolveFuseRows rows below the triangle do their
// rectangular part inside the *_diag kernel (no tiles, one launch per level for
// the many small supernodes of the lower tree levels).
// Deterministic: children are accumulated in a fixed order and the backward
// partial sums over row tiles are reduced in tile order.
#pragma once

#include "kernels.cuh"
#include "solve_tile.hpp"

namespace gmrf {

// acc[rr] -= Σ_j li[j·ld] · v[rr·vs + j] for j = 0..nj-1, in ascending j (the
// same accumulation order as a plain loop), with kGemvU independent L loads in
// flight per thread: a thread walks one row of a column-major panel, so its
// loads are strided and each batch costs a full memory round trip.
template <int NR>
__device__ __forceinline__ void row_gemv_sub(double (&acc)[NR], const double* __restrict__ li,
                                             int64_t ld, const double* v, int vs, int nrhs,
                                             int nj) {
  constexpr int U = NR == 1 ? 32 : 16;
  int j = 0;
  for (; j + U <= nj; j += U) {
    double l[U];
#pragma unroll
    for (int u = 0; u < U; ++u) l[u] = li[static_cast<int64_t>(j + u) * ld];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) acc[rr] -= l[u] * v[rr * vs + j + u];
  }
  for (; j + 8 <= nj; j += 8) {
    double l[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) l[u] = li[static_cast<int64_t>(j + u) * ld];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) acc[rr] -= l[u] * v[rr * vs + j + u];
  }
  for (; j < nj; ++j) {
    const double l = li[static_cast<int64_t>(j) * ld];
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) acc[rr] -= l * v[rr * vs + j];
  }
  (void)nrhs;
}


// Warp dot products over CJ columns at once: acc[c][rr] += Σ_i col_c[i] · x[rr·xs + i]
// for i = lane, lane+32, … < nt (per-lane partials in ascending i, as a
// one-column loop), columns col0 + c·cs for c < nc; CJ columns' loads in flight.
template <int NR, int CJ>
__device__ __forceinline__ void warp_col_dots(double (&acc)[CJ][NR], const double* __restrict__ col0,
                                              int64_t cs, int nc, const double* x, int xs, int nt,
                                              int lane) {
#pragma unroll
  for (int c = 0; c < CJ; ++c)
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) acc[c][rr] = 0.0;
#pragma unroll 4
  for (int ii = lane; ii < nt; ii += 32) {
    double l[CJ];
#pragma unroll
    for (int c = 0; c < CJ; ++c) l[c] = c < nc ? col0[c * cs + ii] : 0.0;
#pragma unroll
    for (int c = 0; c < CJ; ++c)
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) acc[c][rr] += l[c] * x[rr * xs + ii];
  }
}

// ---- forward: diagonal triangle + children assembly -------------------------
template <int NR>
__global__ void __launch_bounds__(256) k_fsolve_diag(const int32_t* __restrict__ sns, SymDev sd,
                                                     const double* __restrict__ L,
                                                     double* __restrict__ y, int nrhs,
                                                     double* __restrict__ Uv,
                                                     const int64_t* __restrict__ uvptr,
                                                     const double* __restrict__ rdiag) {
  extern __shared__ double sm[];
  __shared__ double rdl[64];  // 1/L_jj of the current chunk
  const int s = sns[blockIdx.x];
  const int f0 = sd.sn_first[s];
  const int w = sd.sn_first[s + 1] - f0;
  const int rows = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]);
  const int r = rows - w;
  const int n = sd.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Ls = L + sd.lptr[s];
  double* fJ = sm;                 // [rr*w + a]
  double* Lb = sm + w * NR;        // [j*65 + i]
  double* uS = Uv + uvptr[s] * nrhs;  // [i + rr*r]
  for (int idx = tid; idx < w * nrhs; idx += blockDim.x) {
    const int a = idx % w, rr = idx / w;
    fJ[rr * w + a] = y[f0 + a + static_cast<int64_t>(rr) * n];
  }
  for (int idx = tid; idx < r * nrhs; idx += blockDim.x) uS[idx] = 0.0;
  __syncthreads();
  for (int q = sd.ch_ptr[s]; q < sd.ch_ptr[s + 1]; ++q) {
    const int c = sd.ch_list[q];
    const int wc = sd.sn_first[c + 1] - sd.sn_first[c];
    const int rc = static_cast<int>(sd.sn_rptr[c + 1] - sd.sn_rptr[c]) - wc;
    const int32_t* rel = sd.relmap + sd.sn_rptr[c] + wc;
    const double* uc = Uv + uvptr[c] * nrhs;
    child_scatter<4>(rel, uc, rc, nrhs, [&](int a, int rr) {
      return a < w ? fJ + rr * w + a : uS + (a - w) + rr * r;
    });
    __syncthreads();
  }
  for (int c0 = 0; c0 < w; c0 += 64) {
    const int wk = min(64, w - c0);
    for (int idx = tid; idx < wk * wk; idx += blockDim.x) {
      const int i = idx % wk, j = idx / wk;
      if (i >= j) cpasync8(&Lb[j * 65 + i], Ls + (c0 + i) + static_cast<int64_t>(c0 + j) * rows);
    }
    if (tid < wk) cpasync8(&rdl[tid], rdiag + f0 + c0 + tid);
    cpasync_wait_all();
    __syncthreads();
    if (warp == 0) {
      double v0[NR], v1[NR];
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        v0[rr] = (rr < nrhs && lane < wk) ? fJ[rr * w + c0 + lane] : 0.0;
        v1[rr] = (rr < nrhs && lane + 32 < wk) ? fJ[rr * w + c0 + 32 + lane] : 0.0;
      }
      for (int j = 0; j < wk; ++j) {
        const double rjj = rdl[j];  // 1/L_jj, from the factorization
        const double l0 = (lane > j && lane < wk) ? Lb[j * 65 + lane] : 0.0;
        const double l1 = (lane + 32 > j && lane + 32 < wk) ? Lb[j * 65 + lane + 32] : 0.0;
#pragma unroll
        for (int rr = 0; rr < NR; ++rr) {
          const double src = j < 32 ? v0[rr] : v1[rr];
          const double xj = __shfl_sync(0xffffffffu, src, j & 31) * rjj;
          if (lane == (j & 31)) {
            if (j < 32) v0[rr] = xj; else v1[rr] = xj;
          }
          v0[rr] -= l0 * xj;
          v1[rr] -= l1 * xj;
        }
      }
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        if (rr >= nrhs) break;
        if (lane < wk) fJ[rr * w + c0 + lane] = v0[rr];
        if (lane + 32 < wk) fJ[rr * w + c0 + 32 + lane] = v1[rr];
      }
    }
    __syncthreads();
    // remaining rows of the triangle: f_i -= L[i, chunk] · x_chunk
    for (int i = c0 + wk + tid; i < w; i += blockDim.x) {
      double acc[NR];
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) acc[rr] = rr < nrhs ? fJ[rr * w + i] : 0.0;
      row_gemv_sub<NR>(acc, Ls + i + static_cast<int64_t>(c0) * rows, rows, fJ + c0, w, nrhs, wk);
#pragma unroll
      for (int rr = 0; rr < NR; ++rr)
        if (rr < nrhs) fJ[rr * w + i] = acc[rr];
    }
    __syncthreads();
  }
  if (r <= kSolveFuseRows) {  // u_R = f_R − L_RJ y_J here (no off-diagonal tiles)
    for (int i = tid; i < r; i += blockDim.x) {
      double acc[NR];
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) acc[rr] = rr < nrhs ? uS[i + rr * r] : 0.0;
      row_gemv_sub<NR>(acc, Ls + w + i, rows, fJ, w, nrhs, w);
#pragma unroll
      for (int rr = 0; rr < NR; ++rr)
        if (rr < nrhs) uS[i + rr * r] = acc[rr];
    }
  }
  for (int idx = tid; idx < w * nrhs; idx += blockDim.x) {
    const int a = idx % w, rr = idx / w;
    y[f0 + a + static_cast<int64_t>(rr) * n] = fJ[rr * w + a];
  }
}

// ---- forward: u_R = f_R − L_RJ y_J, 128-row tiles ---------------------------
// Row tiles of wide supernodes are split into column blocks (kSolveSplitCols):
// each block writes its partial Σ_j L_ij y_j to PF, and the CTA that arrives
// last for the row tile subtracts the partials from u in block order (fixed
// order; the arrival counter wraps back to 0 by itself via atomicInc).
template <int NR>
__global__ void __launch_bounds__(kSolveRows) k_fsolve_off(const SolveTile* __restrict__ tiles,
                                                          SymDev sd, const double* __restrict__ L,
                                                          const double* __restrict__ y, int nrhs,
                                                          double* __restrict__ Uv,
                                                          const int64_t* __restrict__ uvptr,
                                                          double* __restrict__ PF,
                                                          unsigned* __restrict__ ctr) {
  constexpr int CW = kSolveOffCols;
  __shared__ double yJ[CW * NR];  // [rr*CW + j], one column chunk of y_J
  __shared__ bool last;
  const SolveTile t = tiles[blockIdx.x];
  const int s = t.sn;
  const int f0 = sd.sn_first[s];
  const int w = sd.sn_first[s + 1] - f0;
  const int rows = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]);
  const int r = rows - w;
  const int n = sd.n;
  const int i = t.r0 + threadIdx.x;
  const bool active = i < r;
  const bool split = t.nparts > 1;
  const double* Lr = L + sd.lptr[s] + w + i;
  double* u = Uv + uvptr[s] * nrhs;
  double acc[NR];
#pragma unroll
  for (int rr = 0; rr < NR; ++rr) acc[rr] = (active && rr < nrhs && !split) ? u[i + rr * r] : 0.0;
  for (int c0 = t.c0; c0 < t.c1; c0 += CW) {
    const int wc = min(CW, t.c1 - c0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < wc * nrhs; idx += blockDim.x) {
      const int a = idx % wc, rr = idx / wc;
      yJ[rr * CW + a] = y[f0 + c0 + a + static_cast<int64_t>(rr) * n];
    }
    __syncthreads();
    if (!active) continue;
    row_gemv_sub<NR>(acc, Lr + static_cast<int64_t>(c0) * rows, rows, yJ, CW, nrhs, wc);
  }
  if (!split) {
    if (!active) return;
#pragma unroll
    for (int rr = 0; rr < NR; ++rr)
      if (rr < nrhs) u[i + rr * r] = acc[rr];
    return;
  }
  // partial (already negated) → PF[slot][rr][row]
  double* mine = PF + static_cast<int64_t>(t.pf + t.part) * NR * kSolveRows;
#pragma unroll
  for (int rr = 0; rr < NR; ++rr) mine[rr * kSolveRows + threadIdx.x] = acc[rr];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicInc(ctr + t.ctr, t.nparts - 1) == static_cast<unsigned>(t.nparts - 1);
  __syncthreads();
  if (!last || !active) return;
  __threadfence();
  const double* base = PF + static_cast<int64_t>(t.pf) * NR * kSolveRows;
#pragma unroll
  for (int rr = 0; rr < NR; ++rr) {
    if (rr >= nrhs) break;
    double v = u[i + rr * r];
    for (int p = 0; p < t.nparts; ++p)
      v += __ldcg(base + static_cast<int64_t>(p) * NR * kSolveRows + rr * kSolveRows + threadIdx.x);
    u[i + rr * r] = v;
  }
}

// ---- backward: partial sums t = L_RJᵀ x_R over 128-row tiles ----------------
template <int NR>
__global__ void __launch_bounds__(256) k_bsolve_off(const SolveTile* __restrict__ tiles, SymDev sd,
                                                    const double* __restrict__ L,
                                                    const double* __restrict__ x, int nrhs,
                                                    double* __restrict__ P,
                                                    const int64_t* __restrict__ pptr) {
  __shared__ double xR[kSolveRows * NR];
  const SolveTile t = tiles[blockIdx.x];
  const int s = t.sn;
  const int f0 = sd.sn_first[s];
  const int w = sd.sn_first[s + 1] - f0;
  const int rows = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]);
  const int r = rows - w;
  const int n = sd.n;
  const int nt = min(kSolveRows, r - t.r0);
  const int32_t* srows = sd.sn_rows + sd.sn_rptr[s] + w + t.r0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < nt * nrhs; idx += blockDim.x) {
    const int ii = idx % nt, rr = idx / nt;
    xR[rr * kSolveRows + ii] = x[srows[ii] + static_cast<int64_t>(rr) * n];
  }
  __syncthreads();
  const double* Lt = L + sd.lptr[s] + w + t.r0;
  double* Pt = P + (pptr[s] + static_cast<int64_t>(t.tidx) * w) * nrhs;  // [rr*w + j]
  constexpr int CJ = NR <= 4 ? 4 : 1;  // columns j, j+8, … per warp pass
  for (int j0 = t.c0 + warp; j0 < t.c1; j0 += 8 * CJ) {
    double acc[CJ][NR];
    const int nc = min(CJ, (t.c1 - j0 + 7) / 8);
    warp_col_dots<NR, CJ>(acc, Lt + static_cast<int64_t>(j0) * rows, 8 * static_cast<int64_t>(rows),
                          nc, xR, kSolveRows, nt, lane);
#pragma unroll
    for (int c = 0; c < CJ; ++c)
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        double v = acc[c][rr];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && rr < nrhs && c < nc) Pt[rr * w + j0 + 8 * c] = v;
      }
  }
}

// ---- backward: diagonal triangle  L_JJᵀ x_J = y_J − Σ_tiles t ---------------
template <int NR>
__global__ void __launch_bounds__(256) k_bsolve_diag(const int32_t* __restrict__ sns, SymDev sd,
                                                     const double* __restrict__ L,
                                                     double* __restrict__ x, int nrhs,
                                                     const double* __restrict__ P,
                                                     const int64_t* __restrict__ pptr,
                                                     const double* __restrict__ rdiag) {
  extern __shared__ double sm[];
  __shared__ double rdl[64];  // 1/L_jj of the current chunk
  const int s = sns[blockIdx.x];
  const int f0 = sd.sn_first[s];
  const int w = sd.sn_first[s + 1] - f0;
  const int rows = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]);
  const int r = rows - w;
  const int n = sd.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Ls = L + sd.lptr[s];
  double* bJ = sm;           // [rr*w + a]
  double* Lb = sm + w * NR;  // [j*65 + i]
  if (r <= kSolveFuseRows) {  // b_J = y_J − L_RJᵀ x_R here (no off-diagonal tiles)
    double* xR = Lb + 64 * 65;  // [rr*r + i]
    const int32_t* srows = sd.sn_rows + sd.sn_rptr[s] + w;
    for (int idx = tid; idx < r * nrhs; idx += blockDim.x) {
      const int i = idx % r, rr = idx / r;
      xR[rr * r + i] = x[srows[i] + static_cast<int64_t>(rr) * n];
    }
    __syncthreads();
    constexpr int CJ = NR <= 4 ? 4 : 1;  // columns j, j+8, … per warp pass
    for (int j0 = warp; j0 < w; j0 += 8 * CJ) {
      double acc[CJ][NR];
      const int nc = min(CJ, (w - j0 + 7) / 8);
      warp_col_dots<NR, CJ>(acc, Ls + w + static_cast<int64_t>(j0) * rows,
                            8 * static_cast<int64_t>(rows), nc, xR, r, r, lane);
#pragma unroll
      for (int c = 0; c < CJ; ++c)
#pragma unroll
        for (int rr = 0; rr < NR; ++rr) {
          double v = acc[c][rr];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          const int j = j0 + 8 * c;
          if (lane == 0 && rr < nrhs && c < nc)
            bJ[rr * w + j] = x[f0 + j + static_cast<int64_t>(rr) * n] - v;
        }
    }
  } else {
    const int ntiles = (r + kSolveRows - 1) / kSolveRows;
    const double* Ps = P + pptr[s] * nrhs;
    for (int idx = tid; idx < w * nrhs; idx += blockDim.x) {
      const int a = idx % w, rr = idx / w;
      double v = x[f0 + a + static_cast<int64_t>(rr) * n];
      for (int t = 0; t < ntiles; ++t) v -= Ps[(static_cast<int64_t>(t) * w) * nrhs + rr * w + a];
      bJ[rr * w + a] = v;
    }
  }
  __syncthreads();
  const int nch = (w + 63) / 64;
  for (int ck = nch - 1; ck >= 0; --ck) {
    const int c0 = ck * 64, wk = min(64, w - c0);
    // contributions of the already-solved rows below the chunk inside the triangle
    for (int j = warp; j < wk; j += 8) {
      const double* col = Ls + static_cast<int64_t>(c0 + j) * rows;
      double acc[NR];
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) acc[rr] = 0.0;
      int i = c0 + wk + lane;
      for (; i + 96 < w; i += 128) {  // 4 independent loads in flight per lane
        const double l0 = col[i], l1 = col[i + 32], l2 = col[i + 64], l3 = col[i + 96];
#pragma unroll
        for (int rr = 0; rr < NR; ++rr)
          acc[rr] += l0 * bJ[rr * w + i] + l1 * bJ[rr * w + i + 32] +
                     l2 * bJ[rr * w + i + 64] + l3 * bJ[rr * w + i + 96];
      }
      for (; i < w; i += 32) {
        const double l = col[i];
#pragma unroll
        for (int rr = 0; rr < NR; ++rr) acc[rr] += l * bJ[rr * w + i];
      }
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        double v = acc[rr];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && rr < nrhs) bJ[rr * w + c0 + j] -= v;
      }
    }
    for (int idx = tid; idx < wk * wk; idx += blockDim.x) {
      const int i = idx % wk, j = idx / wk;
      if (i >= j) cpasync8(&Lb[j * 65 + i], Ls + (c0 + i) + static_cast<int64_t>(c0 + j) * rows);
    }
    if (tid < wk) cpasync8(&rdl[tid], rdiag + f0 + c0 + tid);
    cpasync_wait_all();
    __syncthreads();
    if (warp == 0) {
      double v0[NR], v1[NR];
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        v0[rr] = (rr < nrhs && lane < wk) ? bJ[rr * w + c0 + lane] : 0.0;
        v1[rr] = (rr < nrhs && lane + 32 < wk) ? bJ[rr * w + c0 + 32 + lane] : 0.0;
      }
      for (int j = wk - 1; j >= 0; --j) {
        const double rjj = rdl[j];  // 1/L_jj, from the factorization
        // (Lᵀ)_{i,j} = L_{j,i}, stored at Lb[i*65 + j] for i < j
        const double l0 = (lane < j) ? Lb[lane * 65 + j] : 0.0;
        const double l1 = (lane + 32 < j) ? Lb[(lane + 32) * 65 + j] : 0.0;
#pragma unroll
        for (int rr = 0; rr < NR; ++rr) {
          const double src = j < 32 ? v0[rr] : v1[rr];
          const double xj = __shfl_sync(0xffffffffu, src, j & 31) * rjj;
          if (lane == (j & 31)) {
            if (j < 32) v0[rr] = xj; else v1[rr] = xj;
          }
          v0[rr] -= l0 * xj;
          v1[rr] -= l1 * xj;
        }
      }
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        if (rr >= nrhs) break;
        if (lane < wk) bJ[rr * w + c0 + lane] = v0[rr];
        if (lane + 32 < wk) bJ[rr * w + c0 + 32 + lane] = v1[rr];
      }
    }
    __syncthreads();
  }
  for (int idx = tid; idx < w * nrhs; idx += blockDim.x) {
    const int a = idx % w, rr = idx / w;
    x[f0 + a + static_cast<int64_t>(rr) * n] = bJ[rr * w + a];
  }
}

}  // namespace gmrf
