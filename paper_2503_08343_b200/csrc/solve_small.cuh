// Triangular solves for SMALL supernodes (w <= 64, rows <= 128): one warp per
// supernode, no block barriers, no shared-memory staging of L.
//
// The lower tree levels hold tens of thousands of small supernodes (config 4:
// ~20k leaves of a few dozen columns). The one-CTA-per-supernode kernels of
// solve.cuh spend most of their time in __syncthreads-separated memory round
// trips on one warp's serial chain; here a warp owns a supernode and 8
// supernodes share a CTA, so ~50 chains per SM overlap their latencies and the
// level streams L at close to HBM speed.
//
//   forward  (cholesky.hpp:186-193, column-oriented): lane l owns front rows
//            a = l + 32k (k < 4). The front vector (y_J and the zero-started
//            update vector u_R) is assembled in the warp's shared slice with the
//            children's update vectors in child order, then ONE right-looking
//            sweep over the w columns: x_j = f_j / L_jj (× 1/L_jj from the
//            factorization), f_a -= L_aj x_j for every row a > j — the rows
//            below the triangle accumulate u_R = f_R - L_RJ x_J in the same pass.
//   backward (cholesky.hpp:194-201, dot-product form): lane l owns columns
//            j = l + 32k (k < 2). b_j = y_j - Σ_i L_{w+i,j} x_{R_i} (rows in
//            order), then the triangle right-looking on Lᵀ from the last column:
//            x_j = b_j / L_jj, b_k -= L_jk x_j for k < j.
// L is read straight from the panel (column-major): forward loads are
// coalesced across lanes; backward lanes walk their own columns, consecutive
// rows hitting the same sectors in L1. Each group of 4 columns (forward) or 8
// rows (backward) has all its loads in flight before its part of the chain.
// Every sum is taken in a fixed order (deterministic).
#pragma once

#include "kernels.cuh"

namespace gmrf {

constexpr int kSmallSolveW = 64;      // widest supernode handled here
constexpr int kSmallSolveRows = 128;  // most front rows handled here
constexpr int kSmallSolveWarps = 8;   // supernodes per CTA

template <int NR>
__global__ void __launch_bounds__(32 * kSmallSolveWarps, NR == 1 ? 3 : 2) k_fsolve_small(
    const int32_t* __restrict__ sns, int nsn, SymDev sd, const double* __restrict__ L,
    double* __restrict__ y, int nrhs, double* __restrict__ Uv, const int64_t* __restrict__ uvptr,
    const double* __restrict__ rdiag) {
  __shared__ double Fs[kSmallSolveWarps][NR][kSmallSolveRows];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int q = blockIdx.x * kSmallSolveWarps + wid;
  if (q >= nsn) return;
  const int s = sns[q];
  const int f0 = sd.sn_first[s];
  const int w = sd.sn_first[s + 1] - f0;
  const int rows = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]);
  const int r = rows - w;
  const int n = sd.n;
  const double* Ls = L + sd.lptr[s];
  double(*F)[kSmallSolveRows] = Fs[wid];
  for (int a = lane; a < kSmallSolveRows; a += 32)
#pragma unroll
    for (int rr = 0; rr < NR; ++rr)
      F[rr][a] = (a < w && rr < nrhs) ? y[f0 + a + static_cast<int64_t>(rr) * n] : 0.0;
  __syncwarp();
  for (int p = sd.ch_ptr[s]; p < sd.ch_ptr[s + 1]; ++p) {  // children in order
    const int c = sd.ch_list[p];
    const int wc = sd.sn_first[c + 1] - sd.sn_first[c];
    const int rc = static_cast<int>(sd.sn_rptr[c + 1] - sd.sn_rptr[c]) - wc;
    const int32_t* rel = sd.relmap + sd.sn_rptr[c] + wc;
    const double* uc = Uv + uvptr[c] * nrhs;
    for (int ia = lane; ia < rc; ia += 32) {
      const int a = rel[ia];
#pragma unroll
      for (int rr = 0; rr < NR; ++rr)
        if (rr < nrhs) F[rr][a] += uc[ia + rr * rc];
    }
    __syncwarp();
  }
  double v[4][NR];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) v[k][rr] = F[rr][lane + 32 * k];
  const double rd0 = lane < w ? rdiag[f0 + lane] : 0.0;
  const double rd1 = lane + 32 < w ? rdiag[f0 + 32 + lane] : 0.0;
  // column j of the panel, rows a = lane + 32k (0 beyond the front)
  auto ldcol = [&](int j, double (&lc)[4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int a = lane + 32 * k;
      lc[k] = (j < w && a > j && a < rows) ? __ldg(Ls + static_cast<int64_t>(j) * rows + a) : 0.0;
    }
  };
  for (int j0 = 0; j0 < w; j0 += 4) {
    double cur[4][4];  // the group's 4 columns, all loads in flight before the chain
#pragma unroll
    for (int u = 0; u < 4; ++u) ldcol(j0 + u, cur[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u;
      if (j >= w) break;
      const double rjj = __shfl_sync(0xffffffffu, j < 32 ? rd0 : rd1, j & 31);
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        const double src = j < 32 ? v[0][rr] : v[1][rr];
        const double xj = __shfl_sync(0xffffffffu, src, j & 31) * rjj;
        if (lane == (j & 31)) {
          if (j < 32) v[0][rr] = xj;
          else v[1][rr] = xj;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k][rr] -= cur[u][k] * xj;
      }
    }
  }
  double* uS = Uv + uvptr[s] * nrhs;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int a = lane + 32 * k;
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {
      if (rr >= nrhs) break;
      if (a < w) y[f0 + a + static_cast<int64_t>(rr) * n] = v[k][rr];
      else if (a < rows) uS[(a - w) + rr * r] = v[k][rr];
    }
  }
}

template <int NR>
__global__ void __launch_bounds__(32 * kSmallSolveWarps, NR == 1 ? 3 : 2) k_bsolve_small(
    const int32_t* __restrict__ sns, int nsn, SymDev sd, const double* __restrict__ L,
    double* __restrict__ x, int nrhs, const double* __restrict__ rdiag) {
  __shared__ double XRs[kSmallSolveWarps][NR][kSmallSolveRows];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int q = blockIdx.x * kSmallSolveWarps + wid;
  if (q >= nsn) return;
  const int s = sns[q];
  const int f0 = sd.sn_first[s];
  const int w = sd.sn_first[s + 1] - f0;
  const int rows = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]);
  const int r = rows - w;
  const int n = sd.n;
  const double* Ls = L + sd.lptr[s];
  double(*XR)[kSmallSolveRows] = XRs[wid];
  const int32_t* srows = sd.sn_rows + sd.sn_rptr[s] + w;
  for (int i = lane; i < r; i += 32) {
    const int64_t g = srows[i];
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) XR[rr][i] = rr < nrhs ? x[g + static_cast<int64_t>(rr) * n] : 0.0;
  }
  double b[2][NR];
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {
      const int j = lane + 32 * k;
      b[k][rr] = (j < w && rr < nrhs) ? x[f0 + j + static_cast<int64_t>(rr) * n] : 0.0;
    }
  const double rd0 = lane < w ? rdiag[f0 + lane] : 0.0;
  const double rd1 = lane + 32 < w ? rdiag[f0 + 32 + lane] : 0.0;
  __syncwarp();
  // entries L[i, j] of row i for the lane's columns j = lane + 32k (0 unless j < min(w, i))
  auto ldrow = [&](int i, double (&lr)[2]) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int j = lane + 32 * k;
      lr[k] = (i < rows && j < w && j < i) ? __ldg(Ls + static_cast<int64_t>(j) * rows + i) : 0.0;
    }
  };
  // rectangular part: b_J -= L_RJᵀ x_R, rows in order
  for (int i0 = 0; i0 < r; i0 += 8) {
    double cur[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) ldrow(w + i0 + u, cur[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u;
      if (i >= r) break;
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        const double xi = XR[rr][i];
#pragma unroll
        for (int k = 0; k < 2; ++k) b[k][rr] -= cur[u][k] * xi;
      }
    }
  }
  // triangle: from the last column up
  for (int j0 = w - 1; j0 >= 0; j0 -= 8) {
    double cur[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) ldrow(j0 - u >= 0 ? j0 - u : rows, cur[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 - u;
      if (j < 0) break;
      const double rjj = __shfl_sync(0xffffffffu, j < 32 ? rd0 : rd1, j & 31);
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        const double src = j < 32 ? b[0][rr] : b[1][rr];
        const double xj = __shfl_sync(0xffffffffu, src, j & 31) * rjj;
        if (lane == (j & 31)) {
          if (j < 32) b[0][rr] = xj;
          else b[1][rr] = xj;
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) b[k][rr] -= cur[u][k] * xj;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int j = lane + 32 * k;
#pragma unroll
    for (int rr = 0; rr < NR; ++rr)
      if (j < w && rr < nrhs) x[f0 + j + static_cast<int64_t>(rr) * n] = b[k][rr];
  }
}

}  // namespace gmrf
