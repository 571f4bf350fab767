// Triangle part of the supernodal solves for WIDE supernodes (w > kWideW).
//
// The narrow-supernode kernels (solve.cuh) walk a supernode's w×w triangle
// with ONE CTA, 64 columns at a time; at the top of the tree (w ≈ 2000 for
// the 10⁶-unknown space-time case) that is a serial chain of 32 chunk steps,
// each paying a full memory round trip. Here every 64-row block b of the
// triangle gets its own CTA:
//   forward  — block b waits for blocks m = 0..b-1 IN ORDER, subtracts
//              L[b,m]·y_m, solves its 64×64 diagonal block, publishes y_b;
//   backward — block b waits for blocks m = nb-1..b+1 IN ORDER, subtracts
//              L[m,b]ᵀ·x_m, solves with L_bbᵀ, publishes x_b.
// The L tiles do not depend on the exchange, so each CTA prefetches them with
// cp.async (double buffered) while it waits; the dependent chain per block is
// one L2 round trip for the polled block values + a 64×64 GEMV + the 64-step
// warp solve. The update order of every entry is fixed (m order, 4 fixed partial sums), so
// results are bit-identical from run to run. All CTAs of a launch are
// co-resident (cooperative launch), and a CTA only waits on CTAs with a lower
// blockIdx (tasks are ordered by dependency), so the spin-waits cannot deadlock.
#pragma once

#include "kernels.cuh"
#include "panel.cuh"
#include "solve_tile.hpp"

namespace gmrf {

constexpr int kWideLd = 65;  // padded tile leading dimension (conflict-free)

template <int NR>
constexpr int wide_smem_bytes() {
  return (3 * 64 * kWideLd + 6 * 64 * NR + 64) * static_cast<int>(sizeof(double));
}

// Block exchange without flags: each solved 64-row block is published into its
// own slot of XW (64·nrhs doubles, reset to the all-ones NaN pattern before the
// sweep), and a consumer polls the values it needs until none is the sentinel.
// The value is its own ready flag, so there is no fence + flag store on the
// producer and no flag round trip before the data load on the consumer.
constexpr unsigned long long kWideSentinel = ~0ull;
__device__ __forceinline__ void wide_publish(double* slot, double v) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  if (b == kWideSentinel) b = 0x7ff8000000000000ull;  // a NaN result must not read as "not ready"
  __stcg(reinterpret_cast<unsigned long long*>(slot), b);
}
__device__ __forceinline__ double wide_poll(const double* slot) {
  const volatile unsigned long long* p = reinterpret_cast<const volatile unsigned long long*>(slot);
  unsigned long long b = *p;
  while (b == kWideSentinel) {
    __nanosleep(20);
    b = *p;
  }
  return __longlong_as_double(static_cast<long long>(b));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Children assembly for the wide supernodes of a level: y_J += children's
// update vectors, Uv_s (R part) = Σ children (same order as k_fsolve_diag).
template <int NR>
__global__ void __launch_bounds__(256) k_fsolve_wide_prep(const int32_t* __restrict__ sns,
                                                          SymDev sd, double* __restrict__ y,
                                                          int nrhs, double* __restrict__ Uv,
                                                          const int64_t* __restrict__ uvptr) {
  const int s = sns[blockIdx.x];
  const int f0 = sd.sn_first[s];
  const int w = sd.sn_first[s + 1] - f0;
  const int r = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]) - w;
  const int n = sd.n, tid = threadIdx.x;
  double* uS = Uv + uvptr[s] * nrhs;
  for (int idx = tid; idx < r * nrhs; idx += blockDim.x) uS[idx] = 0.0;
  __syncthreads();
  for (int q = sd.ch_ptr[s]; q < sd.ch_ptr[s + 1]; ++q) {
    const int c = sd.ch_list[q];
    const int wc = sd.sn_first[c + 1] - sd.sn_first[c];
    const int rc = static_cast<int>(sd.sn_rptr[c + 1] - sd.sn_rptr[c]) - wc;
    const int32_t* rel = sd.relmap + sd.sn_rptr[c] + wc;
    const double* uc = Uv + uvptr[c] * nrhs;
    child_scatter<4>(rel, uc, rc, nrhs, [&](int a, int rr) {
      return a < w ? y + f0 + a + static_cast<int64_t>(rr) * n : uS + (a - w) + rr * r;
    });
    __syncthreads();
  }
}

// stage the lower triangle of the 64×64 diagonal block b and its pivots
__device__ __forceinline__ void wide_stage_diag(double* Lb, double* rdl, const double* Ls,
                                                int rows, int i0, int nbr, const double* rdiag) {
  for (int idx = threadIdx.x; idx < nbr * nbr; idx += blockDim.x) {
    const int i = idx % nbr, j = idx / nbr;
    if (i >= j) cpasync8(&Lb[j * kWideLd + i], Ls + (i0 + i) + static_cast<int64_t>(i0 + j) * rows);
  }
  if (static_cast<int>(threadIdx.x) < nbr) cpasync8(&rdl[threadIdx.x], rdiag + threadIdx.x);
}

// stage the inverted diagonal block (k_tri_inv64 output, 64×64 slot, only nbr × nbr written)
__device__ __forceinline__ void wide_stage_inv(double* Lb, const double* Wb, int nbr) {
  for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x) {
    const int i = idx & 63, j = idx >> 6;
    if (i < nbr && j < nbr) cpasync8(&Lb[j * kWideLd + i], Wb + i + j * 64);
    else Lb[j * kWideLd + i] = 0.0;
  }
}

// stage the tile L[r0 .. r0+nr) × [c0 .. c0+nc) (column-major, zero padded to 64×64)
__device__ __forceinline__ void wide_stage_tile(double* T, const double* Ls, int rows, int r0,
                                                int nr, int c0, int nc) {
  for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x) {
    const int i = idx & 63, j = idx >> 6;
    if (i < nr && j < nc)
      cpasync8(&T[j * kWideLd + i], Ls + (r0 + i) + static_cast<int64_t>(c0 + j) * rows);
    else
      T[j * kWideLd + i] = 0.0;
  }
}

// ---- forward -----------------------------------------------------------------
template <int NR>
__global__ void __launch_bounds__(256) k_fsolve_wide(const WideBlock* __restrict__ tasks,
                                                     SymDev sd, const double* __restrict__ L,
                                                     double* __restrict__ y, int nrhs,
                                                     const double* __restrict__ rdiag,
                                                     double* __restrict__ xw,
                                                     const double* __restrict__ winv) {
  extern __shared__ double sm[];
  double* Lb = sm;                      // diagonal block (or its inverse), [j*65 + i]
  double* T0 = Lb + 64 * kWideLd;       // L[b, m] tiles, double buffered
  double* acc = T0 + 2 * 64 * kWideLd;  // [rr*64 + i]
  double* ym = acc + 64 * NR;           // [rr*64 + j]
  double* red = ym + 64 * NR;           // [(q*NR + rr)*64 + i]
  double* rdl = red + 4 * 64 * NR;
  const WideBlock t = tasks[blockIdx.x];
  const int s = t.sn;
  const int f0 = sd.sn_first[s];
  const int w = sd.sn_first[s + 1] - f0;
  const int rows = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]);
  const int n = sd.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Ls = L + sd.lptr[s];
  const int i0 = t.b * 64, nbr = min(64, w - i0);
  if (winv) wide_stage_inv(Lb, winv + static_cast<int64_t>(t.flag0 + t.b) * 64 * 64, nbr);
  else wide_stage_diag(Lb, rdl, Ls, rows, i0, nbr, rdiag + f0 + i0);
  cp_commit();
  if (t.b > 0) wide_stage_tile(T0, Ls, rows, i0, nbr, 0, 64);
  cp_commit();
  for (int idx = tid; idx < 64 * nrhs; idx += blockDim.x) {
    const int i = idx & 63, rr = idx >> 6;
    acc[rr * 64 + i] = i < nbr ? y[f0 + i0 + i + static_cast<int64_t>(rr) * n] : 0.0;
  }
  const int i = tid & 63, q = tid >> 6;  // row i, column quarter q
  for (int m = 0; m < t.b; ++m) {
    double* Tm = T0 + (m & 1) * 64 * kWideLd;
    if (m + 1 < t.b)
      wide_stage_tile(T0 + ((m + 1) & 1) * 64 * kWideLd, Ls, rows, i0, nbr, (m + 1) * 64, 64);
    cp_commit();
    {
      const double* slot = xw + static_cast<int64_t>(t.flag0 + m) * 64 * nrhs;
      for (int idx = tid; idx < 64 * nrhs; idx += blockDim.x) ym[idx] = wide_poll(slot + idx);
    }
    cp_wait<1>();  // tile m (and the diagonal block) landed
    __syncthreads();
    double part[NR];
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) part[rr] = 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double l = Tm[(q * 16 + u) * kWideLd + i];
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) part[rr] += l * ym[rr * 64 + q * 16 + u];
    }
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) red[(q * NR + rr) * 64 + i] = part[rr];
    __syncthreads();
    if (tid < nbr) {
#pragma unroll
      for (int rr = 0; rr < NR; ++rr)
        if (rr < nrhs)
          acc[rr * 64 + tid] -= (red[rr * 64 + tid] + red[(NR + rr) * 64 + tid]) +
                                (red[(2 * NR + rr) * 64 + tid] + red[(3 * NR + rr) * 64 + tid]);
    }
  }
  cp_wait<0>();
  __syncthreads();
  if (winv) {
    // y_b = L_bb⁻¹ acc: one 64×64 GEMV on all threads (column quarters, fixed sum order)
    double part[NR];
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) part[rr] = 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double l = Lb[(q * 16 + u) * kWideLd + i];
#pragma unroll
      for (int rr = 0; rr < NR; ++rr)
        if (rr < nrhs) part[rr] += l * acc[rr * 64 + q * 16 + u];
    }
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) red[(q * NR + rr) * 64 + i] = part[rr];
    __syncthreads();
    if (tid < nbr) {
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        if (rr >= nrhs) break;
        const double v = (red[rr * 64 + tid] + red[(NR + rr) * 64 + tid]) +
                         (red[(2 * NR + rr) * 64 + tid] + red[(3 * NR + rr) * 64 + tid]);
        if (t.b + 1 < t.nb)
          wide_publish(xw + static_cast<int64_t>(t.flag0 + t.b) * 64 * nrhs + rr * 64 + tid, v);
        y[f0 + i0 + tid + static_cast<int64_t>(rr) * n] = v;
      }
    }
  } else if (warp == 0) {
    double v0[NR], v1[NR];
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {
      v0[rr] = (rr < nrhs && lane < nbr) ? acc[rr * 64 + lane] : 0.0;
      v1[rr] = (rr < nrhs && lane + 32 < nbr) ? acc[rr * 64 + 32 + lane] : 0.0;
    }
    for (int j = 0; j < nbr; ++j) {
      const double rjj = rdl[j];
      const double l0 = (lane > j && lane < nbr) ? Lb[j * kWideLd + lane] : 0.0;
      const double l1 = (lane + 32 > j && lane + 32 < nbr) ? Lb[j * kWideLd + lane + 32] : 0.0;
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
      double* slot = xw + static_cast<int64_t>(t.flag0 + t.b) * 64 * nrhs + rr * 64;
      if (t.b + 1 < t.nb) {  // later blocks of this supernode wait on these values
        if (lane < nbr) wide_publish(slot + lane, v0[rr]);
        if (lane + 32 < nbr) wide_publish(slot + 32 + lane, v1[rr]);
      }
      if (lane < nbr) y[f0 + i0 + lane + static_cast<int64_t>(rr) * n] = v0[rr];
      if (lane + 32 < nbr) y[f0 + i0 + 32 + lane + static_cast<int64_t>(rr) * n] = v1[rr];
    }
  }
}

// ---- backward: L_JJᵀ x_J = y_J − Σ_tiles P (row-tile partials of L_RJᵀ x_R) ----
template <int NR>
__global__ void __launch_bounds__(256) k_bsolve_wide(const WideBlock* __restrict__ tasks,
                                                     SymDev sd, const double* __restrict__ L,
                                                     double* __restrict__ x, int nrhs,
                                                     const double* __restrict__ P,
                                                     const int64_t* __restrict__ pptr,
                                                     const double* __restrict__ rdiag,
                                                     double* __restrict__ xw,
                                                     const double* __restrict__ winv) {
  extern __shared__ double sm[];
  double* Lb = sm;
  double* T0 = Lb + 64 * kWideLd;       // L[m, b] tiles, double buffered
  double* acc = T0 + 2 * 64 * kWideLd;  // [rr*64 + j]
  double* xm = acc + 64 * NR;           // [rr*64 + i]
  double* red = xm + 64 * NR;           // [(q*NR + rr)*64 + j]
  double* rdl = red + 4 * 64 * NR;
  const WideBlock t = tasks[blockIdx.x];
  const int s = t.sn;
  const int f0 = sd.sn_first[s];
  const int w = sd.sn_first[s + 1] - f0;
  const int rows = static_cast<int>(sd.sn_rptr[s + 1] - sd.sn_rptr[s]);
  const int r = rows - w;
  const int n = sd.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Ls = L + sd.lptr[s];
  const int i0 = t.b * 64, nbr = min(64, w - i0);
  if (winv) wide_stage_inv(Lb, winv + static_cast<int64_t>(t.flag0 + t.b) * 64 * 64, nbr);
  else wide_stage_diag(Lb, rdl, Ls, rows, i0, nbr, rdiag + f0 + i0);
  cp_commit();
  const int mlast = t.nb - 1;
  if (mlast > t.b) wide_stage_tile(T0, Ls, rows, mlast * 64, w - mlast * 64, i0, nbr);
  cp_commit();
  {
    const int ntiles = (r + kSolveRows - 1) / kSolveRows;
    const double* Ps = P + pptr[s] * nrhs;
    for (int idx = tid; idx < 64 * nrhs; idx += blockDim.x) {
      const int a = idx & 63, rr = idx >> 6;
      double v = 0.0;
      if (a < nbr) {
        v = x[f0 + i0 + a + static_cast<int64_t>(rr) * n];
        for (int tt = 0; tt < ntiles; ++tt)
          v -= Ps[(static_cast<int64_t>(tt) * w) * nrhs + rr * w + i0 + a];
      }
      acc[rr * 64 + a] = v;
    }
  }
  const int j = tid & 63, q = tid >> 6;  // column j of block b, row quarter q
  for (int m = mlast, it = 0; m > t.b; --m, ++it) {
    double* Tm = T0 + (it & 1) * 64 * kWideLd;
    if (m - 1 > t.b)
      wide_stage_tile(T0 + ((it + 1) & 1) * 64 * kWideLd, Ls, rows, (m - 1) * 64, 64, i0, nbr);
    cp_commit();
    const int nm = min(64, w - m * 64);
    {
      const double* slot = xw + static_cast<int64_t>(t.flag0 + m) * 64 * nrhs;
      for (int idx = tid; idx < 64 * nrhs; idx += blockDim.x)
        xm[idx] = (idx & 63) < nm ? wide_poll(slot + idx) : 0.0;
    }
    cp_wait<1>();
    __syncthreads();
    double part[NR];
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) part[rr] = 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double l = Tm[j * kWideLd + q * 16 + u];
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) part[rr] += l * xm[rr * 64 + q * 16 + u];
    }
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) red[(q * NR + rr) * 64 + j] = part[rr];
    __syncthreads();
    if (tid < nbr) {
#pragma unroll
      for (int rr = 0; rr < NR; ++rr)
        if (rr < nrhs)
          acc[rr * 64 + tid] -= (red[rr * 64 + tid] + red[(NR + rr) * 64 + tid]) +
                                (red[(2 * NR + rr) * 64 + tid] + red[(3 * NR + rr) * 64 + tid]);
    }
  }
  cp_wait<0>();
  __syncthreads();
  if (winv) {
    // x_b = L_bb⁻ᵀ acc: x_j = Σ_i W_ij acc_i (row quarters, fixed sum order)
    double part[NR];
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) part[rr] = 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double l = Lb[j * kWideLd + q * 16 + u];
#pragma unroll
      for (int rr = 0; rr < NR; ++rr)
        if (rr < nrhs) part[rr] += l * acc[rr * 64 + q * 16 + u];
    }
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) red[(q * NR + rr) * 64 + j] = part[rr];
    __syncthreads();
    if (tid < nbr) {
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        if (rr >= nrhs) break;
        const double v = (red[rr * 64 + tid] + red[(NR + rr) * 64 + tid]) +
                         (red[(2 * NR + rr) * 64 + tid] + red[(3 * NR + rr) * 64 + tid]);
        if (t.b > 0)
          wide_publish(xw + static_cast<int64_t>(t.flag0 + t.b) * 64 * nrhs + rr * 64 + tid, v);
        x[f0 + i0 + tid + static_cast<int64_t>(rr) * n] = v;
      }
    }
  } else if (warp == 0) {
    double v0[NR], v1[NR];
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {
      v0[rr] = (rr < nrhs && lane < nbr) ? acc[rr * 64 + lane] : 0.0;
      v1[rr] = (rr < nrhs && lane + 32 < nbr) ? acc[rr * 64 + 32 + lane] : 0.0;
    }
    for (int jj = nbr - 1; jj >= 0; --jj) {
      const double rjj = rdl[jj];
      const double l0 = (lane < jj) ? Lb[lane * kWideLd + jj] : 0.0;
      const double l1 = (lane + 32 < jj) ? Lb[(lane + 32) * kWideLd + jj] : 0.0;
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        const double src = jj < 32 ? v0[rr] : v1[rr];
        const double xj = __shfl_sync(0xffffffffu, src, jj & 31) * rjj;
        if (lane == (jj & 31)) {
          if (jj < 32) v0[rr] = xj; else v1[rr] = xj;
        }
        v0[rr] -= l0 * xj;
        v1[rr] -= l1 * xj;
      }
    }
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {
      if (rr >= nrhs) break;
      double* slot = xw + static_cast<int64_t>(t.flag0 + t.b) * 64 * nrhs + rr * 64;
      if (t.b > 0) {  // earlier blocks of this supernode wait on these values
        if (lane < nbr) wide_publish(slot + lane, v0[rr]);
        if (lane + 32 < nbr) wide_publish(slot + 32 + lane, v1[rr]);
      }
      if (lane < nbr) x[f0 + i0 + lane + static_cast<int64_t>(rr) * n] = v0[rr];
      if (lane + 32 < nbr) x[f0 + i0 + 32 + lane + static_cast<int64_t>(rr) * n] = v1[rr];
    }
  }
}

}  // namespace gmrf
