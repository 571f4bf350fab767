// Split-K for the batched GEMM tiles: a tile whose K exceeds a threshold is
// replaced by K-slices that write partial 64×64 tiles to a scratch buffer, and
// a reduction task sums the partials in slice order (deterministic) into the
// destination with the original alpha/beta. Top-of-tree tiles of the
// factorization (K = supernode width) and of the selected inversion (K = rows
// below the chunk) otherwise leave one CTA streaming thousands of K steps.
#pragma once

#include <vector>

#include "kernels.cuh"

namespace gmrf {

constexpr int kSplitKMin = 512;    // split tiles with K above this
constexpr int kSplitKSlice = 256;  // K per slice

__global__ void __launch_bounds__(256) k_reduce_parts(const ReduceTask* __restrict__ tasks,
                                                      const double* __restrict__ parts) {
  const ReduceTask& t = tasks[blockIdx.x];
  const double* p0 = parts + t.part0 * (kTile * kTile);
  for (int idx = threadIdx.x; idx < t.m * t.n; idx += blockDim.x) {
    const int i = idx % t.m, j = idx / t.m;
    double s = 0.0;
    for (int q = 0; q < t.nparts; ++q) s += p0[static_cast<int64_t>(q) * kTile * kTile + i + j * kTile];
    double* c = t.c + i + static_cast<int64_t>(j) * t.ldc;
    *c = t.beta == 0.0 ? t.alpha * s : t.beta * *c + t.alpha * s;
  }
}

// Number of partial tiles split_k_level would create for a task list.
inline int64_t split_k_parts(const std::vector<GemmTask>& in) {
  int64_t n = 0;
  for (const GemmTask& g : in)
    if (g.k[0] + g.k[1] > kSplitKMin)
      for (int seg = 0; seg < 2; ++seg) n += (g.k[seg] + kSplitKSlice - 1) / kSplitKSlice;
  return n;
}

// Host: rewrites one level's task list. Partial c pointers are set relative to
// `scratch` (partial index × kTile²); returns the number of partial tiles used.
inline int64_t split_k_level(const std::vector<GemmTask>& in, std::vector<GemmTask>& out,
                             std::vector<ReduceTask>& red, double* scratch) {
  int64_t nparts = 0;
  for (const GemmTask& g : in) {
    const int K = g.k[0] + g.k[1];
    if (K <= kSplitKMin) {
      out.push_back(g);
      continue;
    }
    ReduceTask r{g.c, g.ldc, g.m, g.n, 0, nparts, g.alpha, g.beta};
    for (int seg = 0; seg < 2; ++seg) {
      const bool ta = (g.flags >> (2 * seg)) & 1, tb = (g.flags >> (2 * seg + 1)) & 1;
      for (int k0 = 0; k0 < g.k[seg]; k0 += kSplitKSlice) {
        GemmTask h{};
        h.c = scratch + (nparts + r.nparts) * static_cast<int64_t>(kTile * kTile);
        h.ldc = kTile;
        h.m = g.m;
        h.n = g.n;
        h.a[0] = ta ? g.a[seg] + k0 : g.a[seg] + static_cast<int64_t>(k0) * g.lda[seg];
        h.b[0] = tb ? g.b[seg] + static_cast<int64_t>(k0) * g.ldb[seg] : g.b[seg] + k0;
        h.lda[0] = g.lda[seg];
        h.ldb[0] = g.ldb[seg];
        h.k[0] = std::min(kSplitKSlice, g.k[seg] - k0);
        h.flags = (ta ? 1 : 0) | (tb ? 2 : 0);
        h.alpha = 1.0;
        h.beta = 0.0;
        out.push_back(h);
        ++r.nparts;
      }
    }
    nparts += r.nparts;
    red.push_back(r);
  }
  return nparts;
}

}  // namespace gmrf
