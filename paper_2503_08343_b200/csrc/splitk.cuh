// Split-K for the batched GEMM tiles: a tile whose K exceeds a threshold, in a
// launch with too few tiles to fill the GPU, is replaced by K-slices that write
// partial 64×64 tiles to a scratch buffer, and
// a reduction task sums the partials in slice order (deterministic) into the
// destination with the original alpha/beta. Top-of-tree tiles of the
// factorization (K = supernode width) and of the selected inversion (K = rows
// below the chunk) otherwise leave one CTA streaming thousands of K steps.
#pragma once

#include <algorithm>
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

// K slices of one tile. A level that already launches enough tiles to keep
// every SM busy is not split (this also bounds the partial-tile scratch, which
// grows with tiles × slices); otherwise long-K tiles get just enough slices to
// fill ~kSplitWave CTAs. `level_tiles` counts the launch's tiles over ALL
// supernodes (every rank of a partitioned factor), so each tile is split the
// same way everywhere and the summation order does not depend on the partition.
constexpr int64_t kSplitWave = 148 * 4 * 2;
inline int split_slices(int K, int64_t level_tiles) {
  if (K <= kSplitKMin || level_tiles >= kSplitWave) return 1;
  const int64_t want = (kSplitWave + std::max<int64_t>(level_tiles, 1) - 1) /
                       std::max<int64_t>(level_tiles, 1);
  const int64_t most = (K + kSplitKSlice - 1) / kSplitKSlice;
  return static_cast<int>(std::min<int64_t>(most, std::max<int64_t>(2, want)));
}
// K per slice (a multiple of the GEMM's K stage)
inline int split_len(int K, int slices) {
  const int l = (K + slices - 1) / slices;
  return (l + 15) / 16 * 16;
}

// Number of partial tiles split_k_level would create for a task list.
inline int64_t split_k_parts(const std::vector<GemmTask>& in, int64_t level_tiles) {
  int64_t n = 0;
  for (const GemmTask& g : in) {
    const int K = g.k[0] + g.k[1];
    const int sl = split_slices(K, level_tiles);
    if (sl == 1) continue;
    const int len = split_len(K, sl);
    for (int seg = 0; seg < 2; ++seg) n += (g.k[seg] + len - 1) / len;
  }
  return n;
}

// Host: rewrites one level's task list. Partial c pointers are set relative to
// `scratch` (partial index × kTile²); returns the number of partial tiles used.
inline int64_t split_k_level(const std::vector<GemmTask>& in, std::vector<GemmTask>& out,
                             std::vector<ReduceTask>& red, double* scratch, int64_t level_tiles) {
  int64_t nparts = 0;
  for (const GemmTask& g : in) {
    const int K = g.k[0] + g.k[1];
    const int sl = split_slices(K, level_tiles);
    if (sl == 1) {
      out.push_back(g);
      continue;
    }
    const int len = split_len(K, sl);
    ReduceTask r{g.c, g.ldc, g.m, g.n, 0, nparts, g.alpha, g.beta};
    for (int seg = 0; seg < 2; ++seg) {
      const bool ta = (g.flags >> (2 * seg)) & 1, tb = (g.flags >> (2 * seg + 1)) & 1;
      for (int k0 = 0; k0 < g.k[seg]; k0 += len) {
        GemmTask h{};
        h.c = scratch + (nparts + r.nparts) * static_cast<int64_t>(kTile * kTile);
        h.ldc = kTile;
        h.m = g.m;
        h.n = g.n;
        h.a[0] = ta ? g.a[seg] + k0 : g.a[seg] + static_cast<int64_t>(k0) * g.lda[seg];
        h.b[0] = tb ? g.b[seg] + static_cast<int64_t>(k0) * g.ldb[seg] : g.b[seg] + k0;
        h.lda[0] = g.lda[seg];
        h.ldb[0] = g.ldb[seg];
        h.k[0] = std::min(len, g.k[seg] - k0);
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
