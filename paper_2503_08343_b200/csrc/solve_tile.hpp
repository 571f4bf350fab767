// Work item of the rectangular-block solve kernels (solve.cuh).
#pragma once

#include <cstdint>

namespace gmrf {

constexpr int kSolveRows = 128;
constexpr int kSolveOffCols = 256;  // y_J columns staged per pass in k_fsolve_off
constexpr int kSolveSplitCols = 64;
constexpr int kSolveFuseRows = 256;  // narrow supernodes with r ≤ this: no off-diagonal tiles  // wider supernodes split their row tiles by column blocks

struct SolveTile {
  int32_t sn;
  int32_t r0;      // first row of the tile inside the supernode's R block
  int32_t tidx;    // row-tile index inside the supernode
  int32_t c0, c1;  // column range [c0, c1) of L_RJ handled by this tile
  int32_t part;    // column block index, 0 .. nparts-1
  int32_t nparts;  // column blocks of this row tile (1: no split)
  int32_t pf;      // forward partials: first slot of this row tile (nparts > 1)
  int32_t ctr;     // forward partials: arrival counter of this row tile (nparts > 1)
};

}  // namespace gmrf
