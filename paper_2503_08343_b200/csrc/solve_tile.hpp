// Work item of the rectangular-block solve kernels (solve.cuh).
#pragma once

#include <cstdint>

namespace gmrf {

constexpr int kSolveRows = 128;
constexpr int kSolveOffCols = 256;  // y_J columns staged per pass in k_fsolve_off

struct SolveTile {
  int32_t sn;
  int32_t r0;    // first row of the tile inside the supernode's R block
  int32_t tidx;  // tile index inside the supernode
};

}  // namespace gmrf
