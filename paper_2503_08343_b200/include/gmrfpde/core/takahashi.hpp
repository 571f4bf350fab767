// Drop-in replacement for the reference's gmrfpde/core/takahashi.hpp
// (/root/reference/proj/include/gmrfpde/core/takahashi.hpp): supernodal
// selected inversion on the B200 through the C-ABI. Same names and results
// (Σ on the pattern of L+Lᵀ in original indices; its diagonal).
#pragma once

#include <cstdint>
#include <vector>

#include "gmrfpde/core/cholesky.hpp"

namespace gmrfpde {

/// takahashi_selected_inverse (takahashi.hpp:19).
inline SparseMatrixCSC takahashi_selected_inverse(const CholeskyFactor& f) {
  const Index n = f.dim();
  Vector d(n);
  b200::check(gmrf_selinv_diag(f.device->h, d.data()));
  int64_t nnz = 0;
  b200::check(gmrf_selinv_pattern_nnz(f.device->h, &nnz));
  std::vector<int64_t> cp(n + 1);
  SparseMatrixCSC s(n, n);
  s.row_idx.resize(nnz);
  s.values.resize(nnz);
  b200::check(gmrf_selinv_pattern(f.device->h, cp.data(), s.row_idx.data(), s.values.data()));
  s.col_ptr.assign(cp.begin(), cp.end());
  return s;
}

/// takahashi_diagonal (takahashi.hpp:67): diag(Q⁻¹) without the host pattern.
inline Vector takahashi_diagonal(const CholeskyFactor& f) {
  Vector d(f.dim());
  b200::check(gmrf_selinv_diag(f.device->h, d.data()));
  return d;
}

}  // namespace gmrfpde
