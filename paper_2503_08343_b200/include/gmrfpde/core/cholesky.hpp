// Drop-in replacement for the reference's gmrfpde/core/cholesky.hpp
// (/root/reference/proj/include/gmrfpde/core/cholesky.hpp), backed by the
// B200 engine through the C-ABI (include/gmrf_b200.h).
//
// Put this directory BEFORE the reference include directory: every reference
// header that includes "gmrfpde/core/cholesky.hpp" (gmrf.hpp, takahashi.hpp,
// gauss_newton.hpp, spatiotemporal.hpp, the tests) then factors and solves on
// the GPU with unchanged source. Same names, signatures, argument meaning and
// exceptions as the reference (cholesky.hpp:16-229); the carrier types
// (SparseMatrixCSC, Index, exceptions) and amd_order still come from the
// reference headers.
//
// Differences, all documented in INTEGRATION.md:
//  * cholesky_factor(q) orders with nested dissection (METIS), not AMD;
//  * CholeskyFactor::L is materialised on the host eagerly (reference layout,
//    exact pattern) only when n <= GMRF_HOST_L_MAX (default 200000); larger
//    factors stay device-resident and L is left empty.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "gmrf_b200.h"
#include "gmrfpde/core/amd.hpp"
#include "gmrfpde/core/sparse.hpp"
#include "gmrfpde/core/types.hpp"

namespace gmrfpde {

namespace b200 {

[[noreturn]] inline void raise(int rc, int32_t bad = -1) {
  std::string msg = gmrf_last_error();
  switch (rc) {
    case GMRF_ERR_NOT_SPD: throw NotPositiveDefiniteError(msg, bad);
    case GMRF_ERR_DIMENSION: throw DimensionError(msg);
    case GMRF_ERR_STRUCTURAL: throw StructuralError(msg);
    case GMRF_ERR_CONTRACT: throw ContractError(msg);
    default: throw NumericalError(msg);
  }
}
inline void check(int rc) {
  if (rc != GMRF_OK) raise(rc);
}

inline std::vector<int64_t> colptr64(const SparseMatrixCSC& q) {
  return std::vector<int64_t>(q.col_ptr.begin(), q.col_ptr.end());
}

// Device factors of a symbolic are pooled: a CholeskyFactor that goes out of
// scope hands its device storage (panels, plans, captured CUDA graph) back to
// its SymbolicFactor, and the next cholesky_refactor of that symbolic reuses it
// (gauss_newton.hpp:139-140 refactors once per iteration on one symbolic).
struct SymbolicHandle {
  gmrf_symbolic_t* h = nullptr;
  std::vector<int64_t> cp;
  std::vector<Index> ri;
  std::mutex mu;
  std::vector<gmrf_factor_t*> pool;
  ~SymbolicHandle() {
    for (gmrf_factor_t* f : pool) gmrf_factor_free(f);
    if (h) gmrf_symbolic_free(h);
  }
  gmrf_factor_t* acquire() {
    {
      std::lock_guard<std::mutex> g(mu);
      if (!pool.empty()) {
        gmrf_factor_t* f = pool.back();
        pool.pop_back();
        return f;
      }
    }
    gmrf_factor_t* f = nullptr;
    const int rc = gmrf_factor_create(h, &f);
    if (rc != GMRF_OK) raise(rc);
    return f;
  }
  void release(gmrf_factor_t* f) {
    std::lock_guard<std::mutex> g(mu);
    pool.push_back(f);
  }
  // the reference re-permutes q on every refactor (cholesky.hpp:117); here the
  // values are consumed in the analysed CSC order, so the pattern must match
  bool same_pattern(const SparseMatrixCSC& q) const {
    if (static_cast<int64_t>(q.col_ptr.size()) != static_cast<int64_t>(cp.size()) ||
        q.row_idx.size() != ri.size() || q.values.size() != ri.size())
      return false;
    for (std::size_t j = 0; j < cp.size(); ++j)
      if (static_cast<int64_t>(q.col_ptr[j]) != cp[j]) return false;
    return ri.empty() || std::memcmp(q.row_idx.data(), ri.data(), ri.size() * sizeof(Index)) == 0;
  }
};
struct FactorHandle {
  gmrf_factor_t* h = nullptr;
  std::shared_ptr<SymbolicHandle> sym;
  std::shared_ptr<void> owner;  // set: h is a borrowed view kept alive by owner
  ~FactorHandle() {
    if (!h || owner) return;
    if (sym) sym->release(h);
    else gmrf_factor_free(h);
  }
};

inline int64_t host_l_max() {
  const char* e = std::getenv("GMRF_HOST_L_MAX");
  return e ? std::atoll(e) : 200000;
}

}  // namespace b200

/// Symbolic phase (cholesky.hpp:16-23): same fields, plus the device handle.
struct SymbolicFactor {
  std::vector<Index> perm;      // new -> old
  std::vector<Index> perm_inv;  // old -> new
  std::vector<Index> parent;    // elimination tree over permuted indices
  std::vector<Index> col_ptr;   // column layout of L (including diagonal)
  Index n = 0;
  Index nnz_L = 0;
  std::shared_ptr<b200::SymbolicHandle> handle;
};

/// symbolic_analyze (cholesky.hpp:68). Bit-exact parent/col_ptr for the same perm.
inline SymbolicFactor symbolic_analyze(const SparseMatrixCSC& q, const std::vector<Index>& perm) {
  if (q.nrows != q.ncols) throw DimensionError("symbolic_analyze: matrix not square");
  auto h = std::make_shared<b200::SymbolicHandle>();
  h->cp = b200::colptr64(q);
  h->ri = q.row_idx;
  const Index n = q.nrows;
  if (static_cast<Index>(perm.size()) != n)
    throw DimensionError("symbolic_analyze: permutation length mismatch");
  b200::check(gmrf_symbolic_analyze(n, h->cp.data(), h->ri.data(), perm.data(), &h->h));
  SymbolicFactor s;
  s.n = n;
  s.perm.resize(n);
  s.parent.resize(n);
  std::vector<int64_t> cpl(n + 1);
  b200::check(gmrf_symbolic_export(h->h, s.perm.data(), s.parent.data(), cpl.data()));
  s.perm_inv = invert_permutation(s.perm);
  s.col_ptr.assign(cpl.begin(), cpl.end());
  s.nnz_L = static_cast<Index>(cpl[n]);
  s.handle = std::move(h);
  return s;
}

/// P Q Pᵀ = L Lᵀ (cholesky.hpp:92-109); the numeric factor lives on the GPU.
struct CholeskyFactor {
  SparseMatrixCSC L;            // reference layout, filled when n <= GMRF_HOST_L_MAX
  std::vector<Index> perm;      // new -> old
  std::vector<Index> perm_inv;  // old -> new
  std::shared_ptr<b200::FactorHandle> device;

  Index dim() const { return static_cast<Index>(perm.size()); }

  Vector apply_perm(const Vector& x) const {
    Vector y(x.size());
    for (std::size_t i = 0; i < x.size(); ++i) y[i] = x[perm[i]];
    return y;
  }
  Vector apply_perm_inv(const Vector& x) const {
    Vector y(x.size());
    for (std::size_t i = 0; i < x.size(); ++i) y[perm[i]] = x[i];
    return y;
  }
};

/// cholesky_refactor (cholesky.hpp:113): numeric factorization on the GPU.
inline CholeskyFactor cholesky_refactor(const SymbolicFactor& s, const SparseMatrixCSC& q) {
  const Index n = s.n;
  if (q.nrows != n || q.ncols != n) throw DimensionError("cholesky_refactor: dimension mismatch");
  if (!s.handle->same_pattern(q))
    throw StructuralError("cholesky_refactor: sparsity pattern differs from the analysed one");
  auto fh = std::make_shared<b200::FactorHandle>();
  fh->sym = s.handle;
  fh->h = s.handle->acquire();
  int32_t bad = -1;
  const int rc = gmrf_factor_numeric(fh->h, q.values.data(), &bad);
  if (rc != GMRF_OK) b200::raise(rc, bad);
  CholeskyFactor f;
  f.perm = s.perm;
  f.perm_inv = s.perm_inv;
  f.device = fh;
  f.L.nrows = f.L.ncols = n;
  if (n <= b200::host_l_max()) {
    std::vector<int64_t> cp(n + 1);
    f.L.row_idx.resize(s.nnz_L);
    f.L.values.resize(s.nnz_L);
    b200::check(gmrf_factor_l(fh->h, cp.data(), f.L.row_idx.data(), f.L.values.data(), nullptr));
    f.L.col_ptr.assign(cp.begin(), cp.end());
  }
  return f;
}

namespace b200 {
/// A CholeskyFactor over a device factor that another object owns (an update
/// system, gmrfpde/b200/update_system.hpp): perm from its symbolic, the host L
/// as cholesky_refactor materialises it.
inline CholeskyFactor wrap_factor(gmrf_factor_t* fh, const gmrf_symbolic_t* sh,
                                  std::shared_ptr<void> owner) {
  gmrf_symbolic_info_t info{};
  check(gmrf_symbolic_info(sh, &info));
  const Index n = info.n;
  CholeskyFactor f;
  f.perm.resize(n);
  check(gmrf_symbolic_export(sh, f.perm.data(), nullptr, nullptr));
  f.perm_inv = invert_permutation(f.perm);
  auto h = std::make_shared<FactorHandle>();
  h->h = fh;
  h->owner = std::move(owner);
  f.device = h;
  f.L.nrows = f.L.ncols = n;
  if (n <= host_l_max()) {
    std::vector<int64_t> cp(n + 1);
    f.L.row_idx.resize(info.nnz_l);
    f.L.values.resize(info.nnz_l);
    check(gmrf_factor_l(fh, cp.data(), f.L.row_idx.data(), f.L.values.data(), nullptr));
    f.L.col_ptr.assign(cp.begin(), cp.end());
  }
  return f;
}
}  // namespace b200

/// cholesky_factor(q, perm) (cholesky.hpp:164).
inline CholeskyFactor cholesky_factor(const SparseMatrixCSC& q, const std::vector<Index>& perm) {
  return cholesky_refactor(symbolic_analyze(q, perm), q);
}

/// cholesky_factor(q) (cholesky.hpp:170): nested dissection instead of AMD.
inline CholeskyFactor cholesky_factor(const SparseMatrixCSC& q) {
  if (q.nrows != q.ncols) throw DimensionError("symbolic_analyze: matrix not square");
  std::vector<int64_t> cp = b200::colptr64(q);
  std::vector<Index> perm(q.nrows);
  b200::check(gmrf_nd_order(q.nrows, cp.data(), q.row_idx.data(), perm.data()));
  return cholesky_factor(q, perm);
}

enum class TriangularMode { kLower, kUpper, kFull };

/// solve_triangular (cholesky.hpp:179): kLower/kUpper in permuted coordinates,
/// kFull returns Q⁻¹ b in original coordinates.
inline Vector solve_triangular(const CholeskyFactor& f, const Vector& b, TriangularMode mode) {
  const Index n = f.dim();
  if (static_cast<Index>(b.size()) != n)
    throw DimensionError("solve_triangular: dimension mismatch");
  Vector x(n);
  b200::check(gmrf_solve(f.device->h, static_cast<int>(mode), 1, b.data(), x.data()));
  return x;
}

/// solve (cholesky.hpp:225).
inline Vector solve(const CholeskyFactor& f, const Vector& b) {
  return solve_triangular(f, b, TriangularMode::kFull);
}

}  // namespace gmrfpde
