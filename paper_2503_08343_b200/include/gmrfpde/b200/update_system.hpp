// C++ handle over gmrf_update_system_* (include/gmrf_b200.h): the fixed-pattern
// update H = symmetrize(B + c·Aᵀ diag(w) A) and its device factor, used by the
// drop-in gmrf.hpp (condition_affine), solver/gauss_newton.hpp (gauss_newton,
// laplace_posterior) and priors/matern.hpp (matern_prior).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "gmrf_b200.h"
#include "gmrfpde/core/cholesky.hpp"
#include "gmrfpde/core/sparse.hpp"

namespace gmrfpde::b200 {

class UpdateSystem : public std::enable_shared_from_this<UpdateSystem> {
 public:
  enum Base { kPrecision = 0, kSqrt = 1 };  // B = Q, or B = symmetrize(S Sᵀ)

  // b: Q (kPrecision) or S (kSqrt); a: the operator's CSC pattern (values per call)
  static std::shared_ptr<UpdateSystem> make(Base kind, const SparseMatrixCSC& b,
                                            const SparseMatrixCSC& a) {
    auto u = std::shared_ptr<UpdateSystem>(new UpdateSystem());
    const std::vector<int64_t> bcp(b.col_ptr.begin(), b.col_ptr.end());
    u->acp_.assign(a.col_ptr.begin(), a.col_ptr.end());
    u->m_ = a.nrows;
    u->n_ = b.nrows;
    if (a.ncols != b.nrows) throw DimensionError("update system: operator columns != dimension");
    check(gmrf_update_system_create(b.nrows, kind, b.ncols, bcp.data(), b.row_idx.data(),
                                    b.values.data(), a.nrows, u->acp_.data(), a.row_idx.data(),
                                    nullptr, &u->h_));
    return u;
  }
  ~UpdateSystem() {
    if (h_) gmrf_update_system_free(h_);
  }

  bool same_operator(const SparseMatrixCSC& a) const {
    if (a.nrows != m_ || a.ncols != n_) return false;
    const std::vector<int64_t> cp(a.col_ptr.begin(), a.col_ptr.end());
    return gmrf_update_system_same_operator(h_, a.nrows, cp.data(), a.row_idx.data()) == 1;
  }
  // H from a's values and w, factorized on the device (cholesky_refactor of H)
  void refactor(const SparseMatrixCSC& a, const Vector& w) {
    int32_t bad = -1;
    const int rc = gmrf_update_system_refactor(h_, a.values.data(), w.data(), &bad);
    if (rc != GMRF_OK) raise(rc, bad);
  }
  // refactor + solve H x = b in one call (the forward sweep rides along with the
  // factorization on the device)
  Vector refactor_solve(const SparseMatrixCSC& a, const Vector& w, const Vector& b) {
    int32_t bad = -1;
    Vector x(b.size());
    const int rc =
        gmrf_update_system_refactor_solve(h_, a.values.data(), w.data(), b.data(), x.data(), &bad);
    if (rc != GMRF_OK) raise(rc, bad);
    return x;
  }
  // H's values only, c scaling the product
  void assemble(const SparseMatrixCSC& a, const Vector& w, Real c) {
    check(gmrf_update_system_assemble(h_, a.values.data(), w.data(), c, nullptr));
  }
  // H (last refactor / assemble) on the union pattern, host CSC
  SparseMatrixCSC matrix() const {
    SparseMatrixCSC h(n_, n_);
    std::vector<int64_t> cp(n_ + 1);
    check(gmrf_update_system_matrix(h_, cp.data(), nullptr, nullptr));
    h.row_idx.resize(cp[n_]);
    h.values.resize(cp[n_]);
    check(gmrf_update_system_matrix(h_, cp.data(), h.row_idx.data(), h.values.data()));
    h.col_ptr.assign(cp.begin(), cp.end());
    return h;
  }
  // the factor of the last refactor, as the reference's CholeskyFactor
  CholeskyFactor factor() {
    return wrap_factor(gmrf_update_system_factor(h_), gmrf_update_system_symbolic(h_),
                       shared_from_this());
  }
  Vector solve(const Vector& b) {
    Vector x(b.size());
    check(gmrf_solve(gmrf_update_system_factor(h_), GMRF_SOLVE_FULL, 1, b.data(), x.data()));
    return x;
  }

 private:
  UpdateSystem() = default;
  gmrf_update_system_t* h_ = nullptr;
  std::vector<int64_t> acp_;
  Index m_ = 0, n_ = 0;
};

}  // namespace gmrfpde::b200
