// Fixed-pattern update system: H = sym(B + Aᵀ diag(w) A) and its factor, with
// B either a given precision Q or sym(S Sᵀ) of a square root S. One object
// serves the reference's three update sites (north_star row 2):
//   condition_affine   B = Q,            A = observation operator, w = Λ  (gmrf.hpp:150-161)
//   gauss_newton       B = sym(S Sᵀ)|Q,  A = J_k, w = Λ_pde           (gauss_newton.hpp:110-140)
//   laplace_posterior  B = Q,            A = J(mode), w = Λ_pde       (gauss_newton.hpp:228-232)
// The union pattern, its symbolic analysis (nested dissection unless an
// ordering is given), the device factor and the Gram product map are built
// once; a refactorization streams A's values and writes H straight into the
// factor panels (no per-call permute / sort, cholesky.hpp:117).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "factor.hpp"
#include "gram.hpp"
#include "symbolic.hpp"

namespace gmrf {

class UpdateSystem {
 public:
  // base_kind 0: B = Q (n × n CSC, bcols = n); 1: B = sym(S Sᵀ), S n × bcols CSC.
  // A: m × n CSC pattern (values per refactor, in this CSC order).
  UpdateSystem(i32 n, int base_kind, i32 bcols, const i64* bcp, const i32* bri, const double* bv,
               i32 m, const i64* acp, const i32* ari, const i32* perm,
               cudaStream_t stream = nullptr);
  // H from A's values (CSC order) and the m weights; factor. Returns -1 or the
  // original index of the failing pivot (cholesky.hpp:153-156).
  // rhs (host, n values, optional): the forward sweep of H x = rhs rides along
  // with the factorization (DeviceFactor::factor_panels); solve_pending(x) finishes it.
  int32_t refactor(const double* a_values, const double* w, const double* rhs = nullptr);
  void solve_pending(double* x);
  // values only: H = sym(B + c·AᵀWA) into the pattern-order buffer (no factor)
  void assemble(const double* a_values, const double* w, double c);
  bool same_operator(i32 m, const i64* acp, const i32* ari) const;

  i32 n() const { return n_; }
  i32 m() const { return m_; }
  // created by the first refactor (ensure_factor)
  std::shared_ptr<const Symbolic> symbolic() {
    ensure_factor();
    return sym_;
  }
  DeviceFactor& factor() {
    ensure_factor();
    return *fac_;
  }
  void ensure_factor();
  const std::vector<i64>& col_ptr() const { return pcp_; }
  const std::vector<i32>& row_idx() const { return pri_; }
  void copy_values(double* out) const;  // H of the last refactor / assemble, pattern order

 private:
  i32 n_, m_;
  cudaStream_t stream_;
  std::vector<i64> pcp_, acp_;
  std::vector<i32> pri_, ari_, perm_;
  std::shared_ptr<const Symbolic> sym_;
  std::unique_ptr<DeviceFactor> fac_;
  std::unique_ptr<GramPlan> gram_a_;
  void stage(const double* a_values, const double* w);
  DevBuf<double> base_, h_, a_, w_, rhs_, x_;
};

}  // namespace gmrf
