// Fixed-pattern weighted Gram update — the one device primitive behind the
// north_star's rows (1) and (2):
//
//   out[p] = ½(base[p] + c·Σ_k A_kR (w_k A_kC)) + ½(base[p] + c·Σ_k A_kC (w_k A_kR))
//
// for every entry p = (R, C) of a fixed symmetric CSC pattern P, with A an
// m × n sparse operator whose pattern is fixed and whose values / weights
// change per call. It is the reference's
//   symmetrize(add(base, multiply(transpose(A), scale_rows(w, A))))
// (gmrf.hpp:150-155 with A the observation operator and w = Λ;
//  gauss_newton.hpp:137-138 / :231-232 with A = J_k and w = Λ_pde;
//  gauss_newton.hpp:112-113 with A = Sᵀ, w = 1 → q_eff = sym(S Sᵀ))
// and, with base = 0 and c = 1/τ², the Matérn precision
//   symmetrize(scale(multiply(Kᵀ M̃⁻¹, K), 1/τ²))  (priors/matern.hpp:70-80).
// The per-entry sums run over the shared rows k in ascending order, the terms
// in the reference's operand order, both triangles summed separately and
// averaged: the same floating-point operations as the reference's column
// SpGEMM with a dense workspace (core/sparse.hpp:202-231) followed by
// symmetrize (:284-286). No atomics; every entry is written once.
//
// The product map (for each pattern entry, the value-index pairs of the rows
// it shares) is built once per (pattern, A pattern) on the host; calls only
// stream values. Writes go to a values array in pattern order and/or straight
// into the supernodal factor panels through the symbolic's qmap (entries the
// factorization reads), so a Gauss-Newton update never materialises H.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "factor.hpp"

namespace gmrf {

// Full symmetric CSC pattern of AᵀA for an m × n CSR operator (with the diagonal).
void gram_pattern(i32 n, i32 m, const i64* arp, const i32* aci, std::vector<i64>& cp,
                  std::vector<i32>& ri);
// Union of two sorted CSC patterns with n columns.
void pattern_union(i32 n, const std::vector<i64>& acp, const std::vector<i32>& ari,
                   const std::vector<i64>& bcp, const std::vector<i32>& bri, std::vector<i64>& cp,
                   std::vector<i32>& ri);

class GramPlan {
 public:
  // Pattern P: n × n full symmetric CSC (pcp, pri). A: m × n, CSR (arp, aci),
  // columns ascending per row. Every product A_kR A_kC must land in P
  // (StructuralError otherwise). lower_only: build sums only for entries with
  // R >= C in the pattern's own numbering that `need` marks (need == nullptr:
  // all entries).
  // vmap (optional): CSR position → index of that value in the caller's value
  // array (e.g. A handed over in CSC order). base_transpose: the base is not
  // assumed exactly symmetric — the (C, R) half of the average uses base(C, R)
  // (the reference symmetrizes base + product, gmrf.hpp:155).
  GramPlan(i32 n, const i64* pcp, const i32* pri, i32 m, const i64* arp, const i32* aci,
           const std::vector<char>* need, cudaStream_t stream, const i64* vmap = nullptr,
           bool base_transpose = false);

  // d_a: A values (CSR order, nnz), d_w: m weights (nullptr = 1), c: scale of
  // the product, d_base: pattern-order base values (nullptr = 0). Writes
  // d_out[p] (pattern order, may be nullptr) and, when d_qmap/d_L are given,
  // d_L[d_qmap[p]] for entries with d_qmap[p] >= 0.
  void apply(const double* d_a, const double* d_w, double c, const double* d_base, double* d_out,
             const i64* d_qmap, double* d_L, cudaStream_t stream);

  i64 nnz_pattern() const { return np_; }
  i64 entries() const { return ne_; }  // computed entries per apply
  int launches(bool weighted) const;
  i64 nnz_a() const { return na_; }
  i64 pairs() const { return npairs_; }
  // algorithmic bytes of one apply (A values + weights gathered once, base and
  // map read, pairs read, outputs written)
  double bytes(bool base, bool out, bool panels) const;

 private:
  i64 np_ = 0, na_ = 0, npairs_ = 0, ne_ = 0;
  i32 m_ = 0;
  DevBuf<i64> ent_;     // computed entries (pattern positions) when a mask was given
  DevBuf<i64> tpos_;    // per computed entry: pattern position of its transpose (base_transpose)
  DevBuf<i64> off_;     // np+1 pair offsets
  DevBuf<int2> pairs_;  // (index of A_kR, index of A_kC) in A's CSR value order
  DevBuf<i32> arow_;    // row k of every A value
  DevBuf<double> wa_;   // w_k A_kC scratch
};

}  // namespace gmrf
