// Fixed-pattern update system (update_system.hpp).
#include "update_system.hpp"

#include <algorithm>
#include <cstring>

namespace gmrf {

namespace {

// CSC (m × n: cp[n+1], ri) → CSR (rp[m+1], ci) plus, per CSR position, the
// CSC index of the value (the caller hands values over in CSC order)
void csc_to_csr(i32 m, i32 n, const i64* cp, const i32* ri, std::vector<i64>& rp,
                std::vector<i32>& ci, std::vector<i64>& vmap) {
  const i64 nnz = cp[n];
  rp.assign(static_cast<size_t>(m) + 1, 0);
  for (i64 p = 0; p < nnz; ++p) {
    require(ri[p] >= 0 && ri[p] < m, kDimension, "update system: operator row out of range");
    rp[ri[p] + 1]++;
  }
  for (i32 i = 0; i < m; ++i) rp[i + 1] += rp[i];
  ci.resize(nnz);
  vmap.resize(nnz);
  std::vector<i64> nx(rp.begin(), rp.end() - 1);
  for (i32 j = 0; j < n; ++j)
    for (i64 p = cp[j]; p < cp[j + 1]; ++p) {
      const i64 q = nx[ri[p]]++;
      ci[q] = j;
      vmap[q] = p;
    }
}

// symmetric closure of a square CSC pattern (rows sorted per column)
void symmetric_pattern(i32 n, const i64* cp, const i32* ri, std::vector<i64>& oc,
                       std::vector<i32>& orow) {
  std::vector<i64> a(cp, cp + n + 1), tc;
  std::vector<i32> ar(ri, ri + cp[n]), tr;
  tc.assign(static_cast<size_t>(n) + 1, 0);
  for (i64 p = 0; p < cp[n]; ++p) tc[ri[p] + 1]++;
  for (i32 j = 0; j < n; ++j) tc[j + 1] += tc[j];
  tr.resize(cp[n]);
  std::vector<i64> nx(tc.begin(), tc.end() - 1);
  for (i32 j = 0; j < n; ++j)
    for (i64 p = cp[j]; p < cp[j + 1]; ++p) tr[nx[ri[p]]++] = j;
  pattern_union(n, a, ar, tc, tr, oc, orow);
}

}  // namespace

UpdateSystem::UpdateSystem(i32 n, int base_kind, i32 bcols, const i64* bcp, const i32* bri,
                           const double* bv, i32 m, const i64* acp, const i32* ari,
                           const i32* perm, cudaStream_t stream)
    : n_(n), m_(m), stream_(stream) {
  require(n >= 0 && m >= 0, kDimension, "update system: negative dimension");
  require(base_kind == 0 || base_kind == 1, kContract, "update system: base kind is 0 or 1");
  require(base_kind == 1 || bcols == n, kDimension, "update system: Q must be n × n");
  acp_.assign(acp, acp + n + 1);
  ari_.assign(ari, ari + acp[n]);
  std::vector<i64> arp, avmap;
  std::vector<i32> aci;
  csc_to_csr(m, n, acp, ari, arp, aci, avmap);
  // pattern: B's (symmetric closure) ∪ AᵀA
  std::vector<i64> bpc, gcp;
  std::vector<i32> bpr, gri;
  if (base_kind == 0) {
    symmetric_pattern(n, bcp, bri, bpc, bpr);
  } else {
    gram_pattern(n, bcols, bcp, bri, bpc, bpr);  // S Sᵀ: rows of Sᵀ are S's columns
  }
  gram_pattern(n, m, arp.data(), aci.data(), gcp, gri);
  pattern_union(n, bpc, bpr, gcp, gri, pcp_, pri_);
  if (perm) perm_.assign(perm, perm + n);
  const size_t np = pri_.size();
  base_.alloc(np);
  h_.alloc(np);
  if (base_kind == 0) {  // Q's values at their union positions, zero elsewhere
    std::vector<double> b(np, 0.0);
    for (i32 j = 0; j < n; ++j) {
      i64 q = pcp_[j];
      for (i64 p = bcp[j]; p < bcp[j + 1]; ++p) {
        while (pri_[q] < bri[p]) ++q;
        b[q] = bv[p];
      }
    }
    base_.upload(b, stream_);
  } else {  // sym(S Sᵀ) on the device (gauss_newton.hpp:112-113)
    GramPlan gs(n, pcp_.data(), pri_.data(), bcols, bcp, bri, nullptr, stream_);
    DevBuf<double> sv;
    sv.upload(std::vector<double>(bv, bv + bcp[bcols]), stream_);
    gs.apply(sv.p, nullptr, 1.0, nullptr, base_.p, nullptr, nullptr, stream_);
    cuda_check(cudaStreamSynchronize(stream_), "q_eff");
  }
  // A's product map over the entries the factorization reads, values in CSC order
  gram_a_ = std::make_unique<GramPlan>(n, pcp_.data(), pri_.data(), m, arp.data(), aci.data(),
                                       nullptr, stream_, avmap.data(), base_kind == 0);
  a_.alloc(std::max<i64>(acp[n], 1));
  w_.alloc(std::max(m, 1));
}

bool UpdateSystem::same_operator(i32 m, const i64* acp, const i32* ari) const {
  if (m != m_) return false;
  if (!std::equal(acp_.begin(), acp_.end(), acp)) return false;
  return ari_.empty() || std::memcmp(ari_.data(), ari, ari_.size() * sizeof(i32)) == 0;
}

void UpdateSystem::stage(const double* a_values, const double* w) {
  const i64 na = acp_[n_];
  if (na)
    cuda_check(cudaMemcpyAsync(a_.p, a_values, na * 8, cudaMemcpyHostToDevice, stream_), "A");
  if (m_)
    cuda_check(cudaMemcpyAsync(w_.p, w, static_cast<size_t>(m_) * 8, cudaMemcpyHostToDevice,
                               stream_),
               "w");
}

void UpdateSystem::assemble(const double* a_values, const double* w, double c) {
  stage(a_values, w);
  gram_a_->apply(a_.p, w_.p, c, base_.p, h_.p, nullptr, nullptr, stream_);
}

void UpdateSystem::ensure_factor() {
  if (fac_) return;  // symbolic analysis and factor storage on first use (assemble needs neither)
  sym_ = std::make_shared<const Symbolic>(
      analyze(n_, pcp_.data(), pri_.data(), perm_.empty() ? nullptr : perm_.data()));
  fac_ = std::make_unique<DeviceFactor>(sym_, stream_);
}

int32_t UpdateSystem::refactor(const double* a_values, const double* w, const double* rhs) {
  ensure_factor();
  stage(a_values, w);
  if (rhs) {
    if (rhs_.n < static_cast<size_t>(std::max(n_, 1))) rhs_.alloc(std::max(n_, 1));
    cuda_check(cudaMemcpyAsync(rhs_.p, rhs, n_ * sizeof(double), cudaMemcpyHostToDevice, stream_),
               "rhs");
  }
  fac_->begin_numeric();
  gram_a_->apply(a_.p, w_.p, 1.0, base_.p, h_.p, fac_->d_qmap(), fac_->d_l(), stream_);
  return fac_->factor_panels(rhs ? rhs_.p : nullptr);
}

void UpdateSystem::solve_pending(double* x) {
  if (x_.n < static_cast<size_t>(std::max(n_, 1))) x_.alloc(std::max(n_, 1));
  fac_->solve_pending(x_.p);
  cuda_check(cudaMemcpyAsync(x, x_.p, n_ * sizeof(double), cudaMemcpyDeviceToHost, stream_), "x");
  cuda_check(cudaStreamSynchronize(stream_), "solve");
}

void UpdateSystem::copy_values(double* out) const {
  cuda_check(cudaMemcpyAsync(out, h_.p, pri_.size() * 8, cudaMemcpyDeviceToHost, stream_), "H");
  cuda_check(cudaStreamSynchronize(stream_), "H");
}

}  // namespace gmrf
