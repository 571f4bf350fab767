// Matérn SPDE regression posterior on the device (configs 1-2):
//
//   matern_prior (priors/matern.hpp:53-80)                Q = GramPlan(K̂; 1/m̃, 1/τ²)   (row 1)
//   point_observation_operator (info_operator.hpp:108-123,
//     eval_basis / locate, fem/space.hpp:67-109,376-394)  A on the host (m point locations)
//   condition_affine (gmrf.hpp:145-170)                   Q_post = GramPlan(A; Λ) over base Q,
//                                                         written straight into the panels (row 2)
//                                                         rhs = Aᵀ Λ (y − Aμ − b), μ = b = 0
//   cholesky_factor(Q_post) + solve                       supernodal factor / solves (rows 3-4)
//   variance_takahashi (gmrf.hpp:205)                     selected inversion (row 5)
//   sample_direct(post, Rng(seed)) × n_samples            batched upper solves (gmrf.hpp:173-184)
//
// The spatial matrices (P1 mass, Laplacian, lumped mass) are n_s-sized host
// inputs (fem.hpp); everything of the posterior's size runs on the device.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "factor.hpp"
#include "fem.hpp"
#include "gram.hpp"

namespace gmrf {

struct MeshSpec {
  int dim = 1;        // 1: interval [xa, xb]; 2: unit square
  i32 n_el = 999;     // elements (1-D) or cells per side (2-D)
  double xa = 0.0, xb = 1.0;
  i32 n_nodes() const { return dim == 1 ? n_el + 1 : (n_el + 1) * (n_el + 1); }
};

// eval_basis(space, points, {0, 0}) for P1 (space.hpp:376-394): row i holds the
// shape values of the element containing point i (locate, space.hpp:67-109),
// CSR with ascending columns. Points are dim-interleaved. Throws ContractError
// for a point outside the mesh, as the reference.
void point_operator(const MeshSpec& mesh, i32 m, const double* pts, std::vector<i64>& rp,
                    std::vector<i32>& ci, std::vector<double>& v);


class RegressionPosterior {
 public:
  // perm: optional fill-reducing ordering (new -> old) for the factor; nullptr
  // selects nested dissection. (Samples depend on the ordering, as the
  // reference's: pass its AMD ordering to reproduce its draws.)
  RegressionPosterior(const MeshSpec& mesh, const MaternSpec& spec, i32 m, const double* points,
                      const i32* perm, cudaStream_t stream = nullptr);
  ~RegressionPosterior();
  RegressionPosterior(const RegressionPosterior&) = delete;
  RegressionPosterior& operator=(const RegressionPosterior&) = delete;

  // y, noise_prec: m host values. Mean (and variances, samples) stay on the device.
  void run(const double* y, const double* noise_prec, bool variances, int n_samples,
           uint64_t seed);

  i32 n() const { return n_; }
  i32 m() const { return m_; }
  const Symbolic& symbolic() const { return *sym_; }
  std::shared_ptr<const Symbolic> symbolic_ptr() const { return sym_; }
  DeviceFactor& factor() { return *fac_; }
  const double* d_mean() const { return mean_.p; }
  const double* d_var() const { return var_.p; }
  const double* d_samples() const { return samples_.p; }
  int n_samples() const { return ns_done_; }
  // host copies for tests
  void copy_operator(std::vector<i64>& rp, std::vector<i32>& ci, std::vector<double>& v) const;
  void copy_precisions(std::vector<i64>& cp, std::vector<i32>& ri, std::vector<double>& q_prior,
                       std::vector<double>& q_post) const;
  struct Times {
    double setup_host_ms = 0, prior_ms = 0, update_ms = 0, numeric_ms = 0, solve_ms = 0,
           selinv_ms = 0, sample_ms = 0, total_ms = 0;
    i64 kernel_launches = 0;
  };
  const Times& times() const { return times_; }
  KernelProfiler prof_;

 private:
  MeshSpec mesh_;
  MaternSpec spec_;
  cudaStream_t stream_;
  i32 n_ = 0, m_ = 0;
  int ns_done_ = 0;
  Times times_;
  // host
  std::vector<i64> pcp_, arp_, acp_, amap_;
  std::vector<i32> pri_, aci_, ari_;
  std::vector<double> av_;
  bool sqrt_form_ = false;  // α >= 3: Q = Gram(Lᵀ) with the host square root
  std::shared_ptr<const Symbolic> sym_;
  std::unique_ptr<DeviceFactor> fac_;
  std::unique_ptr<GramPlan> gram_k_, gram_a_;
  // device
  DevBuf<double> d_kv_, d_kw_, d_av_, d_q_, d_qpost_, d_y_, d_lam_, d_wr_, rhs_, mean_, var_,
      samples_;
  DevBuf<i64> d_acp_, d_amap_;
  DevBuf<i32> d_ari_;
  cudaEvent_t ev_[2] = {};
};

}  // namespace gmrf
