// Space-time GMRF posterior on the device: SPDE prior assembly (row 1), IC
// conditioning, fixed-pattern Gauss-Newton update H = q_eff + JᵀΛJ written
// straight into the supernodal factor storage (row 2), the Gauss-Newton loop
// with Armijo backtracking (solver/gauss_newton.hpp:93-224), the Laplace
// precision (gauss_newton.hpp:228-240) and its marginal variances.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "factor.hpp"
#include "fem.hpp"
#include "fem_device.hpp"
#include "gram.hpp"

namespace gmrf {

// Device view of the Allen-Cahn residual data (spacetime.cu).
struct AcDev {
  int ns, nt, nk;
  const double* dt;  // per-step Δt [nt-1]
  double eps2;
  const char* slack;
  const int* kept;
  const i64* rp;
  const i32* ci;
  const double *mv, *kv, *ml;
};

struct SpaceTimeSpec {
  i32 n_el = 999;          // spatial elements (n_s = n_el + 1)
  double xa = -1.0, xb = 1.0;
  i32 n_t = 1000;          // time slices over [0, t_end] (uniform)
  double t_end = 1.0;
  double diffusion = 0.01 / 3.141592653589793;  // proxy ν (also the Burgers ν)
  double advection = 0.5;                        // proxy c
  MaternSpec noise{10.0, 1, 1.0}, init{10.0, 2, 1.0};
  double tau = 1.0;
  double eps = 1e-10;      // Dirichlet slack variance (priors/boundary.hpp:20)
  bool dirichlet = true;
  double ic_noise_prec = 1e8;
  int residual = 1;        // 0: linear (conditioned prior is the posterior), 1: Burgers weak IE,
                           // 2: Allen-Cahn weak IE (lumped cubic)
  double pde_noise_prec = 1e12;
  int dim = 1;             // 1: interval [xa, xb]; 2: unit square, n_el × n_el cells (triangles)
};

struct GnConfig {
  i32 max_iters = 10;
  double decrement_tol = 1e-5;
  double armijo_c = 1e-4;
  double shrink = 0.5;
  i32 max_backtracks = 30;
};

struct GnIter {
  i32 iter;
  double objective, decrement, step_size;
  i32 backtracks;
};

struct PhaseTimes {
  double setup_host_ms = 0;   // host: spatial blocks, patterns, symbolic (ND)
  double init_ms = 0;         // one-off device setup: uploads, first assembly
  double assemble_ms = 0;     // device: prior / q_eff assembly (per run)
  double condition_ms = 0;    // IC conditioning factor + mean solve
  double gn_ms = 0;           // Gauss-Newton loop
  double laplace_ms = 0;      // Laplace precision + factorization
  double selinv_ms = 0;       // marginal variances
  double numeric_ms = 0;      // sum of all numeric factorizations
  i32 n_factorizations = 0;
  double numeric_pure_ms = 0;  // factorizations with no fused forward sweep
  i32 n_pure_factorizations = 0;
  i64 kernel_launches = 0;
};

class SpaceTimePosterior {
 public:
  // part: partitioned factorization (partition.hpp) across ranks; the O(n)
  // work (assembly, residuals, line search) is replicated on every rank.
  explicit SpaceTimePosterior(const SpaceTimeSpec& spec, cudaStream_t stream = nullptr,
                              const PartitionSpec* part = nullptr);
  // Host part only (patterns, geometric ND, symbolic analysis): no device.
  static std::shared_ptr<const Symbolic> host_symbolic(const SpaceTimeSpec& spec);
  ~SpaceTimePosterior();

  // Full pipeline from the IC values u0 (n_s, host). Returns the GN trace.
  std::vector<GnIter> run(const double* u0, const GnConfig& cfg, bool variances);

  i32 n() const { return n_; }
  i32 n_space() const { return ns_; }
  const Symbolic& symbolic() const { return *sym_; }
  DeviceFactor& factor() { return *fac_; }
  const double* d_mean() const { return mean_.p; }   // posterior mean (mode)
  const double* d_var() const { return var_.p; }
  const double* d_mean_cond() const { return mean_cond_.p; }
  const PhaseTimes& times() const { return times_; }
  bool converged() const { return converged_; }
  // trace of the last run, complete also when it ended in a throw (line-search
  // stagnation: GaussNewtonStagnation carries it, gauss_newton.hpp:208-214)
  const std::vector<GnIter>& last_trace() const { return trace_; }
  // Master pattern and the assembled values (tests)
  void copy_pattern(std::vector<i64>& cp, std::vector<i32>& ri) const;
  void copy_values(std::vector<double>& qcond, std::vector<double>& qeff) const;
  void jacobian_csr(const double* d_u, std::vector<i64>& rp, std::vector<i32>& ci,
                    std::vector<double>& v);
  void residual(const double* d_u, double* d_r);
  i32 n_res() const { return nres_; }

 private:
  struct HostOnly {};
  SpaceTimePosterior(const SpaceTimeSpec& spec, HostOnly);
  void build_host();
  void assemble_device();
  void assemble_values();
  void fill_panels(const double* base, bool with_jacobian);
  double objective(const double* d_x, const double* d_fx);
  double dot(const double* a, const double* b, i64 n);
  void eval_residual(const double* d_u, double* d_f);
  void eval_jacobian(const double* d_u);
  AcDev ac_dev() const;

  SpaceTimeSpec spec_;
  cudaStream_t stream_;
  bool host_only_ = false;  // device-free symbolic planning (host_symbolic)
  PartitionSpec pspec_;
  Space1D space_{};
  SpatialOps ops_;
  SpaceTimeBlocks blk_;
  i32 ns_ = 0, nt_ = 0, n_ = 0, nres_ = 0, ms_ = 0;  // ms_: columns of S
  std::shared_ptr<const Symbolic> sym_;
  std::unique_ptr<DeviceFactor> fac_;
  PhaseTimes times_;

 public:
  KernelProfiler prof_;  // per-kernel-class timing (off by default)

 private:
  bool converged_ = false;
  std::vector<GnIter> trace_;
  cudaEvent_t ev_[4] = {};  // phase (0, 1) and factorization (2, 3) timing, reused

  // host patterns
  std::vector<i64> pcp_;
  std::vector<i32> pri_;
  Csc s_;                     // S_cond (CSC, N × M)
  std::vector<i64> jrp_;      // J CSR row pointers
  std::vector<i32> jci_;      // J CSR columns
  std::vector<i64> jcp_;      // J CSC column pointers
  std::vector<i32> jri_;      // J CSC rows
  std::vector<i64> jmap_;     // CSC position -> CSR value index
  // time grid t_s = t_end·s/(n_t−1) (as the oracle builds it), per-step Δt_s,
  // T_s = 1/(Δt_s τ²) and √T_s (spatiotemporal.hpp:118-120)
  std::vector<double> tg_, dts_, tstep_, sqt_;
  // JᵀΛJ (lower entries, straight into the panels) and q_eff = sym(S Sᵀ)
  std::unique_ptr<GramPlan> gram_j_, gram_s_;

  // device
  DevBuf<i64> d_pcp_, d_qmap_, d_scp_, d_srp_, d_jrp_, d_jcp_, d_jmap_;
  DevBuf<i32> d_pri_, d_sri_, d_sci_, d_jci_, d_jri_, kept_;
  DevBuf<double> d_qcond_, d_qeff_, d_sv_, d_svr_, d_jv_, d_lam_, d_tstep_, d_dts_, d_xn_, d_wf_;
  DevBuf<i64> d_blk_cp_;
  DevBuf<i32> d_blk_ri_;
  DevBuf<double> d_blk_v_;
  DevBuf<char> d_slack_;
  // Allen-Cahn: spatial M and K on the mass pattern (CSR) and the lumped mass
  DevBuf<i64> d_mrp_;
  DevBuf<i32> d_mci_;
  DevBuf<double> d_mv_, d_kv_, d_ml_;
  DevBuf<double> mean_cond_, mean_, var_, x_, c_, w_, g_, d_, cand_, f_, fc_, r1_, part_, u0_;
};

}  // namespace gmrf
