// Matérn SPDE regression posterior on the device. See regression.hpp.
#include "regression.hpp"

#include "fem_device.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <string>

#include "symbolic.hpp"

namespace gmrf {

namespace {

// wr_i = Λ_i (y_i − 0): the observation residual y − (Aμ + b) with μ = b = 0,
// weighted by the diagonal noise precision (gmrf.hpp:113-118, :157)
__global__ void k_obs_weight(int m, const double* __restrict__ lam, const double* __restrict__ y,
                             double* __restrict__ wr) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    wr[i] = (y[i] - 0.0) * lam[i];
}

// rhs_j = Σ_i A_ij wr_i over column j of A, rows ascending (matvec_transpose)
__global__ void k_at_x(int n, const i64* __restrict__ cp, const i32* __restrict__ ri,
                       const i64* __restrict__ vmap, const double* __restrict__ v,
                       const double* __restrict__ x, double* __restrict__ y) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (i64 p = cp[j]; p < cp[j + 1]; ++p) s += v[vmap[p]] * x[ri[p]];
    y[j] = s;
  }
}

int grid_of(i64 n) {
  return static_cast<int>(std::max<i64>(1, std::min<i64>((n + 255) / 256, 148 * 16)));
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// upper_bound cell on a node axis, clamped to [0, n_cells − 1] (space.hpp:118-122)
i32 axis_cell(const std::vector<double>& axis, double p) {
  const i32 c = static_cast<i32>(std::upper_bound(axis.begin(), axis.end(), p) - axis.begin()) - 1;
  return std::clamp<i32>(c, 0, static_cast<i32>(axis.size()) - 2);
}

}  // namespace

void point_operator(const MeshSpec& mesh, i32 m, const double* pts, std::vector<i64>& rp,
                    std::vector<i32>& ci, std::vector<double>& v) {
  require(mesh.dim == 1 || mesh.dim == 2, kContract, "point operator: dim must be 1 or 2");
  require(m >= 0, kDimension, "point operator: negative point count");
  rp.assign(1, 0);
  ci.clear();
  v.clear();
  std::vector<double> ax(static_cast<size_t>(mesh.n_el) + 1);
  if (mesh.dim == 1) {
    const Space1D s{mesh.n_el, mesh.xa, mesh.xb};
    for (i32 i = 0; i <= mesh.n_el; ++i) ax[i] = s.x(i);
  } else {
    const Space2D s{mesh.n_el};
    for (i32 i = 0; i <= mesh.n_el; ++i) ax[i] = s.coord(i);
  }
  const double tol = 1e-10 * (ax.back() - ax.front());
  for (i32 i = 0; i < m; ++i) {
    if (mesh.dim == 1) {
      const double p = pts[i];
      if (p < ax.front() - tol || p > ax.back() + tol)
        fail(kContract, "locate: point " + std::to_string(p) + " outside the mesh");
      const i32 e = axis_cell(ax, p);
      const double h = ax[e + 1] - ax[e];
      const double xi = (p - ax[e]) / h;  // eval_element (space.hpp:317-324): unclamped
      ci.push_back(e);
      v.push_back(1.0 - xi);
      ci.push_back(e + 1);
      v.push_back(xi);
    } else {
      const double x = pts[2 * i], y = pts[2 * i + 1];
      if (x < ax.front() - tol || x > ax.back() + tol || y < ax.front() - tol ||
          y > ax.back() + tol)
        fail(kContract, "locate: point (" + std::to_string(x) + ", " + std::to_string(y) +
                            ") outside the mesh");
      const i32 ix = axis_cell(ax, x), iy = axis_cell(ax, y);
      const double s = std::clamp((x - ax[ix]) / (ax[ix + 1] - ax[ix]), 0.0, 1.0);
      const double t = std::clamp((y - ax[iy]) / (ax[iy + 1] - ax[iy]), 0.0, 1.0);
      const i32 side = mesh.n_el + 1;
      const i32 v00 = iy * side + ix, v10 = v00 + 1, v11 = v00 + side + 1, v01 = v00 + side;
      // triangle (v00, v10, v11) for t <= s, else (v00, v11, v01) (mesh.hpp:140-147)
      const bool lower = t <= s;
      const i32 tri[3] = {v00, lower ? v10 : v11, lower ? v11 : v01};
      auto nx = [&](i32 d) { return ax[d % side]; };
      auto ny = [&](i32 d) { return ax[d / side]; };
      // inverse Jacobian of the element map, then barycentric shapes (space.hpp:283-306,326-336)
      const double x0 = nx(tri[0]), y0 = ny(tri[0]);
      const double j00 = nx(tri[1]) - x0, j10 = ny(tri[1]) - y0;
      const double j01 = nx(tri[2]) - x0, j11 = ny(tri[2]) - y0;
      const double det = j00 * j11 - j01 * j10;
      const double ji0 = j11 / det, ji1 = -j01 / det, ji2 = -j10 / det, ji3 = j00 / det;
      const double dx = x - x0, dy = y - y0;
      const double xi = ji0 * dx + ji1 * dy, eta = ji2 * dx + ji3 * dy;
      std::pair<i32, double> e3[3] = {{tri[0], 1.0 - xi - eta}, {tri[1], xi}, {tri[2], eta}};
      std::sort(e3, e3 + 3, [](const auto& a, const auto& b) { return a.first < b.first; });
      for (const auto& e : e3) {
        ci.push_back(e.first);
        v.push_back(e.second);
      }
    }
    rp.push_back(static_cast<i64>(ci.size()));
  }
}

RegressionPosterior::RegressionPosterior(const MeshSpec& mesh, const MaternSpec& spec, i32 m,
                                         const double* points, const i32* perm,
                                         cudaStream_t stream)
    : mesh_(mesh), spec_(spec), stream_(stream), m_(m) {
  const double t0 = now_ms();
  require(spec.kappa > 0 && spec.alpha >= 1 && spec.tau > 0, kContract, "matern: bad spec");
  require(mesh.n_el >= 1, kContract, "mesh: need at least one element");
  // P1 element assembly, lumping and constraint folding on the device (fem_device.cu)
  FemDeviceScope fem_scope;
  SpatialOps ops = mesh.dim == 1 ? spatial_ops_device(Space1D{mesh.n_el, mesh.xa, mesh.xb}, 0.0, 0.0,
                                                      false, stream_)
                                 : spatial_ops_device(Space2D{mesh.n_el}, 1.0, stream_);
  n_ = ops.n;
  // prior operator rows (row 1): α <= 2 → K̂ = K_Δ + κ²M with weights 1/m̃ and
  // scale 1/τ² (matern.hpp:56-73, α = 1 and 2 give the same Q); α >= 3 → the
  // square root L_α (matern.hpp:74-78) and Q = L Lᵀ = Gram(Lᵀ)
  std::vector<i64> kcp;
  std::vector<i32> kri;
  std::vector<double> kv, kw;
  double c = 1.0;
  if (spec.alpha <= 2) {
    const Csc k = add(ops.lap, ops.mass, 1.0, spec.kappa * spec.kappa);
    const Csc kr = transpose(k);  // CSR rows of K̂
    kcp = kr.cp;
    kri = kr.ri;
    kv = kr.v;
    const std::vector<double> lum = lumped_mass(ops.mass);
    kw.resize(lum.size());
    for (size_t i = 0; i < lum.size(); ++i) kw[i] = 1.0 / lum[i];
    c = 1.0 / (spec.tau * spec.tau);
  } else {
    sqrt_form_ = true;
    const MaternPrior mp = matern_prior(ops, spec, 1e-10);
    kcp = mp.sqrt.cp;  // columns of L = rows of Lᵀ
    kri = mp.sqrt.ri;
    kv = mp.sqrt.v;
  }
  const i32 mk = static_cast<i32>(kcp.size()) - 1;
  // observation operator (host: m point locations)
  point_operator(mesh, m, points, arp_, aci_, av_);
  // pattern: KᵀK (contains AᵀA for P1: an element's vertices are mutually adjacent)
  gram_pattern(n_, mk, kcp.data(), kri.data(), pcp_, pri_);
  {
    std::vector<i64> acp, ucp;
    std::vector<i32> ari, uri;
    gram_pattern(n_, m, arp_.data(), aci_.data(), acp, ari);
    pattern_union(n_, pcp_, pri_, acp, ari, ucp, uri);
    pcp_.swap(ucp);
    pri_.swap(uri);
  }
  // A by columns for Aᵀx, with the CSR value index of each entry
  acp_.assign(static_cast<size_t>(n_) + 1, 0);
  for (i32 col : aci_) acp_[col + 1]++;
  for (i32 j = 0; j < n_; ++j) acp_[j + 1] += acp_[j];
  ari_.resize(aci_.size());
  amap_.resize(aci_.size());
  {
    std::vector<i64> nx(acp_.begin(), acp_.end() - 1);
    for (i32 i = 0; i < m; ++i)
      for (i64 p = arp_[i]; p < arp_[i + 1]; ++p) {
        const i64 q = nx[aci_[p]]++;
        ari_[q] = i;
        amap_[q] = p;
      }
  }
  // symbolic (ND unless an ordering is given), device factor, product maps
  SymbolicOptions opt;
  sym_ = std::make_shared<const Symbolic>(analyze(n_, pcp_.data(), pri_.data(), perm, opt));
  fac_ = std::make_unique<DeviceFactor>(sym_, stream_);
  fac_->set_profiler(&prof_);
  fac_->set_selinv_inplace(true);
  gram_k_ = std::make_unique<GramPlan>(n_, pcp_.data(), pri_.data(), mk, kcp.data(), kri.data(),
                                       nullptr, stream_);
  gram_a_ = std::make_unique<GramPlan>(n_, pcp_.data(), pri_.data(), m, arp_.data(), aci_.data(),
                                       nullptr, stream_);
  d_kv_.upload(kv, stream_);
  if (!kw.empty()) d_kw_.upload(kw, stream_);
  d_av_.upload(av_, stream_);
  d_acp_.upload(acp_, stream_);
  d_ari_.upload(ari_, stream_);
  d_amap_.upload(amap_, stream_);
  const size_t np = pri_.size();
  d_q_.alloc(np);
  d_qpost_.alloc(np);
  d_y_.alloc(std::max(m, 1));
  d_lam_.alloc(std::max(m, 1));
  d_wr_.alloc(std::max(m, 1));
  for (DevBuf<double>* b : {&rhs_, &mean_, &var_}) b->alloc(std::max(n_, 1));
  // prior precision once (row 1)
  prof_.run(stream_, "assemble.prior", 0.0, gram_k_->bytes(false, true, false), [&] {
    gram_k_->apply(d_kv_.p, kw.empty() ? nullptr : d_kw_.p, c, nullptr, d_q_.p, nullptr, nullptr,
                   stream_);
  });
  for (cudaEvent_t& e : ev_) cuda_check(cudaEventCreate(&e), "event");
  cuda_check(cudaStreamSynchronize(stream_), "regression setup");
  times_.setup_host_ms = now_ms() - t0;
}

RegressionPosterior::~RegressionPosterior() {
  for (cudaEvent_t e : ev_)
    if (e) cudaEventDestroy(e);
}

void RegressionPosterior::run(const double* y, const double* noise_prec, bool variances,
                              int n_samples, uint64_t seed) {
  require(n_samples >= 0, kContract, "sample_direct: negative sample count");
  const double setup = times_.setup_host_ms;
  times_ = Times{};
  times_.setup_host_ms = setup;
  cudaEventRecord(ev_[0], stream_);
  if (m_ > 0) {
    cuda_check(cudaMemcpyAsync(d_y_.p, y, m_ * sizeof(double), cudaMemcpyHostToDevice, stream_),
               "y");
    cuda_check(cudaMemcpyAsync(d_lam_.p, noise_prec, m_ * sizeof(double), cudaMemcpyHostToDevice,
                               stream_),
               "noise");
  }
  // Q_post = sym(Q + AᵀΛA) into the panels and (pattern order) d_qpost_  (row 2)
  fac_->begin_numeric();
  prof_.run(stream_, "update.q_atla", 0.0, gram_a_->bytes(true, true, true), [&] {
    gram_a_->apply(d_av_.p, d_lam_.p, 1.0, d_q_.p, d_qpost_.p, fac_->d_qmap(), fac_->d_l(),
                   stream_);
  });
  // rhs = Aᵀ Λ (y − Aμ − b)
  k_obs_weight<<<grid_of(m_), 256, 0, stream_>>>(m_, d_lam_.p, d_y_.p, d_wr_.p);
  k_at_x<<<grid_of(n_), 256, 0, stream_>>>(n_, d_acp_.p, d_ari_.p, d_amap_.p, d_av_.p, d_wr_.p,
                                           rhs_.p);
  times_.kernel_launches += gram_a_->launches(true) + 2;
  const int32_t bad = fac_->factor_panels();
  times_.kernel_launches += fac_->launches_numeric();
  if (bad >= 0)
    fail(kNotSpd, "condition_affine: cholesky: non-positive pivot at index " + std::to_string(bad));
  fac_->solve(2, 1, rhs_.p, mean_.p, true);  // μ_post = 0 + Q_post⁻¹ rhs
  times_.kernel_launches += fac_->launches_solve();
  if (n_samples > 0) {
    samples_.alloc(static_cast<size_t>(n_) * n_samples);
    fac_->sample_direct(mean_.p, n_samples, seed, samples_.p);
  }
  if (variances) {  // last use of the factor: Σ overwrites L in place
    fac_->selinv(var_.p, true);
    times_.kernel_launches += fac_->launches_selinv();
  }
  ns_done_ = n_samples;
  cudaEventRecord(ev_[1], stream_);
  cuda_check(cudaEventSynchronize(ev_[1]), "regression run");
  float ms = 0;
  cudaEventElapsedTime(&ms, ev_[0], ev_[1]);
  times_.total_ms = ms;
}

void RegressionPosterior::copy_operator(std::vector<i64>& rp, std::vector<i32>& ci,
                                        std::vector<double>& v) const {
  rp = arp_;
  ci = aci_;
  v = av_;
}

void RegressionPosterior::copy_precisions(std::vector<i64>& cp, std::vector<i32>& ri,
                                          std::vector<double>& q_prior,
                                          std::vector<double>& q_post) const {
  cp = pcp_;
  ri = pri_;
  q_prior.resize(pri_.size());
  q_post.resize(pri_.size());
  cuda_check(cudaMemcpy(q_prior.data(), d_q_.p, q_prior.size() * 8, cudaMemcpyDeviceToHost), "Q");
  cuda_check(cudaMemcpy(q_post.data(), d_qpost_.p, q_post.size() * 8, cudaMemcpyDeviceToHost),
             "Q_post");
}

}  // namespace gmrf
