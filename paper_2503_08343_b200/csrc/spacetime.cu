// Space-time GMRF posterior on the device. See spacetime.hpp.
#include "spacetime.hpp"

#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <string>

namespace gmrf {

namespace {

constexpr int kBlkCmm = 0, kBlkCgg = 1, kBlkCmg = 2, kBlkQ1 = 3, kBlkGmm = 4, kBlkGff = 5,
              kBlkGmf = 6, kBlkGl1 = 7, kNumBlk = 8;

struct BlkDev {
  const i64* cp;   // kNumBlk * (n+1)
  const i32* ri;
  const double* v;
  i32 n;
};

__device__ __forceinline__ double blk_at(const BlkDev& b, int k, int i, int j) {
  const i64* cp = b.cp + static_cast<i64>(k) * (b.n + 1);
  i64 lo = cp[j], hi = cp[j + 1];
  while (lo < hi) {
    i64 mid = (lo + hi) >> 1;
    if (b.ri[mid] < i) lo = mid + 1; else hi = mid;
  }
  return (lo < cp[j + 1] && b.ri[lo] == i) ? b.v[lo] : 0.0;
}

// Joint value of the space-time precision at (R, C) before symmetrization:
// the triplets spatiotemporal.hpp:112-156 appends, with the per-step
// T_s = 1/(Δt_s τ²): slice s's diagonal block collects T_{s-1}·C_gg (step s−1)
// and T_s·C_mm (step s) (slice 0: Q1 + T_0·C_mm), the off-diagonal blocks
// (−T_s)·C_mg and its transpose. Two terms per entry at most, so the sum is
// order-independent.
__device__ __forceinline__ double st_entry(const BlkDev& b, const double* T, int sr, int a, int sc,
                                           int c, int nt) {
  if (sr == sc) {
    double v = 0.0;
    if (sr < nt - 1) v += T[sr] * blk_at(b, kBlkCmm, a, c);
    if (sr >= 1) v += T[sr - 1] * blk_at(b, kBlkCgg, a, c);
    if (sr == 0) v += blk_at(b, kBlkQ1, a, c);
    return v;
  }
  if (sc == sr + 1) return (-T[sr]) * blk_at(b, kBlkCmg, a, c);
  if (sr == sc + 1) return (-T[sc]) * blk_at(b, kBlkCmg, c, a);
  return 0.0;
}

// Row 1: assembly of Q_cond = sym(Q_prior) + AᵀΛA on the master pattern, one
// thread per joint column (q_eff = sym(S Sᵀ) is a GramPlan product). Slack
// (constrained) coordinates carry only 1/ε on the diagonal
// (spatiotemporal.hpp:166-183); the IC observation A = I on slice 0 adds Λ_ic
// on that slice's diagonal.
__global__ void k_st_assemble(const i64* __restrict__ pcp, const i32* __restrict__ pri, int N,
                              int ns, int nt, const double* __restrict__ T, double inv_eps,
                              double ic_prec, const char* __restrict__ slack, BlkDev b,
                              double* __restrict__ qcond) {
  for (int C = blockIdx.x * blockDim.x + threadIdx.x; C < N; C += gridDim.x * blockDim.x) {
    const int sc = C / ns, c = C - sc * ns;
    for (i64 p = pcp[C]; p < pcp[C + 1]; ++p) {
      const int R = pri[p];
      const int sr = R / ns, a = R - sr * ns;
      double vq;
      if (slack[a] || slack[c]) {
        vq = (R == C) ? inv_eps : 0.0;
      } else {
        vq = 0.5 * st_entry(b, T, sr, a, sc, c, nt) + 0.5 * st_entry(b, T, sc, c, sr, a, nt);
      }
      if (R == C && sr == 0) vq += ic_prec;
      qcond[p] = vq;
    }
  }
}

// Conditioning base: L[qmap[p]] = base[p] (the Gauss-Newton and Laplace
// updates add JᵀΛJ through GramPlan, gram.hpp).
__global__ void k_fill_panels(const i64* __restrict__ pcp, const i32* __restrict__ pri, int N,
                              const i64* __restrict__ qmap, const double* __restrict__ base,
                              const i64* __restrict__ jcp, const i32* __restrict__ jri,
                              const i64* __restrict__ jmap, const double* __restrict__ jv,
                              double lam, double* __restrict__ L) {
  for (int C = blockIdx.x * blockDim.x + threadIdx.x; C < N; C += gridDim.x * blockDim.x) {
    for (i64 p = pcp[C]; p < pcp[C + 1]; ++p) {
      const i64 o = qmap[p];
      if (o < 0) continue;
      double v = base[p];
      if (jcp) {
        const int R = pri[p];
        i64 x = jcp[R], xe = jcp[R + 1], y = jcp[C], ye = jcp[C + 1];
        double s = 0.0;
        while (x < xe && y < ye) {
          const int rx = jri[x], ry = jri[y];
          if (rx < ry) {
            ++x;
          } else if (ry < rx) {
            ++y;
          } else {
            s += lam * jv[jmap[x]] * jv[jmap[y]];
            ++x;
            ++y;
          }
        }
        v += s;
      }
      L[o] = v;
    }
  }
}

// y = A x for a CSR (or, with rp/ci of a CSC, y = Aᵀ x). vmap optional.
__global__ void k_spmv(int nrows, const i64* __restrict__ rp, const i32* __restrict__ ci,
                       const double* __restrict__ v, const i64* __restrict__ vmap,
                       const double* __restrict__ x, double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (i64 p = rp[i]; p < rp[i + 1]; ++p) s += (vmap ? v[vmap[p]] : v[p]) * x[ci[p]];
    y[i] = s;
  }
}

__global__ void k_weighted_misfit(int m, double lam, const double* __restrict__ f,
                                  double* __restrict__ w) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    w[i] = lam * (0.0 - f[i]);
}

__global__ void k_axpby(int n, double a, const double* __restrict__ x, double b,
                        const double* __restrict__ y, double* __restrict__ z) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    z[i] = a * x[i] + b * y[i];
}

// Deterministic dot product: fixed grid, fixed per-thread order, tree reduce.
constexpr int kDotBlocks = 296, kDotThreads = 256;
__global__ void k_dot_partial(i64 n, const double* __restrict__ a, const double* __restrict__ b,
                              double* __restrict__ part) {
  __shared__ double sh[kDotThreads];
  double s = 0.0;
  for (i64 i = blockIdx.x * static_cast<i64>(kDotThreads) + threadIdx.x; i < n;
       i += static_cast<i64>(kDotBlocks) * kDotThreads)
    s += a[i] * b[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = kDotThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void k_dot_final(double* __restrict__ part, double* __restrict__ out) {
  __shared__ double sh[512];
  const int t = threadIdx.x;
  sh[t] = t < kDotBlocks ? part[t] : 0.0;
  __syncthreads();
  for (int o = 256; o > 0; o >>= 1) {
    if (t < o) sh[t] += sh[t + o];
    __syncthreads();
  }
  if (t == 0) out[0] = sh[0];
}

// ---- Burgers weak residual, P1, implicit Euler (residual.hpp:244-382) ------
// Element e spans nodes e, e+1 with its own length x[e+1] − x[e] (the node
// coordinates are rounded, mesh.hpp:63-70); step s has its own Δt_s
// (t_grid differences, residual.hpp:304,371).
struct BurgersDev {
  int ns, nt, nk;           // spatial dofs, slices, kept rows per step
  double nu;
  const double* x;          // node coordinates [ns]
  const double* dt;         // per-step Δt [nt-1]
  const char* slack;
  const int* kept;          // kept row k -> dof
};

__device__ __forceinline__ double um(const BurgersDev& B, const double* u, int s, int j) {
  return (j < 0 || j >= B.ns || B.slack[j]) ? 0.0 : u[static_cast<i64>(s) * B.ns + j];
}
__device__ __forceinline__ double elen(const BurgersDev& B, int e) { return B.x[e + 1] - B.x[e]; }

// 2-point Gauss-Legendre on [0,1] (degree-3 rule of residual.hpp:208-209)
__device__ __forceinline__ void gl2(double* xi, double* w) {
  const double d = 0.5 / sqrt(3.0);
  xi[0] = 0.5 - d;
  xi[1] = 0.5 + d;
  w[0] = w[1] = 0.5;
}

// weak advection a_d(v) = ∫ φ_d v ∂x v, v slack-masked (residual.hpp:206-235):
// per quadrature point v_q = Σ v φ, ∂x v_q = Σ v φ'/h, term (w h) φ_d v_q ∂x v_q
__device__ double adv_row(const BurgersDev& B, const double* u, int s, int d) {
  double xi[2], w[2];
  gl2(xi, w);
  double acc = 0.0;
  for (int e = d - 1; e <= d; ++e) {
    if (e < 0 || e >= B.ns - 1) continue;
    const double h = elen(B, e);
    const double vl = um(B, u, s, e), vr = um(B, u, s, e + 1);
    const double dv = vl * (-1.0 / h) + vr * (1.0 / h);
    for (int q = 0; q < 2; ++q) {
      const double phi = (d == e) ? 1.0 - xi[q] : xi[q];
      const double vq = vl * (1.0 - xi[q]) + vr * xi[q];
      acc += w[q] * h * phi * vq * dv;
    }
  }
  return acc;
}

// P1 mass / stiffness entries of row d (closed form per element, slack masked)
__device__ __forceinline__ double mass_ij(const BurgersDev& B, int d, int j) {
  if (j < 0 || j >= B.ns || B.slack[j]) return 0.0;
  if (j == d) {
    double v = 0.0;
    if (d > 0) v += elen(B, d - 1) / 3.0;
    if (d < B.ns - 1) v += elen(B, d) / 3.0;
    return v;
  }
  return elen(B, j < d ? j : d) / 6.0;
}
__device__ __forceinline__ double stiff_ij(const BurgersDev& B, int d, int j) {
  if (j < 0 || j >= B.ns || B.slack[j]) return 0.0;
  if (j == d) {
    double v = 0.0;
    if (d > 0) v += 1.0 / elen(B, d - 1);
    if (d < B.ns - 1) v += 1.0 / elen(B, d);
    return v;
  }
  return -1.0 / elen(B, j < d ? j : d);
}

__global__ void k_burgers_res(BurgersDev B, const double* __restrict__ u, double* __restrict__ f) {
  const int nrow = (B.nt - 1) * B.nk;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < nrow; row += gridDim.x * blockDim.x) {
    const int s = row / B.nk, d = B.kept[row - s * B.nk];
    double mdu = 0.0, kd = 0.0;
    for (int j = d - 1; j <= d + 1; ++j) {
      mdu += mass_ij(B, d, j) * (um(B, u, s + 1, j) - um(B, u, s, j));
      kd += stiff_ij(B, d, j) * um(B, u, s + 1, j);
    }
    f[row] = mdu / B.dt[s] + (B.nu * kd + adv_row(B, u, s + 1, d));
  }
}

// Jacobian row (step s, dof d): slice s → (−1/Δt)·M (θ = 1), slice s+1 →
// (ν K̂ + J_adv) + (1/Δt)·M, columns ascending, slack columns skipped
// (residual.hpp:353-377: θ-scaled slice Jacobian plus mass_coeff·M̂).
__global__ void k_burgers_jac(BurgersDev B, const double* __restrict__ u, const i64* __restrict__ rp,
                              double* __restrict__ jv) {
  const int nrow = (B.nt - 1) * B.nk;
  double xi[2], w[2];
  gl2(xi, w);
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < nrow; row += gridDim.x * blockDim.x) {
    const int s = row / B.nk, d = B.kept[row - s * B.nk];
    const double inv_dt = 1.0 / B.dt[s];
    i64 p = rp[row];
    for (int j = d - 1; j <= d + 1; ++j) {
      if (j < 0 || j >= B.ns || B.slack[j]) continue;
      jv[p++] = (-inv_dt) * mass_ij(B, d, j);
    }
    for (int j = d - 1; j <= d + 1; ++j) {
      if (j < 0 || j >= B.ns || B.slack[j]) continue;
      double ja = 0.0;
      for (int e = d - 1; e <= d; ++e) {
        if (e < 0 || e >= B.ns - 1) continue;
        if (j != e && j != e + 1) continue;
        const double h = elen(B, e);
        const double vl = um(B, u, s + 1, e), vr = um(B, u, s + 1, e + 1);
        const double dv = vl * (-1.0 / h) + vr * (1.0 / h);
        const double dphij = (j == e ? -1.0 : 1.0) / h;
        for (int q = 0; q < 2; ++q) {
          const double phid = (d == e) ? 1.0 - xi[q] : xi[q];
          const double phij = (j == e) ? 1.0 - xi[q] : xi[q];
          const double vq = vl * (1.0 - xi[q]) + vr * xi[q];
          ja += w[q] * h * phid * (phij * dv + vq * dphij);
        }
      }
      jv[p++] = (B.nu * stiff_ij(B, d, j) + ja) + inv_dt * mass_ij(B, d, j);
    }
  }
}

// ---- Allen-Cahn weak residual, implicit Euler, lumped cubic -----------------
// r_s = M(u_{s+1} − u_s)/Δt + (ε² K u_{s+1} + M̃(u_{s+1}³ − u_{s+1})), the
// restatement in oracle/ref_capi.cpp (burgers_fem_residual layout,
// residual.hpp:244-382; lumped reaction as residual.hpp:431-441), slack
// columns masked. M, K: CSR rows on the stencil (ascending columns).
__global__ void k_ac_res(AcDev A, const double* __restrict__ u, double* __restrict__ f) {
  const int nrow = (A.nt - 1) * A.nk;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < nrow; row += gridDim.x * blockDim.x) {
    const int s = row / A.nk, d = A.kept[row - s * A.nk];
    const double* u0 = u + static_cast<i64>(s) * A.ns;
    const double* u1 = u0 + A.ns;
    double mdu = 0.0, ku = 0.0;
    for (i64 p = A.rp[d]; p < A.rp[d + 1]; ++p) {
      const int j = A.ci[p];
      if (A.slack[j]) continue;
      mdu += A.mv[p] * (u1[j] - u0[j]);
      ku += A.kv[p] * u1[j];
    }
    const double v = u1[d];
    f[row] = mdu / A.dt[s] + (A.eps2 * ku + A.ml[d] * (v * v * v - v));
  }
}

// J row (s, d): slice s → −M/Δt; slice s+1 → (M/Δt + ε² K) + M̃(3u² − 1) on the
// diagonal (the oracle restatement's triplet order, oracle/ref_capi.cpp).
__global__ void k_ac_jac(AcDev A, const double* __restrict__ u, const i64* __restrict__ jrp,
                         double* __restrict__ jv) {
  const int nrow = (A.nt - 1) * A.nk;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < nrow; row += gridDim.x * blockDim.x) {
    const int s = row / A.nk, d = A.kept[row - s * A.nk];
    i64 q = jrp[row];
    for (i64 p = A.rp[d]; p < A.rp[d + 1]; ++p)
      if (!A.slack[A.ci[p]]) jv[q++] = -A.mv[p] / A.dt[s];
    const double v = u[static_cast<i64>(s + 1) * A.ns + d];
    for (i64 p = A.rp[d]; p < A.rp[d + 1]; ++p) {
      const int j = A.ci[p];
      if (A.slack[j]) continue;
      double x = A.mv[p] / A.dt[s] + A.eps2 * A.kv[p];
      if (j == d) x += A.ml[d] * (3.0 * v * v - 1.0);
      jv[q++] = x;
    }
  }
}

__global__ void k_ic_rhs(int ns, const double* __restrict__ u0, double lam, double* __restrict__ rhs) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < ns; d += gridDim.x * blockDim.x)
    rhs[d] = lam * u0[d];
}

int grid_for(i64 n, int threads = 256) {
  return static_cast<int>(std::max<i64>(1, std::min<i64>((n + threads - 1) / threads, 148 * 16)));
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

SpaceTimePosterior::SpaceTimePosterior(const SpaceTimeSpec& spec, cudaStream_t stream,
                                       const PartitionSpec* part)
    : spec_(spec), stream_(stream) {
  if (part) pspec_ = *part;
  double t0 = now_ms();
  build_host();
  times_.setup_host_ms = now_ms() - t0;
  t0 = now_ms();
  assemble_device();
  cuda_check(cudaStreamSynchronize(stream_), "assemble");
  times_.assemble_ms = now_ms() - t0;
}

SpaceTimePosterior::SpaceTimePosterior(const SpaceTimeSpec& spec, HostOnly)
    : spec_(spec), stream_(nullptr), host_only_(true) {
  build_host();
}

std::shared_ptr<const Symbolic> SpaceTimePosterior::host_symbolic(const SpaceTimeSpec& spec) {
  SpaceTimePosterior p(spec, HostOnly{});
  return p.sym_;
}

SpaceTimePosterior::~SpaceTimePosterior() {
  for (cudaEvent_t e : ev_)
    if (e) cudaEventDestroy(e);
}

void SpaceTimePosterior::build_host() {
  require(spec_.n_el >= 2 && spec_.n_t >= 2, kContract, "spacetime: need >= 2 elements and slices");
  require(spec_.dim == 1 || spec_.dim == 2, kContract, "spacetime: dim must be 1 or 2");
  require(spec_.residual >= 0 && spec_.residual <= 2, kContract, "spacetime: unknown residual");
  require(spec_.dim == 1 || (spec_.residual != 1 && spec_.advection == 0.0 && !spec_.dirichlet),
          kContract, "spacetime: 2-D supports the heat proxy, natural BC, linear/Allen-Cahn residuals");
  double t_stage = now_ms();
  auto stage = [&](const char* what) {  // GMRF_VERBOSE: host setup time per stage
    if (std::getenv("GMRF_VERBOSE")) {
      const double t = now_ms();
      std::fprintf(stderr, "[gmrf] host setup: %-28s %8.1f ms\n", what, t - t_stage);
      t_stage = t;
    }
  };
  // element assembly, lumping and constraint folding on the device (fem_device.cu);
  // the device-free planning path (host_symbolic) keeps the host loops: it only
  // needs the patterns
  std::unique_ptr<FemDeviceScope> fem_scope;
  if (!host_only_) fem_scope = std::make_unique<FemDeviceScope>();
  if (spec_.dim == 1) {
    space_ = Space1D{spec_.n_el, spec_.xa, spec_.xb};
    ops_ = host_only_ ? spatial_ops(space_, spec_.diffusion, spec_.advection, spec_.dirichlet)
                      : spatial_ops_device(space_, spec_.diffusion, spec_.advection,
                                           spec_.dirichlet, stream_);
  } else {
    ops_ = host_only_ ? spatial_ops(Space2D{spec_.n_el}, spec_.diffusion)
                      : spatial_ops_device(Space2D{spec_.n_el}, spec_.diffusion, stream_);
  }
  ns_ = ops_.n;
  nt_ = spec_.n_t;
  n_ = ns_ * nt_;
  tg_.resize(nt_);
  for (int i = 0; i < nt_; ++i)
    tg_[i] = spec_.t_end * static_cast<double>(i) / static_cast<double>(nt_ - 1);
  dts_.resize(nt_ - 1);
  tstep_.resize(nt_ - 1);
  sqt_.resize(nt_ - 1);
  for (int i = 0; i + 1 < nt_; ++i) {
    dts_[i] = tg_[i + 1] - tg_[i];
    tstep_[i] = 1.0 / (dts_[i] * spec_.tau * spec_.tau);
    sqt_[i] = std::sqrt(tstep_[i]);
  }
  // uniform grid: the spatial blocks use the first step's Δt (spatiotemporal.hpp:114-126)
  blk_ = spacetime_blocks(ops_, dts_[0], spec_.tau, spec_.noise, spec_.init, spec_.eps);
  const auto& sl = blk_.slack;
  // spatial coupling stencil (P1 element adjacency = the mass pattern)
  Csc stencil = ops_.mass;

  stage("spatial blocks");
  // ---- templates: spatial patterns of the diagonal / upper off-diagonal blocks
  // (every prior block, plus stencil² which carries JᵀΛJ of a residual whose
  // rows couple the stencil of a DoF in two consecutive slices)
  auto pat = [](Csc m) {
    for (double& v : m.v) v = 1.0;
    return m;
  };
  const Csc st2 = pat(multiply(pat(stencil), pat(stencil)));
  Csc dg = st2;
  for (const Csc* m : {&blk_.c_mm, &blk_.c_gg, &blk_.q1, &blk_.g_mm, &blk_.g_ff, &blk_.g_l1})
    dg = add(dg, pat(*m));
  Csc up = st2;
  for (const Csc* m : {&blk_.c_mg, &blk_.g_mf}) up = add(up, pat(*m));
  Csc lo = transpose(up);

  // ---- master pattern (full symmetric, original joint indices)
  pcp_.assign(n_ + 1, 0);
  pri_.clear();
  pri_.reserve(static_cast<size_t>(n_) * (dg.nnz() / ns_ + 2 * up.nnz() / ns_ + 1));
  for (int s = 0; s < nt_; ++s)
    for (int b = 0; b < ns_; ++b) {
      const int C = s * ns_ + b;
      if (sl[b]) {
        pri_.push_back(C);
      } else {
        if (s >= 1)
          for (i64 p = up.cp[b]; p < up.cp[b + 1]; ++p)
            if (!sl[up.ri[p]]) pri_.push_back((s - 1) * ns_ + up.ri[p]);
        for (i64 p = dg.cp[b]; p < dg.cp[b + 1]; ++p)
          if (!sl[dg.ri[p]]) pri_.push_back(s * ns_ + dg.ri[p]);
        if (s < nt_ - 1)
          for (i64 p = lo.cp[b]; p < lo.cp[b + 1]; ++p)
            if (!sl[lo.ri[p]]) pri_.push_back((s + 1) * ns_ + lo.ri[p]);
      }
      pcp_[C + 1] = static_cast<i64>(pri_.size());
    }

  stage("master pattern");
  // ---- symbolic: geometric nested dissection of the space-time grid (separator
  // thickness = the coupling radii of the pattern), shared by every
  // factorization of the run
  {
    const int nx = spec_.dim == 1 ? ns_ : spec_.n_el + 1, ny = ns_ / nx;
    int rx = 1, ry = 1, rt = 1;
    for (int C = 0; C < n_; ++C)
      for (i64 p = pcp_[C]; p < pcp_[C + 1]; ++p) {
        const int R = pri_[p], dr = R % ns_, dc = C % ns_;
        rx = std::max(rx, std::abs(dr % nx - dc % nx));
        ry = std::max(ry, std::abs(dr / nx - dc / nx));
        rt = std::max(rt, std::abs(R / ns_ - C / ns_));
      }
    std::vector<char> first(static_cast<size_t>(n_), 0);
    for (int s = 0; s < nt_; ++s)
      for (int d = 0; d < ns_; ++d) first[static_cast<size_t>(s) * ns_ + d] = sl[d];
    if (std::getenv("GMRF_VERBOSE"))
      std::fprintf(stderr, "[gmrf] spacetime grid %d x %d x %d, coupling radii %d %d %d\n", nx, ny, nt_, rx, ry, rt);
    std::vector<i32> perm = grid_nd_order3(nx, ny, nt_, rx, ry, rt, first);
    SymbolicOptions opt;
    opt.postorder_given = true;
    sym_ = std::make_shared<const Symbolic>(analyze(n_, pcp_.data(), pri_.data(), perm.data(), opt));
  }

  stage("ordering + symbolic");
  // ---- S_cond = [S_prior | Aᵀ L_ε] (gmrf.hpp:165), CSC, columns in the reference order
  s_ = Csc{};
  s_.nr = n_;
  s_.cp.assign(1, 0);
  auto push_col = [&](int slice, const Csc& m, int k, double scale) {
    for (i64 p = m.cp[k]; p < m.cp[k + 1]; ++p)
      if (!sl[m.ri[p]]) {
        s_.ri.push_back(slice * ns_ + m.ri[p]);
        s_.v.push_back(scale * m.v[p]);
      }
  };
  for (int k = 0; k < ns_; ++k) {
    push_col(0, blk_.l1, k, 1.0);
    s_.cp.push_back(s_.nnz());
  }
  for (int i = 0; i + 1 < nt_; ++i)
    for (int k = 0; k < ns_; ++k) {
      push_col(i, blk_.s_m, k, sqt_[i]);
      push_col(i + 1, blk_.f_is, k, -sqt_[i]);
      s_.cp.push_back(s_.nnz());
    }
  for (int d = 0; d < ns_; ++d)
    if (sl[d])
      for (int s = 0; s < nt_; ++s) {
        s_.ri.push_back(s * ns_ + d);
        s_.v.push_back(1.0 / std::sqrt(spec_.eps));
        s_.cp.push_back(s_.nnz());
      }
  for (int d = 0; d < ns_; ++d) {  // IC: Aᵀ L_ε = √Λ on slice 0
    s_.ri.push_back(d);
    s_.v.push_back(std::sqrt(spec_.ic_noise_prec));
    s_.cp.push_back(s_.nnz());
  }
  s_.nc = static_cast<i32>(s_.cp.size()) - 1;
  ms_ = s_.nc;

  stage("square-root pattern");
  // ---- residual Jacobian pattern (CSR rows, then CSC with a value map): row
  // (step s, kept DoF d) couples the stencil of d in slices s and s+1, slack
  // columns skipped (residual.hpp:353-377)
  if (spec_.residual != 0) {
    std::vector<int> kept;
    for (int d = 0; d < ns_; ++d)
      if (!sl[d]) kept.push_back(d);
    const int nk = static_cast<int>(kept.size());
    nres_ = (nt_ - 1) * nk;
    jrp_.assign(nres_ + 1, 0);
    jci_.clear();
    for (int s = 0; s + 1 < nt_; ++s)
      for (int k = 0; k < nk; ++k) {
        const int d = kept[k];
        for (int sl2 = s; sl2 <= s + 1; ++sl2)
          for (i64 p = stencil.cp[d]; p < stencil.cp[d + 1]; ++p)
            if (!sl[stencil.ri[p]]) jci_.push_back(sl2 * ns_ + stencil.ri[p]);
        jrp_[s * nk + k + 1] = static_cast<i64>(jci_.size());
      }
    jcp_.assign(n_ + 1, 0);
    for (i32 c : jci_) jcp_[c + 1]++;
    for (int c = 0; c < n_; ++c) jcp_[c + 1] += jcp_[c];
    jri_.resize(jci_.size());
    jmap_.resize(jci_.size());
    std::vector<i64> nx(jcp_.begin(), jcp_.end() - 1);
    for (int r = 0; r < nres_; ++r)
      for (i64 p = jrp_[r]; p < jrp_[r + 1]; ++p) {
        i64 q = nx[jci_[p]]++;
        jri_[q] = r;
        jmap_[q] = p;
      }
  }
}

void SpaceTimePosterior::assemble_device() {
  double t_stage = now_ms();
  auto stage = [&](const char* what) {  // GMRF_VERBOSE: device setup time per stage
    if (std::getenv("GMRF_VERBOSE")) {
      cudaStreamSynchronize(stream_);
      const double t = now_ms();
      std::fprintf(stderr, "[gmrf] device setup: %-26s %8.1f ms\n", what, t - t_stage);
      t_stage = t;
    }
  };
  const auto& sl = blk_.slack;
  d_pcp_.upload(pcp_, stream_);
  d_pri_.upload(pri_, stream_);
  // spatial blocks, concatenated
  std::vector<i64> bcp;
  std::vector<i32> bri;
  std::vector<double> bv;
  const Csc* blocks[kNumBlk] = {&blk_.c_mm, &blk_.c_gg, &blk_.c_mg, &blk_.q1,
                                &blk_.g_mm, &blk_.g_ff, &blk_.g_mf, &blk_.g_l1};
  for (const Csc* m : blocks) {
    const i64 off = static_cast<i64>(bri.size());
    for (i64 v : m->cp) bcp.push_back(off + v);
    bri.insert(bri.end(), m->ri.begin(), m->ri.end());
    bv.insert(bv.end(), m->v.begin(), m->v.end());
  }
  d_blk_cp_.upload(bcp, stream_);
  d_blk_ri_.upload(bri, stream_);
  d_blk_v_.upload(bv, stream_);
  d_slack_.upload(std::vector<char>(sl.begin(), sl.end()), stream_);
  const i64 np = static_cast<i64>(pri_.size());
  d_qcond_.alloc(np);
  d_qeff_.alloc(np);
  d_tstep_.upload(tstep_, stream_);
  d_dts_.upload(dts_, stream_);
  if (spec_.dim == 1) {
    std::vector<double> xn(ns_);
    for (int d = 0; d < ns_; ++d) xn[d] = space_.x(d);
    d_xn_.upload(xn, stream_);
  }
  // S_cond: CSC (columns, for Sᵀx) and CSR (rows, for S w)
  d_scp_.upload(s_.cp, stream_);
  d_sri_.upload(s_.ri, stream_);
  d_sv_.upload(s_.v, stream_);
  // q_eff = sym(S Sᵀ) (gauss_newton.hpp:112-113): Gram product of Sᵀ, whose rows
  // are S's columns, over the master pattern
  stage("uploads");
  gram_s_ = std::make_unique<GramPlan>(n_, pcp_.data(), pri_.data(), ms_, s_.cp.data(),
                                       s_.ri.data(), nullptr, stream_);
  stage("Gram plan S S^T");
  assemble_values();
  Csc sr = transpose(s_);
  d_srp_.upload(sr.cp, stream_);
  d_sci_.upload(sr.ri, stream_);
  d_svr_.upload(sr.v, stream_);
  if (spec_.residual == 2) {  // spatial M, K rows on the stencil + lumped mass
    const Csc& m = ops_.mass;
    std::vector<double> kv(m.ri.size(), 0.0);
    for (i32 j = 0; j < m.nc; ++j)
      for (i64 p = m.cp[j]; p < m.cp[j + 1]; ++p) kv[p] = ops_.lap.at(m.ri[p], j);
    d_mrp_.upload(m.cp, stream_);
    d_mci_.upload(m.ri, stream_);
    d_mv_.upload(m.v, stream_);
    d_kv_.upload(kv, stream_);
    d_ml_.upload(lumped_mass(m), stream_);
  }
  if (spec_.residual != 0) {
    // JᵀΛJ over the entries the factorization reads (qmap >= 0), written into the panels
    std::vector<char> need(pri_.size());
    for (size_t p = 0; p < need.size(); ++p) need[p] = sym_->qmap[p] >= 0;
    stage("assembly + S rows");
    gram_j_ = std::make_unique<GramPlan>(n_, pcp_.data(), pri_.data(), nres_, jrp_.data(),
                                         jci_.data(), &need, stream_);
    stage("Gram plan J^T J");
    d_lam_.upload(std::vector<double>(nres_, spec_.pde_noise_prec), stream_);
    d_wf_.alloc(std::max(nres_, 1));
    d_jrp_.upload(jrp_, stream_);
    d_jci_.upload(jci_, stream_);
    d_jcp_.upload(jcp_, stream_);
    d_jri_.upload(jri_, stream_);
    d_jmap_.upload(jmap_, stream_);
    d_jv_.alloc(std::max<size_t>(jci_.size(), 1));
    std::vector<i32> kept;
    for (int d = 0; d < ns_; ++d)
      if (!sl[d]) kept.push_back(d);
    kept_.upload(kept, stream_);
  }
  if (std::getenv("GMRF_VERBOSE"))
    std::fprintf(stderr, "[gmrf] spacetime n %d pattern nnz %zu, JtJ pairs %lld, SSt pairs %lld, nnz(L) %lld\n",
                 n_, pri_.size(), static_cast<long long>(gram_j_ ? gram_j_->pairs() : 0),
                 static_cast<long long>(gram_s_->pairs()),
                 static_cast<long long>(sym_->nnz_l_padded));
  stage("Jacobian uploads");
  fac_ = std::make_unique<DeviceFactor>(sym_, stream_, pspec_.nranks > 1 ? &pspec_ : nullptr);
  stage("factor plan + storage");
  auto mem = [&](const char* what) {
    if (!std::getenv("GMRF_VERBOSE")) return;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    std::fprintf(stderr, "[gmrf] after %s: device free %.1f of %.1f GB\n", what, fr * 1e-9, tot * 1e-9);
  };
  mem("factor storage");
  fac_->set_selinv_inplace(true);  // variances are the last use of each factorization
  fac_->prepare_selinv();
  stage("selected-inversion plan");
  mem("selected-inversion storage");
  fac_->set_profiler(&prof_);
  for (DevBuf<double>* v : {&mean_cond_, &mean_, &var_, &x_, &c_, &g_, &d_, &cand_, &r1_, &u0_})
    v->alloc(std::max(n_, 1));
  w_.alloc(std::max(ms_, 1));
  f_.alloc(std::max(nres_, 1));
  fc_.alloc(std::max(nres_, 1));
  part_.alloc(2 * (kDotBlocks + 1));
}

// Row 1: joint prior (Q_cond) and q_eff = sym(S Sᵀ) values on the master pattern (device).
void SpaceTimePosterior::assemble_values() {
  BlkDev b{d_blk_cp_.p, d_blk_ri_.p, d_blk_v_.p, ns_};
  const double np = static_cast<double>(pri_.size());
  // algorithmic bytes: write Q_cond (8 B/entry) + pattern (4 B/entry + 8 B/column)
  prof_.run(stream_, "assemble.prior", 0.0, 12.0 * np + 8.0 * n_, [&] {
    k_st_assemble<<<grid_for(n_), 256, 0, stream_>>>(d_pcp_.p, d_pri_.p, n_, ns_, nt_, d_tstep_.p,
                                                    1.0 / spec_.eps, spec_.ic_noise_prec,
                                                    d_slack_.p, b, d_qcond_.p);
  });
  prof_.run(stream_, "assemble.q_eff", 0.0, gram_s_->bytes(false, true, false), [&] {
    gram_s_->apply(d_sv_.p, nullptr, 1.0, nullptr, d_qeff_.p, nullptr, nullptr, stream_);
  });
  times_.kernel_launches += 1 + gram_s_->launches(false);
}

double SpaceTimePosterior::dot(const double* a, const double* b, i64 n) {
  k_dot_partial<<<kDotBlocks, kDotThreads, 0, stream_>>>(n, a, b, part_.p);
  k_dot_final<<<1, 512, 0, stream_>>>(part_.p, part_.p + kDotBlocks);
  times_.kernel_launches += 2;
  double out = 0.0;
  cuda_check(cudaMemcpyAsync(&out, part_.p + kDotBlocks, sizeof(double), cudaMemcpyDeviceToHost,
                             stream_),
             "dot");
  cuda_check(cudaStreamSynchronize(stream_), "dot");
  return out;
}

// Residual rows and Jacobian values (HBM-bound: the state slices s, s+1 of
// each row's stencil read, one value written per row / per J entry).
void SpaceTimePosterior::eval_residual(const double* d_u, double* d_f) {
  const double bytes = 8.0 * nres_ + 16.0 * n_;
  prof_.run(stream_, "residual.eval", 0.0, bytes, [&] {
    if (spec_.residual == 2) {
      k_ac_res<<<grid_for(nres_), 256, 0, stream_>>>(ac_dev(), d_u, d_f);
    } else {
      BurgersDev B{ns_, nt_, static_cast<int>(kept_.n), spec_.diffusion, d_xn_.p, d_dts_.p,
                   d_slack_.p, kept_.p};
      k_burgers_res<<<grid_for(nres_), 256, 0, stream_>>>(B, d_u, d_f);
    }
  });
  times_.kernel_launches += 1;
}

void SpaceTimePosterior::eval_jacobian(const double* d_u) {
  const double bytes = 8.0 * static_cast<double>(jci_.size()) + 8.0 * nres_ + 16.0 * n_;
  prof_.run(stream_, "residual.jacobian", 0.0, bytes, [&] {
    if (spec_.residual == 2) {
      k_ac_jac<<<grid_for(nres_), 256, 0, stream_>>>(ac_dev(), d_u, d_jrp_.p, d_jv_.p);
    } else {
      BurgersDev B{ns_, nt_, static_cast<int>(kept_.n), spec_.diffusion, d_xn_.p, d_dts_.p,
                   d_slack_.p, kept_.p};
      k_burgers_jac<<<grid_for(nres_), 256, 0, stream_>>>(B, d_u, d_jrp_.p, d_jv_.p);
    }
  });
  times_.kernel_launches += 1;
}

void SpaceTimePosterior::residual(const double* d_u, double* d_r) { eval_residual(d_u, d_r); }

AcDev SpaceTimePosterior::ac_dev() const {
  return AcDev{ns_, nt_, static_cast<int>(kept_.n), d_dts_.p, spec_.diffusion,
               d_slack_.p, kept_.p, d_mrp_.p, d_mci_.p, d_mv_.p, d_kv_.p, d_ml_.p};
}

// ½‖Sᵀ(x−μ)‖² + ½ Σ λ (y − f)², y = 0 (gauss_newton.hpp:65-83); both sums
// are read back with one host synchronization
double SpaceTimePosterior::objective(const double* d_x, const double* d_fx) {
  k_axpby<<<grid_for(n_), 256, 0, stream_>>>(n_, 1.0, d_x, -1.0, mean_cond_.p, c_.p);
  k_spmv<<<grid_for(ms_), 256, 0, stream_>>>(ms_, d_scp_.p, d_sri_.p, d_sv_.p, nullptr, c_.p, w_.p);
  times_.kernel_launches += 2;
  if (nres_ == 0) return 0.5 * dot(w_.p, w_.p, ms_);
  double* p2 = part_.p + kDotBlocks + 1;
  k_dot_partial<<<kDotBlocks, kDotThreads, 0, stream_>>>(ms_, w_.p, w_.p, part_.p);
  k_dot_final<<<1, 512, 0, stream_>>>(part_.p, part_.p + kDotBlocks);
  k_dot_partial<<<kDotBlocks, kDotThreads, 0, stream_>>>(nres_, d_fx, d_fx, p2);
  k_dot_final<<<1, 512, 0, stream_>>>(p2, p2 + kDotBlocks);
  times_.kernel_launches += 4;
  double ww = 0.0, ff = 0.0;
  cuda_check(cudaMemcpyAsync(&ww, part_.p + kDotBlocks, sizeof(double), cudaMemcpyDeviceToHost,
                             stream_),
             "objective");
  cuda_check(cudaMemcpyAsync(&ff, p2 + kDotBlocks, sizeof(double), cudaMemcpyDeviceToHost, stream_),
             "objective");
  cuda_check(cudaStreamSynchronize(stream_), "objective");
  return 0.5 * ww + 0.5 * (spec_.pde_noise_prec * ff);
}

void SpaceTimePosterior::fill_panels(const double* base, bool with_jacobian) {
  fac_->begin_numeric();
  if (with_jacobian) {
    // H = sym(base + Jᵀ Λ J) straight into the panels (gauss_newton.hpp:137-138, :231-232)
    prof_.run(stream_, "update.h_jtlj", 0.0, gram_j_->bytes(true, false, true), [&] {
      gram_j_->apply(d_jv_.p, d_lam_.p, 1.0, base, nullptr, fac_->d_qmap(), fac_->d_l(), stream_);
    });
    times_.kernel_launches += gram_j_->launches(true);
    return;
  }
  // base + pattern + qmap (20 B/entry) read, lower-half L writes (4 B/entry)
  const double np = static_cast<double>(pri_.size());
  prof_.run(stream_, "update.q_base", 0.0, 24.0 * np, [&] {
    k_fill_panels<<<grid_for(n_), 256, 0, stream_>>>(d_pcp_.p, d_pri_.p, n_, fac_->d_qmap(), base,
                                                     nullptr, d_jri_.p, d_jmap_.p, d_jv_.p,
                                                     spec_.pde_noise_prec, fac_->d_l());
  });
  times_.kernel_launches += 1;
}

std::vector<GnIter> SpaceTimePosterior::run(const double* u0, const GnConfig& cfg, bool variances) {
  require(cfg.max_iters >= 1, kContract, "gauss-newton: max_iters must be >= 1");
  require(cfg.decrement_tol > 0.0, kContract, "gauss-newton: decrement_tol must be positive");
  require(cfg.armijo_c > 0.0 && cfg.armijo_c < 1.0, kContract, "gauss-newton: armijo constant in (0,1)");
  require(cfg.shrink > 0.0 && cfg.shrink < 1.0, kContract, "gauss-newton: shrink factor in (0,1)");
  std::vector<GnIter>& trace = trace_;
  trace.clear();
  converged_ = false;
  {
    const double setup = times_.setup_host_ms, init = times_.assemble_ms;
    times_ = PhaseTimes{};
    times_.setup_host_ms = setup;
    times_.init_ms = init;
  }
  if (!ev_[0])
    for (cudaEvent_t& e : ev_) cuda_check(cudaEventCreate(&e), "event");
  cudaEvent_t e0 = ev_[0], e1 = ev_[1];
  auto phase = [&](double& acc, auto&& body) {
    cudaEventRecord(e0, stream_);
    body();
    cudaEventRecord(e1, stream_);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    acc += ms;
  };
  // rhs: the system's right-hand side, whose forward sweep rides along with the
  // factorization (DeviceFactor::factor_panels); solve_pending finishes it
  auto factor_now = [&](const char* what, const double* rhs = nullptr) {
    cudaEvent_t a = ev_[2], b = ev_[3];
    cudaEventRecord(a, stream_);
    int32_t bad = fac_->factor_panels(rhs);
    cudaEventRecord(b, stream_);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    times_.numeric_ms += ms;
    times_.n_factorizations += 1;
    if (!rhs) {
      times_.numeric_pure_ms += ms;
      times_.n_pure_factorizations += 1;
    }
    times_.kernel_launches += fac_->launches_numeric();
    if (bad >= 0)
      throw Error(kNotSpd, std::string(what) + ": cholesky: non-positive pivot at index " +
                               std::to_string(bad));
  };

  // ---- prior + q_eff assembly on the device (spatiotemporal.hpp:79-195) ----
  phase(times_.assemble_ms, [&] { assemble_values(); });

  // ---- IC conditioning (condition_affine, gmrf.hpp:145-170) ----
  phase(times_.condition_ms, [&] {
    cuda_check(cudaMemcpyAsync(u0_.p, u0, ns_ * sizeof(double), cudaMemcpyHostToDevice, stream_),
               "u0");
    cuda_check(cudaMemsetAsync(r1_.p, 0, n_ * sizeof(double), stream_), "rhs");
    k_ic_rhs<<<grid_for(ns_), 256, 0, stream_>>>(ns_, u0_.p, spec_.ic_noise_prec, r1_.p);
    fill_panels(d_qcond_.p, false);
    factor_now("conditioning", r1_.p);
    fac_->solve_pending(mean_cond_.p);
    times_.kernel_launches += 1 + fac_->launches_solve();
  });

  if (spec_.residual == 0) {
    cuda_check(cudaMemcpyAsync(mean_.p, mean_cond_.p, n_ * sizeof(double), cudaMemcpyDeviceToDevice,
                               stream_),
               "mean");
    if (variances)
      phase(times_.selinv_ms, [&] {
        fac_->selinv(var_.p, true);
        times_.kernel_launches += fac_->launches_selinv();
      });
    return trace;
  }

  // ---- Gauss-Newton (gauss_newton.hpp:93-224) ----
  double t_gn0 = now_ms();
  cuda_check(cudaMemcpyAsync(x_.p, mean_cond_.p, n_ * sizeof(double), cudaMemcpyDeviceToDevice,
                             stream_),
             "x0");
  const double lam = spec_.pde_noise_prec;
  // the accepted line-search candidate's residual and objective are the next
  // iterate's (same buffers, same kernels): carried over instead of recomputed
  bool carried = false;
  double obj_carry = 0.0;
  for (int iter = 1; iter <= cfg.max_iters; ++iter) {
    if (!carried) eval_residual(x_.p, f_.p);
    eval_jacobian(x_.p);
    // grad = S(Sᵀ(x−μ)) − Jᵀ Λ (y − f)    (y = 0)
    k_axpby<<<grid_for(n_), 256, 0, stream_>>>(n_, 1.0, x_.p, -1.0, mean_cond_.p, c_.p);
    k_spmv<<<grid_for(ms_), 256, 0, stream_>>>(ms_, d_scp_.p, d_sri_.p, d_sv_.p, nullptr, c_.p, w_.p);
    k_spmv<<<grid_for(n_), 256, 0, stream_>>>(n_, d_srp_.p, d_sci_.p, d_svr_.p, nullptr, w_.p, g_.p);
    // weighted = Λ (y − f) with y = 0; grad −= Jᵀ weighted (gauss_newton.hpp:126-130)
    k_weighted_misfit<<<grid_for(nres_), 256, 0, stream_>>>(nres_, lam, f_.p, d_wf_.p);
    k_spmv<<<grid_for(n_), 256, 0, stream_>>>(n_, d_jcp_.p, d_jri_.p, d_jv_.p, d_jmap_.p, d_wf_.p,
                                              r1_.p);
    k_axpby<<<grid_for(n_), 256, 0, stream_>>>(n_, 1.0, g_.p, -1.0, r1_.p, g_.p);
    k_axpby<<<grid_for(n_), 256, 0, stream_>>>(n_, -1.0, g_.p, 0.0, g_.p, r1_.p);  // rhs = −grad
    times_.kernel_launches += 7;
    fill_panels(d_qeff_.p, true);
    factor_now("gauss-newton", r1_.p);
    fac_->solve_pending(d_.p);
    times_.kernel_launches += fac_->launches_solve();
    const double gd = dot(g_.p, d_.p, n_);
    const double decrement = std::sqrt(std::max(0.0, -gd));
    const double obj = carried ? obj_carry : objective(x_.p, f_.p);
    GnIter rec{iter, obj, decrement, 0.0, 0};
    if (decrement < cfg.decrement_tol || 0.5 * decrement * decrement <= 1e-14 * (1.0 + std::abs(obj))) {
      trace.push_back(rec);
      converged_ = true;
      break;
    }
    const double slope = gd;
    double alpha = 1.0;
    int bt = 0;
    while (true) {
      k_axpby<<<grid_for(n_), 256, 0, stream_>>>(n_, 1.0, x_.p, alpha, d_.p, cand_.p);
      eval_residual(cand_.p, fc_.p);
      times_.kernel_launches += 1;
      const double cobj = objective(cand_.p, fc_.p);
      if (cobj <= obj + cfg.armijo_c * alpha * slope) {
        std::swap(x_.p, cand_.p);
        std::swap(f_.p, fc_.p);
        obj_carry = cobj;
        carried = true;
        break;
      }
      if (++bt > cfg.max_backtracks) {
        trace.push_back(rec);
        throw Error(kNumerical, "gauss-newton: line search failed after " + std::to_string(bt - 1) +
                                    " backtracks at iteration " + std::to_string(iter));
      }
      alpha *= cfg.shrink;
    }
    rec.step_size = alpha;
    rec.backtracks = bt;
    trace.push_back(rec);
  }
  cuda_check(cudaStreamSynchronize(stream_), "gn");
  times_.gn_ms += now_ms() - t_gn0;

  // ---- Laplace posterior (gauss_newton.hpp:228-240): Q_cond + J(mode)ᵀΛJ(mode) ----
  phase(times_.laplace_ms, [&] {
    eval_jacobian(x_.p);
    fill_panels(d_qcond_.p, true);
    factor_now("laplace");
    cuda_check(cudaMemcpyAsync(mean_.p, x_.p, n_ * sizeof(double), cudaMemcpyDeviceToDevice, stream_),
               "mode");
  });
  if (variances)
    phase(times_.selinv_ms, [&] {
      fac_->selinv(var_.p, true);
      times_.kernel_launches += fac_->launches_selinv();
    });
  return trace;
}

void SpaceTimePosterior::copy_pattern(std::vector<i64>& cp, std::vector<i32>& ri) const {
  cp = pcp_;
  ri = pri_;
}

void SpaceTimePosterior::copy_values(std::vector<double>& qcond, std::vector<double>& qeff) const {
  qcond.resize(d_qcond_.n);
  qeff.resize(d_qeff_.n);
  cuda_check(cudaMemcpy(qcond.data(), d_qcond_.p, qcond.size() * 8, cudaMemcpyDeviceToHost), "q");
  cuda_check(cudaMemcpy(qeff.data(), d_qeff_.p, qeff.size() * 8, cudaMemcpyDeviceToHost), "q");
}

void SpaceTimePosterior::jacobian_csr(const double* d_u, std::vector<i64>& rp,
                                      std::vector<i32>& ci, std::vector<double>& v) {
  eval_jacobian(d_u);
  rp = jrp_;
  ci = jci_;
  v.resize(jci_.size());
  cuda_check(cudaMemcpyAsync(v.data(), d_jv_.p, v.size() * 8, cudaMemcpyDeviceToHost, stream_), "J");
  cuda_check(cudaStreamSynchronize(stream_), "J");
}

}  // namespace gmrf
