// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" wrapper around the UNMODIFIED reference headers
// (/root/reference/proj/include/gmrfpde/**, header-only C++20). Built by
// oracle/Makefile into oracle/_ref/libgmrfref.so; only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference legs load it, always as the
// checker or the CPU baseline, never as the thing measured or shipped.
//
// The reference's Index is int (core/types.hpp:12), so every CSC crossing this
// wrapper uses int32 col_ptr/row_idx — exactly the reference layout
// (core/sparse.hpp:25-61).
//
// Problem builders follow SURVEY.md §8(d)'s pinned draw order.

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "gmrfpde/core/amd.hpp"
#include "gmrfpde/core/cg.hpp"
#include "gmrfpde/core/cholesky.hpp"
#include "gmrfpde/core/rng.hpp"
#include "gmrfpde/core/sparse.hpp"
#include "gmrfpde/core/takahashi.hpp"

#ifdef GMRF_ORDERING_PROBE
// Ordering-floor probe build (oracle/_ref/libgmrfref_nd.so, same source): the
// unmodified reference headers with the fill-reducing ordering that the chain
// uses — amd_order in gauss_newton.hpp:139 and the AMD inside
// cholesky_factor(q) at gmrf.hpp:55,160 — redirected to METIS nested
// dissection. The reference's own algorithms then run with another elimination
// order; how far their outputs move (tests/golden/make_golden_full.py floor:*)
// is the reference's FP64 ordering floor, SURVEY §8(c).
extern "C" int METIS_NodeND(int64_t* nvtxs, int64_t* xadj, int64_t* adjncy, int64_t* vwgt,
                            int64_t* options, int64_t* perm, int64_t* iperm);
namespace gmrfpde {
inline std::vector<Index> nd_probe_order(const SparseMatrixCSC& a) {
  const int64_t n = a.ncols;
  std::vector<int64_t> xadj(n + 1, 0), adj;
  for (Index j = 0; j < a.ncols; ++j) {
    for (Index p = a.col_ptr[j]; p < a.col_ptr[j + 1]; ++p)
      if (a.row_idx[p] != j) adj.push_back(a.row_idx[p]);
    xadj[j + 1] = static_cast<int64_t>(adj.size());
  }
  std::vector<int64_t> perm(n), iperm(n);
  int64_t nv = n;
  if (METIS_NodeND(&nv, xadj.data(), adj.data(), nullptr, nullptr, perm.data(), iperm.data()) != 1)
    throw NumericalError("METIS_NodeND failed");
  return std::vector<Index>(perm.begin(), perm.end());  // new -> old, as amd_order
}
inline CholeskyFactor cholesky_factor_probe(const SparseMatrixCSC& q) {
  return cholesky_factor(q, nd_probe_order(q));
}
inline CholeskyFactor cholesky_factor_probe(const SparseMatrixCSC& q, const std::vector<Index>& p) {
  return cholesky_factor(q, p);
}
}  // namespace gmrfpde
#define amd_order nd_probe_order
#define cholesky_factor cholesky_factor_probe
#endif

#include "gmrfpde/fem/assembly.hpp"
#include "gmrfpde/fem/constraints.hpp"
#include "gmrfpde/fem/mesh.hpp"
#include "gmrfpde/fem/space.hpp"
#include "gmrfpde/gmrf.hpp"
#include "gmrfpde/priors/boundary.hpp"
#include "gmrfpde/priors/matern.hpp"
#include "gmrfpde/priors/spatiotemporal.hpp"
#include "gmrfpde/solver/gauss_newton.hpp"
#include "gmrfpde/solver/info_operator.hpp"
#include "gmrfpde/solver/residual.hpp"
#include "oracles.hpp"

using namespace gmrfpde;

namespace {

thread_local std::string g_err;

struct Bundle {
  std::map<std::string, SparseMatrixCSC> mats;
  std::map<std::string, Vector> vecs;
  std::map<std::string, std::vector<Index>> ivecs;
  std::map<std::string, double> scalars;
};

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

SparseMatrixCSC make_csc(int n_rows, int n_cols, const int* cp, const int* ri, const double* v) {
  SparseMatrixCSC m(n_rows, n_cols);
  m.col_ptr.assign(cp, cp + n_cols + 1);
  m.row_idx.assign(ri, ri + cp[n_cols]);
  m.values.assign(v, v + cp[n_cols]);
  return m;
}

// FP64 floor probe (SURVEY §8(c) "floor2"): multiply every input value by
// (1 ± 2⁻⁵²), signs from Rng(seed); seed 0 leaves the input untouched. Running the
// unmodified reference chain on perturbed inputs (initial condition, prior
// precision — re-symmetrized — and prior square root) measures how far its own
// outputs move under one ulp of input noise: the tolerance scale for GPU parity
// (the device assembles Q and q_eff in a different operation order).
void ulp_perturb(Vector& v, double seed) {
  if (seed == 0.0) return;
  Rng r(static_cast<std::uint64_t>(seed));
  for (double& x : v) x *= (r.uniform() < 0.5 ? 1.0 - 0x1p-52 : 1.0 + 0x1p-52);
}
Gmrf ulp_perturb_prior(const Gmrf& g, double seed) {
  if (seed == 0.0) return g;
  SparseMatrixCSC q = g.precision(), s = g.sqrt();
  ulp_perturb(q.values, seed + 1);
  ulp_perturb(s.values, seed + 2);
  return Gmrf(g.mean(), symmetrize(q), std::move(s));
}

// Fixed-step GN trace → flat vectors.
void put_trace(Bundle& b, const std::vector<solver::GaussNewtonIteration>& tr) {
  Vector obj, dec, step, bt;
  for (const auto& r : tr) {
    obj.push_back(r.objective);
    dec.push_back(r.decrement);
    step.push_back(r.step_size);
    bt.push_back(static_cast<double>(r.backtracks));
  }
  b.vecs["gn_objective"] = obj;
  b.vecs["gn_decrement"] = dec;
  b.vecs["gn_step"] = step;
  b.vecs["gn_backtracks"] = bt;
}

// ----- a4-a6: P1 element matrices of one slice -----------
Bundle* build_fem(const double* p, int np) {
  // p: [dim, resolution, xa, xb, diffusion, advection, reaction, dirichlet, eps]
  (void)np;
  const int dim = static_cast<int>(p[0]), res = static_cast<int>(p[1]);
  auto* b = new Bundle();
  fem::FeSpace space(dim == 1 ? fem::build_interval_mesh(res, p[2], p[3])
                              : fem::build_unit_square_mesh(res),
                     1);
  fem::DifferentialOperatorSpec op;
  op.diffusion = p[4];
  if (p[5] != 0.0) op.advection = {p[5]};
  op.reaction = p[6];
  SparseMatrixCSC m = fem::assemble_mass(space);
  SparseMatrixCSC k = fem::assemble_stiffness(space, op);
  b->mats["M"] = m;
  b->mats["K"] = k;
  b->vecs["lumped"] = fem::lumped_mass_vector(m);
  if (p[7] != 0.0) {
    fem::ConstraintSet cs = priors::embed_dirichlet(space, p[8]);
    auto pr = fem::apply_constraints_precision_pair(k, m, cs);
    b->mats["K_c"] = pr.first;
    b->mats["M_c"] = pr.second;
    b->vecs["lumped_c"] = fem::lumped_mass_vector(pr.second);
  }
  return b;
}

// ----- C1/C2: Matérn regression ------------------------
Bundle* build_matern(int dim, const double* p, int np) {
  // p: [resolution, kappa, alpha, tau, n_obs, seed, noise_prec, obs_sd, n_samples,
  //     sample_seed, do_variance]
  (void)np;
  int res = static_cast<int>(p[0]);
  priors::MaternSpec spec{p[1], static_cast<int>(p[2]), p[3]};
  int m = static_cast<int>(p[4]);
  Rng rng(static_cast<std::uint64_t>(p[5]));
  double lam = p[6], sd = p[7];
  int n_samples = static_cast<int>(p[8]);
  auto* b = new Bundle();
  fem::FeSpace space(dim == 1 ? fem::build_interval_mesh(res, 0.0, 1.0)
                              : fem::build_unit_square_mesh(res),
                     1);
  double t0 = now_s();
  Gmrf prior = priors::matern_prior(space, spec);
  b->scalars["t_prior"] = now_s() - t0;
  std::vector<Real> pts(m * dim);
  for (auto& v : pts) v = rng.uniform();
  Vector y(m);
  for (int i = 0; i < m; ++i) {
    double e = rng.normal();
    if (dim == 1)
      y[i] = std::sin(2 * M_PI * pts[i]) + sd * e;
    else
      y[i] = std::sin(3 * M_PI * pts[2 * i]) * std::cos(2 * M_PI * pts[2 * i + 1]) + sd * e;
  }
  auto op = solver::point_observation_operator(space, pts, y, lam);
  t0 = now_s();
  Gmrf post = solver::condition_on(prior, op);
  b->scalars["t_condition"] = now_s() - t0;
  b->mats["Q_prior"] = prior.precision();
  b->mats["S_prior"] = prior.sqrt();
  b->mats["A"] = op.A;
  b->vecs["y"] = op.b;
  b->vecs["noise"] = op.noise_precision;
  b->vecs["points"] = pts;
  b->mats["Q_post"] = post.precision();
  b->vecs["mean_post"] = post.mean();
  b->ivecs["perm_amd"] = post.factor().perm;
  b->mats["L"] = post.factor().L;
  if (p[10] != 0.0) {
    t0 = now_s();
    b->vecs["var_post"] = variance_takahashi(post);
    b->scalars["t_variance"] = now_s() - t0;
  }
  Rng srng(static_cast<std::uint64_t>(p[9]));
  Vector zs, ss;
  t0 = now_s();
  for (int s = 0; s < n_samples; ++s) {
    Vector z = srng.normal_vector(post.dim());
    Vector x = sample_direct(post, z);
    zs.insert(zs.end(), z.begin(), z.end());
    ss.insert(ss.end(), x.begin(), x.end());
  }
  b->scalars["t_samples"] = now_s() - t0;
  b->vecs["z"] = zs;
  b->vecs["samples"] = ss;
  return b;
}

// ----- spatiotemporal prior (+ IC conditioning, + Burgers GN-Laplace) --------
// p: [kind(0 heat, 1 burgers), n_el, x_a, x_b, n_t, t_end, nu, c, noise_kappa,
//     noise_alpha, noise_tau, init_kappa, init_alpha, init_tau, tau, eps,
//     ic_noise_prec, ic_seed, pde_noise_prec, gn_max_iters, do_variance, do_gn,
//     prior_only, floor_seed]
Bundle* build_spatiotemporal(const double* p, int np) {
  (void)np;
  int kind = static_cast<int>(p[0]);
  int n_el = static_cast<int>(p[1]);
  double xa = p[2], xb = p[3];
  int n_t = static_cast<int>(p[4]);
  double t_end = p[5], nu = p[6], c = p[7];
  auto* b = new Bundle();
  fem::FeSpace space(fem::build_interval_mesh(n_el, xa, xb), 1);
  fem::ConstraintSet cs = priors::embed_dirichlet(space, p[15]);
  Vector t_grid(n_t);
  for (int i = 0; i < n_t; ++i) t_grid[i] = t_end * i / static_cast<double>(n_t - 1);
  priors::SpatiotemporalSpec st;
  st.t_grid = t_grid;
  st.spatial_op = kind == 0 ? fem::laplace_operator(nu)
                            : priors::linear_proxy_operator({c}, nu);
  st.noise_spec = {p[8], static_cast<int>(p[9]), p[10]};
  st.initial_spec = {p[11], static_cast<int>(p[12]), p[13]};
  st.tau = p[14];
  double t0 = now_s();
  auto [stp, flat] = priors::spatiotemporal_prior(space, st, cs);
  b->scalars["t_prior"] = now_s() - t0;
  b->mats["Q_prior"] = flat.precision();
  b->mats["S_prior"] = flat.sqrt();
  if (np > 22 && p[22] != 0.0) return b;  // prior only
  int n = space.n_dofs();
  // Initial condition (runner.hpp:555-579 recipe).
  Vector u0(n);
  if (kind == 0) {
    Rng rng(static_cast<std::uint64_t>(p[17]));
    Vector a(10);
    for (int k = 1; k <= 10; ++k) a[k - 1] = rng.normal() / k;
    for (int d = 0; d < n; ++d) {
      double x = space.dof_x(d), v = 0;
      for (int k = 1; k <= 10; ++k) v += a[k - 1] * std::sin(k * M_PI * x);
      u0[d] = v;
    }
  } else {
    for (int d = 0; d < n; ++d) u0[d] = -std::sin(M_PI * space.dof_x(d));
  }
  if (np > 23) {  // p[23]: floor-probe seed (0: off)
    ulp_perturb(u0, p[23]);
    flat = ulp_perturb_prior(flat, p[23]);
  }
  std::vector<Real> ic_points(n);
  for (int d = 0; d < n; ++d) ic_points[d] = space.dof_x(d);
  SparseMatrixCSC e0 = fem::eval_basis(space, ic_points, {0, 0});
  auto [e0f, shift] = fem::fold_pointwise_operator(e0, Vector(n, 0.0), cs);
  std::vector<Triplet> ic_trips;
  for (Index j = 0; j < n; ++j)
    for (Index q = e0f.col_ptr[j]; q < e0f.col_ptr[j + 1]; ++q)
      ic_trips.push_back({e0f.row_idx[q], j, e0f.values[q]});
  solver::LinearInformationOperator ic_op;
  ic_op.A = csc_from_triplets(n, n_t * n, std::move(ic_trips));
  ic_op.b = u0;
  ic_op.noise_precision.assign(n, p[16]);
  b->mats["A_ic"] = ic_op.A;
  b->vecs["y_ic"] = ic_op.b;
  b->vecs["noise_ic"] = ic_op.noise_precision;
  t0 = now_s();
  Gmrf cond = solver::condition_on(flat, ic_op);
  b->scalars["t_condition"] = now_s() - t0;
  b->mats["Q_cond"] = cond.precision();
  b->mats["S_cond"] = cond.sqrt();
  b->vecs["mean_cond"] = cond.mean();
  Gmrf post = cond;
  if (kind == 1 && p[21] != 0.0) {
    auto res = solver::burgers_fem_residual(space, t_grid, cs, nu,
                                            solver::TimeScheme::kImplicitEuler, p[18]);
    b->mats["J_at_mean_cond"] = res.jacobian(cond.mean());
    b->vecs["f_at_mean_cond"] = res.eval(cond.mean());
    solver::GaussNewtonConfig cfg;
    cfg.max_iters = static_cast<Index>(p[19]);
    cfg.decrement_tol = 1e-5;
    t0 = now_s();
    auto gn = solver::gauss_newton(cond, res, cond.mean(), cfg);
    b->scalars["t_gn"] = now_s() - t0;
    put_trace(*b, gn.trace);
    b->vecs["mode"] = gn.mode;
    b->scalars["gn_converged"] = gn.converged ? 1.0 : 0.0;
    t0 = now_s();
    post = solver::laplace_posterior(cond, res, gn.mode);
    b->scalars["t_laplace_build"] = now_s() - t0;
    b->mats["Q_la"] = post.precision();
  }
  b->vecs["mean_post"] = post.mean();
  if (p[20] != 0.0) {
    t0 = now_s();
    b->vecs["var_post"] = variance_takahashi(post);
    b->scalars["t_variance"] = now_s() - t0;
  }
  return b;
}

// ----- C5: Allen-Cahn space-time residual (absent from the reference) --------
// CPU restatement written for this oracle, following the layout of
// burgers_fem_residual (solver/residual.hpp:244-382: rows = steps × kept test
// DoFs, weak (u⁺−u)/Δt time term with the folded mass, implicit Euler) and the
// lumped reaction of nonlinear_elliptic_residual (residual.hpp:431-441,478-482),
// with the Allen-Cahn sign: u_t = ε²Δu − (u³ − u), so per step s
//   r_s = M(u_{s+1} − u_s)/Δt + ε² K u_{s+1} + M̃ (u_{s+1}³ − u_{s+1}),
//   J_s = [−M/Δt | M/Δt + ε² K + diag(M̃ (3u² − 1))]   (slices s, s+1).
// C5 has no constraints (natural BC), so every DoF is a kept row.
solver::NonlinearResidual allen_cahn_residual(const fem::FeSpace& space, const Vector& t_grid,
                                              Real eps2, Real noise_prec) {
  struct Data {
    SparseMatrixCSC mass, stiff;
    Vector lumped, t_grid;
    Index n;
    Real eps2;
  };
  auto d = std::make_shared<Data>();
  d->mass = fem::assemble_mass(space);
  d->stiff = fem::assemble_stiffness(space, fem::laplace_operator(1.0));
  d->lumped = fem::lumped_mass_vector(d->mass);
  d->t_grid = t_grid;
  d->n = space.n_dofs();
  d->eps2 = eps2;
  const Index n_steps = static_cast<Index>(t_grid.size()) - 1;
  solver::NonlinearResidual res;
  res.input_dim = static_cast<Index>(t_grid.size()) * d->n;
  res.output_dim = n_steps * d->n;
  res.noise_precision.assign(res.output_dim, noise_prec);
  res.target.assign(res.output_dim, 0.0);
  res.eval = [d](const Vector& u) {
    const Index n = d->n, ns = static_cast<Index>(d->t_grid.size()) - 1;
    Vector r(ns * n, 0.0);
    for (Index s = 0; s < ns; ++s) {
      const Real dt = d->t_grid[s + 1] - d->t_grid[s];
      Vector du(n), u1(u.begin() + (s + 1) * n, u.begin() + (s + 2) * n);
      for (Index i = 0; i < n; ++i) du[i] = u[(s + 1) * n + i] - u[s * n + i];
      Vector mdu = matvec(d->mass, du), ku = matvec(d->stiff, u1);
      for (Index i = 0; i < n; ++i) {
        const Real v = u1[i];
        r[s * n + i] = mdu[i] / dt + (d->eps2 * ku[i] + d->lumped[i] * (v * v * v - v));
      }
    }
    return r;
  };
  res.jacobian = [d](const Vector& u) {
    const Index n = d->n, ns = static_cast<Index>(d->t_grid.size()) - 1;
    std::vector<Triplet> t;
    for (Index s = 0; s < ns; ++s) {
      const Real dt = d->t_grid[s + 1] - d->t_grid[s];
      for (Index j = 0; j < n; ++j) {
        for (Index p = d->mass.col_ptr[j]; p < d->mass.col_ptr[j + 1]; ++p)
          t.push_back({s * n + d->mass.row_idx[p], s * n + j, -d->mass.values[p] / dt});
        for (Index p = d->mass.col_ptr[j]; p < d->mass.col_ptr[j + 1]; ++p)
          t.push_back({s * n + d->mass.row_idx[p], (s + 1) * n + j, d->mass.values[p] / dt});
        for (Index p = d->stiff.col_ptr[j]; p < d->stiff.col_ptr[j + 1]; ++p)
          t.push_back({s * n + d->stiff.row_idx[p], (s + 1) * n + j, d->eps2 * d->stiff.values[p]});
        const Real v = u[(s + 1) * n + j];
        t.push_back({s * n + j, (s + 1) * n + j, d->lumped[j] * (3.0 * v * v - 1.0)});
      }
    }
    return csc_from_triplets(ns * n, static_cast<Index>(d->t_grid.size()) * n, std::move(t));
  };
  return res;
}

// ----- C5-shaped space-time Allen-Cahn GN-Laplace on the unit square ----------
// p: [n_per_dim, n_t, t_end, eps2, noise_kappa, noise_alpha, noise_tau,
//     init_kappa, init_alpha, init_tau, tau, ic_noise_prec, ic_seed,
//     pde_noise_prec, gn_max_iters, do_variance, do_gn, fd_check, floor_seed]
Bundle* build_allen_cahn(const double* p, int np) {
  (void)np;
  const int npd = static_cast<int>(p[0]);
  const int n_t = static_cast<int>(p[1]);
  const double t_end = p[2], eps2 = p[3];
  auto* b = new Bundle();
  fem::FeSpace space(fem::build_unit_square_mesh(npd), 1);
  fem::ConstraintSet cs;  // natural boundary conditions
  Vector t_grid(n_t);
  for (int i = 0; i < n_t; ++i) t_grid[i] = t_end * i / static_cast<double>(n_t - 1);
  priors::SpatiotemporalSpec st;
  st.t_grid = t_grid;
  st.spatial_op = fem::laplace_operator(eps2);
  st.noise_spec = {p[4], static_cast<int>(p[5]), p[6]};
  st.initial_spec = {p[7], static_cast<int>(p[8]), p[9]};
  st.tau = p[10];
  double t0 = now_s();
  auto [stp, flat] = priors::spatiotemporal_prior(space, st, cs);
  b->scalars["t_prior"] = now_s() - t0;
  b->mats["Q_prior"] = flat.precision();
  b->mats["S_prior"] = flat.sqrt();
  const int n = space.n_dofs();
  // IC draw: u0_d = −0.1 + 0.2·uniform in DoF order
  Rng rng(static_cast<std::uint64_t>(p[12]));
  Vector u0(n);
  for (int d = 0; d < n; ++d) u0[d] = -0.1 + 0.2 * rng.uniform();
  if (np > 18) {  // p[18]: floor-probe seed (0: off)
    ulp_perturb(u0, p[18]);
    flat = ulp_perturb_prior(flat, p[18]);
  }
  b->vecs["u0"] = u0;
  std::vector<Triplet> ic;  // P1 nodes = DoFs: point evaluation at the nodes
  for (int d = 0; d < n; ++d) ic.push_back({d, d, 1.0});
  solver::LinearInformationOperator ic_op;
  ic_op.A = csc_from_triplets(n, n_t * n, std::move(ic));
  ic_op.b = u0;
  ic_op.noise_precision.assign(n, p[11]);
  t0 = now_s();
  Gmrf cond = solver::condition_on(flat, ic_op);
  b->scalars["t_condition"] = now_s() - t0;
  b->mats["Q_cond"] = cond.precision();
  b->mats["S_cond"] = cond.sqrt();
  b->vecs["mean_cond"] = cond.mean();
  Gmrf post = cond;
  auto res = allen_cahn_residual(space, t_grid, eps2, p[13]);
  b->mats["J_at_mean_cond"] = res.jacobian(cond.mean());
  b->vecs["f_at_mean_cond"] = res.eval(cond.mean());
  if (p[17] != 0.0) {  // finite-difference check of the Jacobian (acceptance.cpp:503-608 pattern)
    Vector x = cond.mean();
    for (std::size_t i = 0; i < x.size(); ++i) x[i] += 0.3 * std::sin(0.37 * static_cast<double>(i));
    SparseMatrixCSC jac = res.jacobian(x);
    Vector f0 = res.eval(x);
    Rng drng(77);
    Vector dir(x.size());
    for (auto& v : dir) v = drng.normal();
    const double hstep = 1e-6;
    Vector xp(x), xm(x);
    for (std::size_t i = 0; i < x.size(); ++i) {
      xp[i] += hstep * dir[i];
      xm[i] -= hstep * dir[i];
    }
    Vector fp = res.eval(xp), fm = res.eval(xm), jd = matvec(jac, dir);
    double num = 0, den = 0;
    for (std::size_t i = 0; i < f0.size(); ++i) {
      const double fd = (fp[i] - fm[i]) / (2 * hstep);
      num = std::max(num, std::abs(fd - jd[i]));
      den = std::max(den, std::abs(jd[i]));
    }
    b->scalars["fd_rel_err"] = num / std::max(den, 1e-300);
  }
  if (p[16] != 0.0) {
    solver::GaussNewtonConfig cfg;
    cfg.max_iters = static_cast<Index>(p[14]);
    cfg.decrement_tol = 1e-5;
    t0 = now_s();
    auto gn = solver::gauss_newton(cond, res, cond.mean(), cfg);
    b->scalars["t_gn"] = now_s() - t0;
    put_trace(*b, gn.trace);
    b->vecs["mode"] = gn.mode;
    b->scalars["gn_converged"] = gn.converged ? 1.0 : 0.0;
    t0 = now_s();
    post = solver::laplace_posterior(cond, res, gn.mode);
    b->scalars["t_laplace_build"] = now_s() - t0;
    b->mats["Q_la"] = post.precision();
  }
  b->vecs["mean_post"] = post.mean();
  if (p[15] != 0.0) {
    t0 = now_s();
    b->vecs["var_post"] = variance_takahashi(post);
    b->scalars["t_variance"] = now_s() - t0;
  }
  return b;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ----- bundles ---------------------------------------------------------------
void* ref_build(const char* kind, const double* p, int np) {
  try {
    std::string k(kind);
    if (k == "fem") return build_fem(p, np);
    if (k == "matern1d") return build_matern(1, p, np);
    if (k == "matern2d") return build_matern(2, p, np);
    if (k == "spatiotemporal") return build_spatiotemporal(p, np);
    if (k == "allen_cahn") return build_allen_cahn(p, np);
    if (k == "corpus") {
      // p: [count, seed]; matrices "Q0".."Q{count-1}"
      auto corpus = oracle::spd_corpus(static_cast<int>(p[0]), static_cast<std::uint64_t>(p[1]));
      auto* b = new Bundle();
      for (std::size_t i = 0; i < corpus.size(); ++i) b->mats["Q" + std::to_string(i)] = corpus[i];
      return b;
    }
    g_err = "unknown bundle kind " + k;
  } catch (const std::exception& e) {
    g_err = e.what();
  }
  return nullptr;
}

void ref_bundle_free(void* b) { delete static_cast<Bundle*>(b); }

int ref_bundle_mat_shape(void* hb, const char* name, int* nr, int* nc, int* nnz) {
  auto* b = static_cast<Bundle*>(hb);
  auto it = b->mats.find(name);
  if (it == b->mats.end()) return -1;
  *nr = it->second.nrows;
  *nc = it->second.ncols;
  *nnz = it->second.nnz();
  return 0;
}

int ref_bundle_mat_copy(void* hb, const char* name, int* cp, int* ri, double* v) {
  auto* b = static_cast<Bundle*>(hb);
  auto it = b->mats.find(name);
  if (it == b->mats.end()) return -1;
  const auto& m = it->second;
  std::memcpy(cp, m.col_ptr.data(), sizeof(int) * m.col_ptr.size());
  std::memcpy(ri, m.row_idx.data(), sizeof(int) * m.row_idx.size());
  std::memcpy(v, m.values.data(), sizeof(double) * m.values.size());
  return 0;
}

long long ref_bundle_vec_len(void* hb, const char* name) {
  auto* b = static_cast<Bundle*>(hb);
  auto it = b->vecs.find(name);
  if (it != b->vecs.end()) return static_cast<long long>(it->second.size());
  auto jt = b->ivecs.find(name);
  if (jt != b->ivecs.end()) return -2 - static_cast<long long>(jt->second.size());
  return -1;
}

int ref_bundle_vec_copy(void* hb, const char* name, double* out) {
  auto* b = static_cast<Bundle*>(hb);
  auto it = b->vecs.find(name);
  if (it != b->vecs.end()) {
    std::memcpy(out, it->second.data(), sizeof(double) * it->second.size());
    return 0;
  }
  auto jt = b->ivecs.find(name);
  if (jt != b->ivecs.end()) {
    for (std::size_t i = 0; i < jt->second.size(); ++i) out[i] = jt->second[i];
    return 0;
  }
  return -1;
}

double ref_bundle_scalar(void* hb, const char* name) {
  auto* b = static_cast<Bundle*>(hb);
  auto it = b->scalars.find(name);
  return it == b->scalars.end() ? std::nan("") : it->second;
}

// ----- core linear algebra (core/amd.hpp, core/cholesky.hpp, core/takahashi.hpp)
int ref_amd_order(int n, const int* cp, const int* ri, int* perm) {
  try {
    std::vector<double> v(cp[n], 1.0);
    auto p = amd_order(make_csc(n, n, cp, ri, v.data()));
    std::memcpy(perm, p.data(), sizeof(int) * n);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// symbolic_analyze (cholesky.hpp:68): parent[n], col_ptr_L[n+1]
int ref_symbolic(int n, const int* cp, const int* ri, const int* perm, int* parent,
                 int* colptr_l) {
  try {
    std::vector<double> v(cp[n], 1.0);
    std::vector<Index> pv(perm, perm + n);
    SymbolicFactor s = symbolic_analyze(make_csc(n, n, cp, ri, v.data()), pv);
    std::memcpy(parent, s.parent.data(), sizeof(int) * n);
    std::memcpy(colptr_l, s.col_ptr.data(), sizeof(int) * (n + 1));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

struct RefFactor {
  CholeskyFactor f;
};

// cholesky_factor (cholesky.hpp:164/170). perm == nullptr → AMD. Returns
// nullptr on failure; *bad = original index of a non-positive pivot or -1.
void* ref_factor(int n, const int* cp, const int* ri, const double* v, const int* perm,
                 int* bad) {
  *bad = -1;
  try {
    SparseMatrixCSC q = make_csc(n, n, cp, ri, v);
    auto* h = new RefFactor();
    if (perm) {
      h->f = cholesky_factor(q, std::vector<Index>(perm, perm + n));
    } else {
      h->f = cholesky_factor(q);
    }
    return h;
  } catch (const NotPositiveDefiniteError& e) {
    *bad = e.index();
    g_err = e.what();
  } catch (const std::exception& e) {
    g_err = e.what();
  }
  return nullptr;
}

void ref_factor_free(void* h) { delete static_cast<RefFactor*>(h); }

int ref_factor_nnz(void* h) { return static_cast<RefFactor*>(h)->f.L.nnz(); }

void ref_factor_copy(void* h, int* cp, int* ri, double* v, int* perm) {
  const auto& f = static_cast<RefFactor*>(h)->f;
  std::memcpy(cp, f.L.col_ptr.data(), sizeof(int) * f.L.col_ptr.size());
  std::memcpy(ri, f.L.row_idx.data(), sizeof(int) * f.L.row_idx.size());
  std::memcpy(v, f.L.values.data(), sizeof(double) * f.L.values.size());
  std::memcpy(perm, f.perm.data(), sizeof(int) * f.perm.size());
}

// solve_triangular (cholesky.hpp:179); mode 0 lower, 1 upper, 2 full.
void ref_solve(void* h, int mode, const double* b, double* x) {
  const auto& f = static_cast<RefFactor*>(h)->f;
  Vector bb(b, b + f.dim());
  Vector r = solve_triangular(f, bb, static_cast<TriangularMode>(mode));
  std::memcpy(x, r.data(), sizeof(double) * r.size());
}

// takahashi_diagonal (takahashi.hpp:67)
void ref_takahashi_diag(void* h, double* out) {
  const auto& f = static_cast<RefFactor*>(h)->f;
  Vector d = takahashi_diagonal(f);
  std::memcpy(out, d.data(), sizeof(double) * d.size());
}

// takahashi_selected_inverse (takahashi.hpp:19) → bundle matrix "S"
void* ref_takahashi_full(void* h) {
  auto* b = new Bundle();
  b->mats["S"] = takahashi_selected_inverse(static_cast<RefFactor*>(h)->f);
  return b;
}

// condition_affine (gmrf.hpp:145) with diagonal noise → bundle {Q_post, mean_post}
void* ref_condition_affine(int n, const int* qcp, const int* qri, const double* qv,
                           const double* mu, int m, const int* acp, const int* ari,
                           const double* av, const double* bvec, const double* y,
                           const double* noise) {
  try {
    Gmrf prior(Vector(mu, mu + n), make_csc(n, n, qcp, qri, qv));
    auto obs = AffineObservation::with_diagonal_noise(make_csc(m, n, acp, ari, av),
                                                      Vector(bvec, bvec + m),
                                                      Vector(y, y + m), Vector(noise, noise + m));
    Gmrf post = condition_affine(prior, obs);
    auto* b = new Bundle();
    b->mats["Q_post"] = post.precision();
    b->vecs["mean_post"] = post.mean();
    return b;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// sample_direct (gmrf.hpp:173,182) n_samples times from Rng(seed), and
// rbmc_variance (gmrf.hpp:213-240), on Gmrf(mu, Q) with the factor attached
// for the given permutation (attach_factor, gmrf.hpp:49-51) so the draws use
// the same L ordering as the GPU. out: n × ns column-major / n.
int ref_sample_direct(int n, const int* cp, const int* ri, const double* v, const int* perm,
                      const double* mu, int ns, unsigned long long seed, double* out) {
  try {
    SparseMatrixCSC q = make_csc(n, n, cp, ri, v);
    Gmrf g(Vector(mu, mu + n), q);
    g.attach_factor(std::make_shared<const CholeskyFactor>(
        cholesky_factor(q, std::vector<Index>(perm, perm + n))));
    Rng rng(seed);
    for (int k = 0; k < ns; ++k) {
      Vector x = sample_direct(g, rng);
      std::memcpy(out + static_cast<size_t>(k) * n, x.data(), sizeof(double) * n);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_rbmc_variance(int n, const int* cp, const int* ri, const double* v, const int* perm,
                      const double* mu, int ns, unsigned long long seed, double* out) {
  try {
    SparseMatrixCSC q = make_csc(n, n, cp, ri, v);
    Gmrf g(Vector(mu, mu + n), q);
    g.attach_factor(std::make_shared<const CholeskyFactor>(
        cholesky_factor(q, std::vector<Index>(perm, perm + n))));
    Vector var = rbmc_variance(g, ns, seed);
    std::memcpy(out, var.data(), sizeof(double) * n);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// cg_solve (cg.hpp:98), matrix-backed; out_info = {iterations, final_residual, converged}
int ref_cg_solve(int n, const int* cp, const int* ri, const double* v, const double* b,
                 double rtol, double atol, long long max_iter, int jacobi, double* x,
                 double* out_info) {
  try {
    SparseMatrixCSC q = make_csc(n, n, cp, ri, v);
    CGConfig cfg;
    cfg.rtol = rtol;
    cfg.atol = atol;
    cfg.max_iter = static_cast<Index>(max_iter);
    cfg.preconditioner = jacobi ? Preconditioner::kJacobi : Preconditioner::kNone;
    CGResult r = cg_solve(q, Vector(b, b + n), Vector(), cfg);
    std::memcpy(x, r.x.data(), sizeof(double) * n);
    out_info[0] = static_cast<double>(r.iterations);
    out_info[1] = r.final_residual;
    out_info[2] = r.converged ? 1.0 : 0.0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Timed reference stages on one matrix (for the CPU baseline leg):
// out[0]=amd s, out[1]=symbolic s, out[2]=numeric s, out[3]=full solve s,
// out[4]=takahashi s (if do_taka), out[5]=nnz(L), out[6]=Σ c_j² flops.
int ref_time_stages(int n, const int* cp, const int* ri, const double* v, int do_taka,
                    double* out) {
  try {
    SparseMatrixCSC q = make_csc(n, n, cp, ri, v);
    double t0 = now_s();
    auto perm = amd_order(q);
    double t1 = now_s();
    auto sym = symbolic_analyze(q, perm);
    double t2 = now_s();
    auto f = cholesky_refactor(sym, q);
    double t3 = now_s();
    Vector b(n, 1.0);
    auto x = solve(f, b);
    double t4 = now_s();
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    out[2] = t3 - t2;
    out[3] = t4 - t3;
    out[4] = 0.0;
    if (do_taka) {
      auto d = takahashi_diagonal(f);
      out[4] = now_s() - t4;
    }
    out[5] = f.L.nnz();
    double fl = 0;
    for (int j = 0; j < n; ++j) {
      double cj = f.L.col_ptr[j + 1] - f.L.col_ptr[j];
      fl += cj * cj;
    }
    out[6] = fl;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
