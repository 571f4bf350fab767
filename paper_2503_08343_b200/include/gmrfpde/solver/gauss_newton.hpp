// Drop-in gmrfpde/solver/gauss_newton.hpp: the reference header (reached with
// #include_next) with the Gauss-Newton matrix and the Laplace precision moved
// to the B200 (north_star row 2):
//
//   gauss_newton (gauss_newton.hpp:93-224)   H = symmetrize(q_eff + Jᵀ Λ J) is
//     built by a fixed-pattern update system — q_eff = symmetrize(S Sᵀ) (or Q
//     without a square root) assembled once on the device, each iteration
//     streams J's values and writes H straight into the factor's panels, then
//     factors and solves there. The residual / Jacobian callbacks, gradient,
//     objective and Armijo rule are the reference's (same stop rule, trace and
//     GaussNewtonStagnation).
//   laplace_posterior (:228-240)             Q_LA = symmetrize(Q + J*ᵀ Λ J*) on
//     the device, its factor attached to the returned Gmrf (variance_takahashi
//     and sample_direct then reuse it instead of refactoring).
//
// The CG variant (GnLinearSolver::kCg) is matrix-free and keeps the reference
// loop. The ordering is nested dissection (the reference uses AMD).
#pragma once

#include "gmrfpde/gmrf.hpp"

#define gauss_newton gauss_newton_reference
#define laplace_posterior laplace_posterior_reference
#include_next "gmrfpde/solver/gauss_newton.hpp"
#undef gauss_newton
#undef laplace_posterior

#include "gmrfpde/b200/update_system.hpp"

namespace gmrfpde::solver {

inline GaussNewtonResult gauss_newton(const Gmrf& prior, const NonlinearResidual& res,
                                      const Vector& x0, const GaussNewtonConfig& cfg) {
  if (cfg.linear_solver != GnLinearSolver::kCholesky)
    return gauss_newton_reference(prior, res, x0, cfg);
  cfg.validate();
  require(static_cast<Index>(x0.size()) == prior.dim(),
          "gauss-newton: x0 length must match the prior dimension");
  require(res.input_dim == prior.dim(),
          "gauss-newton: residual input dimension must match the prior");
  const bool use_sqrt = prior.has_sqrt();
  const Index n = prior.dim();

  // ∇ of the prior term: S(Sᵀc) with a square root, Qc without (gauss_newton.hpp:116-119)
  auto prior_grad = [&](const Vector& c) {
    return use_sqrt ? matvec(prior.sqrt(), matvec_transpose(prior.sqrt(), c))
                    : matvec(prior.precision(), c);
  };
  std::shared_ptr<b200::UpdateSystem> sys;  // fixed by the Jacobian's pattern

  GaussNewtonResult out;
  out.mode = x0;
  for (Index iter = 1; iter <= cfg.max_iters; ++iter) {
    const Vector fx = res.eval(out.mode);
    const SparseMatrixCSC jac = res.jacobian(out.mode);
    // grad = prior term − Jᵀ Λ (y − f)
    Vector grad = prior_grad(vec_sub(out.mode, prior.mean()));
    Vector misfit(res.output_dim);
    for (Index i = 0; i < res.output_dim; ++i)
      misfit[i] = res.noise_precision[i] * (res.target[i] - fx[i]);
    const Vector jtm = matvec_transpose(jac, misfit);
    for (Index i = 0; i < n; ++i) grad[i] -= jtm[i];

    // H on the device: one symbolic analysis per Jacobian pattern
    if (!sys || !sys->same_operator(jac))
      sys = b200::UpdateSystem::make(use_sqrt ? b200::UpdateSystem::kSqrt
                                              : b200::UpdateSystem::kPrecision,
                                     use_sqrt ? prior.sqrt() : prior.precision(), jac);
    const Vector direction = sys->refactor_solve(jac, res.noise_precision, scaled(grad, -1.0));

    GaussNewtonIteration rec;
    rec.iter = iter;
    rec.decrement = std::sqrt(std::max(0.0, -dot(grad, direction)));
    rec.objective = detail::negative_log_density(prior, res, out.mode, fx);
    if (rec.decrement < cfg.decrement_tol ||
        0.5 * rec.decrement * rec.decrement <= 1e-14 * (1.0 + std::abs(rec.objective))) {
      out.trace.push_back(rec);
      out.converged = true;
      out.final_decrement = rec.decrement;
      return out;
    }
    // Armijo backtracking on −log π
    const Real slope = dot(grad, direction);
    Real alpha = 1.0;
    Index backtracks = 0;
    for (;;) {
      Vector cand = out.mode;
      axpy(alpha, direction, cand);
      const Real cand_obj = detail::negative_log_density(prior, res, cand, res.eval(cand));
      if (cand_obj <= rec.objective + cfg.armijo_c * alpha * slope) {
        out.mode = std::move(cand);
        break;
      }
      if (++backtracks > cfg.max_backtracks) {
        out.trace.push_back(rec);
        throw GaussNewtonStagnation("gauss-newton: line search failed after " +
                                        std::to_string(backtracks - 1) +
                                        " backtracks at iteration " + std::to_string(iter),
                                    out.trace);
      }
      alpha *= cfg.shrink;
    }
    rec.step_size = alpha;
    rec.backtracks = backtracks;
    out.trace.push_back(rec);
    out.accepted_steps += 1;
    out.final_decrement = rec.decrement;
  }
  return out;
}

inline Gmrf laplace_posterior(const Gmrf& prior, const NonlinearResidual& res, const Vector& mode) {
  const SparseMatrixCSC jac = res.jacobian(mode);
  auto sys = b200::UpdateSystem::make(b200::UpdateSystem::kPrecision, prior.precision(), jac);
  sys->refactor(jac, res.noise_precision);
  std::optional<SparseMatrixCSC> sqrt;
  if (prior.has_sqrt()) {
    Vector ls(res.noise_precision);
    for (Real& v : ls) v = std::sqrt(v);
    sqrt = hcat(prior.sqrt(), multiply(transpose(jac), csc_diagonal(ls)));
  }
  Gmrf post(mode, sys->matrix(), std::move(sqrt));
  post.attach_factor(std::make_shared<const CholeskyFactor>(sys->factor()));
  return post;
}

}  // namespace gmrfpde::solver
