// Drop-in gmrfpde/gmrf.hpp: the reference header (reached with #include_next),
// with condition_affine (gmrf.hpp:145-170) replaced by the device update:
// Q_post = symmetrize(Q + Aᵀ Λ A) is assembled and factored on the B200 by a
// fixed-pattern update system (gmrf_update_system_*), the factor attached to
// the posterior as the reference does. Non-diagonal observation noise keeps
// the reference's host product (its factorization still runs on the device
// through the drop-in cholesky.hpp).
#pragma once

#include "gmrfpde/core/cholesky.hpp"

#define condition_affine condition_affine_reference
#include_next "gmrfpde/gmrf.hpp"
#undef condition_affine

#include "gmrfpde/b200/update_system.hpp"

namespace gmrfpde {

inline Gmrf condition_affine(const Gmrf& prior, const AffineObservation& obs) {
  if (!obs.noise_precision_diag) return condition_affine_reference(prior, obs);
  obs.validate(prior.dim());
  // Q_post on the device, written straight into its factor
  auto sys = b200::UpdateSystem::make(b200::UpdateSystem::kPrecision, prior.precision(), obs.A);
  sys->refactor(obs.A, *obs.noise_precision_diag);
  // μ_post = μ + Q_post⁻¹ Aᵀ Λ (y − (Aμ + b))
  const Vector residual = vec_sub(obs.y, vec_add(matvec(obs.A, prior.mean()), obs.b));
  const Vector rhs = matvec_transpose(obs.A, obs.apply_noise(residual));
  auto factor = std::make_shared<const CholeskyFactor>(sys->factor());
  Vector mean = vec_add(prior.mean(), sys->solve(rhs));
  std::optional<SparseMatrixCSC> sqrt;
  if (prior.has_sqrt()) sqrt = hcat(prior.sqrt(), multiply(transpose(obs.A), obs.noise_sqrt()));
  Gmrf posterior(std::move(mean), sys->matrix(), std::move(sqrt));
  posterior.attach_factor(factor);
  return posterior;
}

}  // namespace gmrfpde
