// Drop-in gmrfpde/priors/matern.hpp: the reference header (#include_next) with
// matern_prior (matern.hpp:53-80) assembling Q = symmetrize((1/τ²) K̂ᵀ M̃⁻¹ K̂)
// on the B200 (fixed-pattern Gram product, gmrf_update_system_assemble; same
// per-entry operation order as the reference's SpGEMM + symmetrize). The
// element matrices, constraint fold and lumping stay the reference's host code
// (n-sized, one-off); α >= 3 (recursive products, matern.hpp:75-78) keeps the
// reference path.
#pragma once

#include "gmrfpde/gmrf.hpp"

#define matern_prior matern_prior_reference
#include_next "gmrfpde/priors/matern.hpp"
#undef matern_prior

#include "gmrfpde/b200/update_system.hpp"

namespace gmrfpde::priors {

inline Gmrf matern_prior(const fem::FeSpace& space, const MaternSpec& spec,
                         const fem::ConstraintSet& cs = {}) {
  if (spec.alpha >= 3) return matern_prior_reference(space, spec, cs);
  spec.validate();
  SparseMatrixCSC mass = fem::assemble_mass(space);
  fem::DifferentialOperatorSpec op;
  op.diffusion = 1.0;
  SparseMatrixCSC k = add(fem::assemble_stiffness(space, op), mass, 1.0, spec.kappa * spec.kappa);
  auto [k_hat, m_hat] = fem::apply_constraints_precision_pair(k, mass, cs);
  const Vector lumped = fem::lumped_mass_vector(m_hat);
  Vector inv(lumped.size()), inv_sqrt(lumped.size());
  for (std::size_t i = 0; i < lumped.size(); ++i) {
    inv[i] = 1.0 / lumped[i];
    inv_sqrt[i] = 1.0 / std::sqrt(lumped[i]);
  }
  // Q = sym((1/τ²) Σ_k (K̂_kR / m̃_k) K̂_kC) on the device: B = 0, A = K̂, w = 1/m̃
  const Index n = space.n_dofs();
  auto sys = b200::UpdateSystem::make(b200::UpdateSystem::kPrecision, SparseMatrixCSC(n, n), k_hat);
  sys->assemble(k_hat, inv, 1.0 / (spec.tau * spec.tau));
  SparseMatrixCSC kt = transpose(k_hat);
  SparseMatrixCSC sqrt_l = scale(scale_cols(kt, inv_sqrt), 1.0 / spec.tau);
  return Gmrf(Vector(n, 0.0), sys->matrix(), std::move(sqrt_l));
}

}  // namespace gmrfpde::priors
