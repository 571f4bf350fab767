// Device P1 element assembly and the small per-slice operators around it
// (SURVEY §8(a) rows a4-a6):
//   a4  assemble_mass / assemble_stiffness  (fem/assembly.hpp:81-161)   k_p1_interval, k_p1_square
//   a5  lumped_mass_vector                  (assembly.hpp:241-262)      k_lump_columns
//   a6  fold_and_mask, T = I                (fem/constraints.hpp:111-128,158-173) k_gather_values
// One thread per matrix column gathers the element contributions of its
// stencil in the element order of the reference's triplet list (no atomics:
// every entry sums in a fixed order), with every operation spelled out
// (__dmul_rn / __dadd_rn / __ddiv_rn / __fma_rn, nothing left to the compiler's
// contraction): the values are bit-identical to the host closed forms of fem.cpp,
// which the CPU tests pin against the reference's quadrature assembly.
#pragma once

#include <cuda_runtime.h>

#include "fem.hpp"

namespace gmrf {

// mass, ∫∇φ·∇φ and the proxy operator of a slice, values computed on the device.
SpatialOps spatial_ops_device(const Space1D& s, double diff, double adv, bool dirichlet,
                              cudaStream_t st = nullptr);
SpatialOps spatial_ops_device(const Space2D& s, double diff, cudaStream_t st = nullptr);
// One P1 matrix on the device: which = 0 mass, 1 stiffness (1-D: diff, adv,
// react; 2-D: diff · ∫∇φ·∇φ).
Csc p1_matrix_device(int dim, i32 n_el, double xa, double xb, int which, double diff, double adv,
                     double react, cudaStream_t st = nullptr);
std::vector<double> lumped_mass_device(const Csc& m, cudaStream_t st = nullptr);
Csc mask_constrained_device(const Csc& a, const std::vector<char>& mask, double diag,
                            cudaStream_t st = nullptr);


// While alive, fem.cpp's lumped_mass / mask_constrained (called inside
// matern_prior and spacetime_blocks) run on the device. Not reentrant across
// threads: pipelines are set up one at a time.
struct FemDeviceScope {
  FemDeviceScope();
  ~FemDeviceScope();
  FemDeviceScope(const FemDeviceScope&) = delete;
  FemDeviceScope& operator=(const FemDeviceScope&) = delete;
};

}  // namespace gmrf
