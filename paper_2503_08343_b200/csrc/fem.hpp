// Host-side spatial discretisation: a small CSC toolkit, P1 FEM on 1D interval
// meshes and on the structured triangulated unit square, homogeneous-Dirichlet
// constraint folding, the Matérn SPDE prior and the per-step spatial blocks of
// the implicit-Euler space-time prior (dimension-generic: they only see the
// spatial mass / Laplacian / proxy-operator matrices).
//
// These are n_s-sized (one time slice) and computed once; the joint space-time
// matrices (n_s·n_t) are assembled on the device from them (assembly.cu).
// Semantics follow the reference:
//   P1 mass/stiffness ........ fem/assembly.hpp:81-161
//   unit-square triangulation  fem/mesh.hpp:108-149
//   Dirichlet fold + mask .... fem/constraints.hpp:111-128,158-173, priors/boundary.hpp:15-29
//   lumped mass .............. fem/assembly.hpp:241-262
//   Matérn Q, sqrt ........... priors/matern.hpp:53-80
//   space-time blocks ........ priors/spatiotemporal.hpp:79-195
#pragma once

#include <vector>

#include "common.hpp"

namespace gmrf {

struct Csc {
  i32 nr = 0, nc = 0;
  std::vector<i64> cp{0};
  std::vector<i32> ri;
  std::vector<double> v;
  i64 nnz() const { return static_cast<i64>(ri.size()); }
  double at(i32 i, i32 j) const;
};

struct Trip {
  i32 r, c;
  double v;
};

Csc csc_from_trips(i32 nr, i32 nc, std::vector<Trip> t);  // sums duplicates
Csc transpose(const Csc& a);
Csc multiply(const Csc& a, const Csc& b);
Csc add(const Csc& a, const Csc& b, double alpha = 1.0, double beta = 1.0);
Csc scale(const Csc& a, double s);
Csc scale_rows(const std::vector<double>& d, const Csc& a);
Csc scale_cols(const Csc& a, const std::vector<double>& d);
Csc symmetrize(const Csc& a);
Csc diagonal(const std::vector<double>& d);

// 1D P1 space on a uniform interval mesh with n_el elements over [xa, xb].
struct Space1D {
  i32 n_el;
  double xa, xb;
  i32 n() const { return n_el + 1; }
  double h() const { return (xb - xa) / n_el; }
  // node coordinate (build_interval_mesh, mesh.hpp:63-70)
  double x(i32 d) const {
    return d == n_el ? xb : xa + (xb - xa) * static_cast<double>(d) / static_cast<double>(n_el);
  }
};

Csc p1_mass(const Space1D& s);
// ∫ diff·φ'_i φ'_j + ∫ φ_i c φ'_j + react ∫ φ_i φ_j
Csc p1_stiffness(const Space1D& s, double diff, double adv, double react);

// P1 on the unit square, n_cells² cells each split along the lower-left →
// upper-right diagonal; node (ix, iy) has DoF iy·(n_cells+1) + ix.
struct Space2D {
  i32 n_cells;
  i32 side() const { return n_cells + 1; }
  i32 n() const { return side() * side(); }
  double h() const { return 1.0 / n_cells; }
  // axis coordinate i/n (build_unit_square_mesh, mesh.hpp:142-147)
  double coord(i32 i) const { return static_cast<double>(i) / static_cast<double>(n_cells); }
};
Csc p1_mass(const Space2D& s);
Csc p1_laplace(const Space2D& s);  // ∫ ∇φ_i · ∇φ_j

// The spatial matrices everything downstream needs, for any dimension.
struct SpatialOps {
  i32 n = 0;
  Csc mass;                 // consistent P1 mass
  Csc lap;                  // ∫ ∇φ·∇φ (Matérn priors)
  Csc op;                   // proxy operator of the space-time prior
  std::vector<char> slack;  // constrained (Dirichlet) DoFs
};
SpatialOps spatial_ops(const Space1D& s, double diff, double adv, bool dirichlet);
SpatialOps spatial_ops(const Space2D& s, double diff);

// Homogeneous Dirichlet on both end nodes: slack coordinates.
std::vector<char> dirichlet_mask(const Space1D& s, bool enabled);
// fold_and_mask with T = I: constrained rows/cols removed, `diag` inserted.
// mask_constrained / lumped_mass run the device kernels of fem_device.cu while a
// FemDeviceScope is alive (the pipelines' setup), the host loops otherwise (the
// device-free symbolic planning entry points and the CPU tests).
Csc mask_constrained(const Csc& a, const std::vector<char>& mask, double diag);
std::vector<double> lumped_mass(const Csc& m);
Csc mask_constrained_host(const Csc& a, const std::vector<char>& mask, double diag);
std::vector<double> lumped_mass_host(const Csc& m);
using LumpFn = std::vector<double> (*)(const Csc&);
using MaskFn = Csc (*)(const Csc&, const std::vector<char>&, double);
void set_fem_hooks(LumpFn lump, MaskFn mask);  // nullptr: host

struct MaternSpec {
  double kappa = 1.0;
  int alpha = 2;
  double tau = 1.0;
};
struct MaternPrior {
  Csc q, sqrt;
};
MaternPrior matern_prior(const SpatialOps& ops, const MaternSpec& spec, double eps);

// Per-step spatial blocks of the space-time prior for a uniform time grid.
struct SpaceTimeBlocks {
  i32 n = 0;                // spatial dofs
  double t = 0.0;           // T = 1/(Δt τ²)
  Csc q1, l1;               // initial Matérn precision and sqrt
  Csc c_mm, c_gg, c_mg;     // Q blocks (spatiotemporal.hpp:102-105,133-140)
  Csc s_m, f_is;            // sqrt blocks (before the √T factor)
  // q_eff blocks: the same joint matrix rebuilt through the square root,
  // S Sᵀ (gauss_newton.hpp:110-114): l1 l1ᵀ, s_m s_mᵀ, f_is f_isᵀ, s_m f_isᵀ
  Csc g_l1, g_mm, g_ff, g_mf;
  std::vector<char> slack;  // constrained (slack) spatial coordinates
  double eps = 1e-10;       // slack noise variance
};
SpaceTimeBlocks spacetime_blocks(const SpatialOps& ops, double dt, double tau,
                                 const MaternSpec& noise, const MaternSpec& init, double eps);

}  // namespace gmrf
