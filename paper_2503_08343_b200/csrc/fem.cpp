// Host-side spatial discretisation. See fem.hpp for the reference mapping.
#include "fem.hpp"

#include <algorithm>
#include <cmath>

namespace gmrf {

double Csc::at(i32 i, i32 j) const {
  auto b = ri.begin() + cp[j], e = ri.begin() + cp[j + 1];
  auto it = std::lower_bound(b, e, i);
  return (it != e && *it == i) ? v[it - ri.begin()] : 0.0;
}

Csc csc_from_trips(i32 nr, i32 nc, std::vector<Trip> t) {
  // stable order within duplicates: summed in insertion order
  std::stable_sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) {
    return a.c != b.c ? a.c < b.c : a.r < b.r;
  });
  Csc m;
  m.nr = nr;
  m.nc = nc;
  m.cp.assign(nc + 1, 0);
  size_t k = 0;
  for (i32 j = 0; j < nc; ++j) {
    while (k < t.size() && t[k].c == j) {
      i32 r = t[k].r;
      double v = t[k].v;
      ++k;
      while (k < t.size() && t[k].c == j && t[k].r == r) v += t[k++].v;
      m.ri.push_back(r);
      m.v.push_back(v);
    }
    m.cp[j + 1] = m.nnz();
  }
  return m;
}

Csc transpose(const Csc& a) {
  Csc t;
  t.nr = a.nc;
  t.nc = a.nr;
  t.cp.assign(a.nr + 1, 0);
  for (i64 p = 0; p < a.nnz(); ++p) t.cp[a.ri[p] + 1]++;
  for (i32 i = 0; i < a.nr; ++i) t.cp[i + 1] += t.cp[i];
  t.ri.resize(a.nnz());
  t.v.resize(a.nnz());
  std::vector<i64> nx(t.cp.begin(), t.cp.end() - 1);
  for (i32 j = 0; j < a.nc; ++j)
    for (i64 p = a.cp[j]; p < a.cp[j + 1]; ++p) {
      i64 q = nx[a.ri[p]]++;
      t.ri[q] = j;
      t.v[q] = a.v[p];
    }
  return t;
}

Csc multiply(const Csc& a, const Csc& b) {
  require(a.nc == b.nr, kDimension, "multiply: inner dimension mismatch");
  Csc c;
  c.nr = a.nr;
  c.nc = b.nc;
  c.cp.assign(b.nc + 1, 0);
  std::vector<double> work(a.nr, 0.0);
  std::vector<i32> mark(a.nr, -1), cols;
  for (i32 j = 0; j < b.nc; ++j) {
    cols.clear();
    for (i64 pb = b.cp[j]; pb < b.cp[j + 1]; ++pb) {
      i32 k = b.ri[pb];
      double bkj = b.v[pb];
      for (i64 pa = a.cp[k]; pa < a.cp[k + 1]; ++pa) {
        i32 i = a.ri[pa];
        if (mark[i] != j) {
          mark[i] = j;
          work[i] = 0.0;
          cols.push_back(i);
        }
        work[i] += a.v[pa] * bkj;
      }
    }
    std::sort(cols.begin(), cols.end());
    for (i32 i : cols) {
      c.ri.push_back(i);
      c.v.push_back(work[i]);
    }
    c.cp[j + 1] = c.nnz();
  }
  return c;
}

Csc add(const Csc& a, const Csc& b, double alpha, double beta) {
  require(a.nr == b.nr && a.nc == b.nc, kDimension, "add: shape mismatch");
  Csc c;
  c.nr = a.nr;
  c.nc = a.nc;
  c.cp.assign(a.nc + 1, 0);
  for (i32 j = 0; j < a.nc; ++j) {
    i64 pa = a.cp[j], ea = a.cp[j + 1], pb = b.cp[j], eb = b.cp[j + 1];
    while (pa < ea || pb < eb) {
      i32 ra = pa < ea ? a.ri[pa] : a.nr;
      i32 rb = pb < eb ? b.ri[pb] : b.nr;
      if (ra < rb) {
        c.ri.push_back(ra);
        c.v.push_back(alpha * a.v[pa++]);
      } else if (rb < ra) {
        c.ri.push_back(rb);
        c.v.push_back(beta * b.v[pb++]);
      } else {
        c.ri.push_back(ra);
        c.v.push_back(alpha * a.v[pa++] + beta * b.v[pb++]);
      }
    }
    c.cp[j + 1] = c.nnz();
  }
  return c;
}

Csc scale(const Csc& a, double s) {
  Csc c = a;
  for (double& v : c.v) v *= s;
  return c;
}

Csc scale_rows(const std::vector<double>& d, const Csc& a) {
  Csc c = a;
  for (i64 p = 0; p < c.nnz(); ++p) c.v[p] *= d[c.ri[p]];
  return c;
}

Csc scale_cols(const Csc& a, const std::vector<double>& d) {
  Csc c = a;
  for (i32 j = 0; j < c.nc; ++j)
    for (i64 p = c.cp[j]; p < c.cp[j + 1]; ++p) c.v[p] *= d[j];
  return c;
}

Csc symmetrize(const Csc& a) { return add(a, transpose(a), 0.5, 0.5); }

Csc diagonal(const std::vector<double>& d) {
  Csc m;
  m.nr = m.nc = static_cast<i32>(d.size());
  m.cp.resize(d.size() + 1);
  for (size_t i = 0; i <= d.size(); ++i) m.cp[i] = static_cast<i64>(i);
  m.ri.resize(d.size());
  for (size_t i = 0; i < d.size(); ++i) m.ri[i] = static_cast<i32>(i);
  m.v = d;
  return m;
}

// P1 element matrices in closed form (quadrature-exact for degree 2 rules,
// assembly.hpp:82-83,107): mass h/6·[[2,1],[1,2]], stiffness diff/h·[[1,-1],[-1,1]],
// advection c/2·[[-1,1],[-1,1]] (∫ φ_i c φ'_j). h is each element's own length
// from the node coordinates (mesh.hpp:44-46, 63-70): the nodes are rounded, so
// element lengths differ by ulps of the coordinates — relative 1e-13 of h at
// 1000 elements, which the ill-conditioned space-time precisions amplify.
Csc p1_mass(const Space1D& s) {
  std::vector<Trip> t;
  for (i32 e = 0; e < s.n_el; ++e) {
    const double h = s.x(e + 1) - s.x(e);
    const double d = h / 3.0, o = h / 6.0;
    t.push_back({e, e, d});
    t.push_back({e + 1, e, o});
    t.push_back({e, e + 1, o});
    t.push_back({e + 1, e + 1, d});
  }
  return csc_from_trips(s.n(), s.n(), std::move(t));
}

Csc p1_stiffness(const Space1D& s, double diff, double adv, double react) {
  std::vector<Trip> t;
  for (i32 e = 0; e < s.n_el; ++e) {
    const double h = s.x(e + 1) - s.x(e);
    double loc[2][2];
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) {
        const double gi = (i == 0 ? -1.0 : 1.0) / h, gj = (j == 0 ? -1.0 : 1.0) / h;
        // fused accumulations written out (std::fma), so the values do not depend on
        // the compiler's contraction choices and k_p1_interval reproduces them exactly
        double v = diff * gi * gj * h;
        v = std::fma(adv * gj * 0.5, h, v);
        v = std::fma(react * h, i == j ? 1.0 / 3.0 : 1.0 / 6.0, v);
        loc[i][j] = v;
      }
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) t.push_back({e + i, e + j, loc[i][j]});
  }
  return csc_from_trips(s.n(), s.n(), std::move(t));
}

// Triangles (v00, v10, v11) and (v00, v11, v01) per cell (mesh.hpp:140-147);
// P1 element mass |T|/12·(1 + δ_ij), stiffness |T| ∇φ_i·∇φ_j (exact).
namespace {
template <typename F>
void for_each_triangle(const Space2D& s, F&& f) {
  const i32 nc = s.n_cells, side = s.side();
  for (i32 iy = 0; iy < nc; ++iy)
    for (i32 ix = 0; ix < nc; ++ix) {
      const i32 v00 = iy * side + ix, v10 = v00 + 1, v11 = v00 + side + 1, v01 = v00 + side;
      const double x0 = s.coord(ix), y0 = s.coord(iy), x1 = s.coord(ix + 1), y1 = s.coord(iy + 1);
      const i32 t0[3] = {v00, v10, v11}, t1[3] = {v00, v11, v01};
      const double p0[3][2] = {{x0, y0}, {x1, y0}, {x1, y1}};
      const double p1[3][2] = {{x0, y0}, {x1, y1}, {x0, y1}};
      f(t0, p0);
      f(t1, p1);
    }
}
}  // namespace

Csc p1_mass(const Space2D& s) {
  std::vector<Trip> t;
  for_each_triangle(s, [&](const i32* v, const double (*p)[2]) {
    const double area = 0.5 * std::fma(p[1][0] - p[0][0], p[2][1] - p[0][1],
                                       -((p[2][0] - p[0][0]) * (p[1][1] - p[0][1])));
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) t.push_back({v[i], v[j], area / 12.0 * (i == j ? 2.0 : 1.0)});
  });
  return csc_from_trips(s.n(), s.n(), std::move(t));
}

Csc p1_laplace(const Space2D& s) {
  std::vector<Trip> t;
  for_each_triangle(s, [&](const i32* v, const double (*p)[2]) {
    const double det = std::fma(p[1][0] - p[0][0], p[2][1] - p[0][1],
                                -((p[2][0] - p[0][0]) * (p[1][1] - p[0][1])));
    const double area = 0.5 * det;
    double g[3][2];
    for (int i = 0; i < 3; ++i) {
      const int j = (i + 1) % 3, k = (i + 2) % 3;
      g[i][0] = (p[j][1] - p[k][1]) / det;
      g[i][1] = (p[k][0] - p[j][0]) / det;
    }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        // ∇φ_i·∇φ_j with the first product fused (written out so that the value does not
        // depend on the compiler's contraction choices; k_p1_square does the same)
        t.push_back({v[i], v[j], area * std::fma(g[i][0], g[j][0], g[i][1] * g[j][1])});
  });
  return csc_from_trips(s.n(), s.n(), std::move(t));
}

std::vector<char> dirichlet_mask(const Space1D& s, bool enabled) {
  std::vector<char> m(s.n(), 0);
  if (enabled) m.front() = m.back() = 1;
  return m;
}

namespace {
LumpFn g_lump = nullptr;
MaskFn g_mask = nullptr;
}  // namespace
void set_fem_hooks(LumpFn lump, MaskFn mask) {
  g_lump = lump;
  g_mask = mask;
}
Csc mask_constrained(const Csc& a, const std::vector<char>& mask, double diag) {
  return g_mask ? g_mask(a, mask, diag) : mask_constrained_host(a, mask, diag);
}
std::vector<double> lumped_mass(const Csc& m) { return g_lump ? g_lump(m) : lumped_mass_host(m); }

Csc mask_constrained_host(const Csc& a, const std::vector<char>& mask, double diag) {
  std::vector<Trip> t;
  for (i32 j = 0; j < a.nc; ++j)
    for (i64 p = a.cp[j]; p < a.cp[j + 1]; ++p)
      if (!mask[a.ri[p]] && !mask[j]) t.push_back({a.ri[p], j, a.v[p]});
  for (i32 j = 0; j < a.nc; ++j)
    if (mask[j]) t.push_back({j, j, diag});
  return csc_from_trips(a.nr, a.nc, std::move(t));
}

std::vector<double> lumped_mass_host(const Csc& m) {
  std::vector<double> d(m.nr, 0.0);
  for (i32 j = 0; j < m.nc; ++j)
    for (i64 p = m.cp[j]; p < m.cp[j + 1]; ++p) d[m.ri[p]] += m.v[p];
  for (double v : d) require(v > 0.0, kNumerical, "lumped mass: non-positive entry");
  return d;
}

SpatialOps spatial_ops(const Space1D& s, double diff, double adv, bool dirichlet) {
  SpatialOps o;
  o.n = s.n();
  o.mass = p1_mass(s);
  o.lap = p1_stiffness(s, 1.0, 0.0, 0.0);
  o.op = p1_stiffness(s, diff, adv, 0.0);
  o.slack = dirichlet_mask(s, dirichlet);
  return o;
}

SpatialOps spatial_ops(const Space2D& s, double diff) {
  SpatialOps o;
  o.n = s.n();
  o.mass = p1_mass(s);
  o.lap = p1_laplace(s);
  o.op = scale(o.lap, diff);  // laplace_operator(diff) (assembly.hpp:48)
  o.slack.assign(o.n, 0);     // natural boundary conditions
  return o;
}

MaternPrior matern_prior(const SpatialOps& ops, const MaternSpec& spec, double eps) {
  require(spec.kappa > 0 && spec.alpha >= 1 && spec.tau > 0, kContract, "matern: bad spec");
  const std::vector<char>& mask = ops.slack;
  const Csc& mass = ops.mass;
  Csc k = add(ops.lap, mass, 1.0, spec.kappa * spec.kappa);
  Csc k_hat = mask_constrained(k, mask, 1.0);
  Csc m_hat = mask_constrained(mass, mask, eps);
  std::vector<double> lum = lumped_mass(m_hat), inv(lum.size()), isq(lum.size());
  for (size_t i = 0; i < lum.size(); ++i) {
    inv[i] = 1.0 / lum[i];
    isq[i] = 1.0 / std::sqrt(lum[i]);
  }
  Csc kt = transpose(k_hat);
  Csc kt_minv = scale_cols(kt, inv);
  Csc q = scale(multiply(kt_minv, k_hat), 1.0 / (spec.tau * spec.tau));
  Csc l = scale(scale_cols(kt, isq), 1.0 / spec.tau);
  for (int a = spec.alpha; a >= 3; a -= 2) {
    q = multiply(kt_minv, multiply(q, transpose(kt_minv)));
    l = multiply(kt_minv, l);
  }
  return {symmetrize(q), l};
}

SpaceTimeBlocks spacetime_blocks(const SpatialOps& ops, double dt, double tau,
                                 const MaternSpec& noise, const MaternSpec& init, double eps) {
  SpaceTimeBlocks b;
  b.n = ops.n;
  b.eps = eps;
  b.slack = ops.slack;
  Csc k_hat = mask_constrained(ops.op, b.slack, 1.0);
  Csc m_hat = mask_constrained(ops.mass, b.slack, eps);
  MaternPrior nz = matern_prior(ops, noise, eps);
  MaternPrior in = matern_prior(ops, init, eps);
  std::vector<double> lum = lumped_mass(m_hat), inv(lum.size());
  for (size_t i = 0; i < lum.size(); ++i) inv[i] = 1.0 / lum[i];
  Csc w1 = scale_cols(m_hat, inv);
  Csc w1_qw = multiply(w1, nz.q);
  b.c_mm = multiply(w1_qw, transpose(w1));
  b.s_m = multiply(w1, nz.sqrt);
  Csc g = add(m_hat, k_hat, 1.0, dt);
  Csc v = scale_rows(inv, g);
  Csc vt = transpose(v);
  b.c_gg = multiply(multiply(vt, nz.q), v);
  b.c_mg = multiply(w1_qw, v);
  b.f_is = multiply(vt, nz.sqrt);
  b.t = 1.0 / (dt * tau * tau);
  b.q1 = in.q;
  b.l1 = in.sqrt;
  b.g_l1 = multiply(b.l1, transpose(b.l1));
  b.g_mm = multiply(b.s_m, transpose(b.s_m));
  b.g_ff = multiply(b.f_is, transpose(b.f_is));
  b.g_mf = multiply(b.s_m, transpose(b.f_is));
  return b;
}

}  // namespace gmrf
