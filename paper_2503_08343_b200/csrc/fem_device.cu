// Device P1 element assembly (see fem_device.hpp).
#include "fem_device.hpp"

#include <algorithm>
#include <string>

namespace gmrf {
namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
struct Tmp {
  T* p = nullptr;
  explicit Tmp(size_t n) { ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc (fem)"); }
  ~Tmp() { cudaFree(p); }
  Tmp(const Tmp&) = delete;
  Tmp& operator=(const Tmp&) = delete;
};

// node coordinate of the interval mesh (Space1D::x; build_interval_mesh, mesh.hpp:63-70)
__device__ __forceinline__ double node_x(int d, int n_el, double xa, double xb) {
  if (d == n_el) return xb;
  return __dadd_rn(xa, __ddiv_rn(__dmul_rn(__dadd_rn(xb, -xa), static_cast<double>(d)),
                                 static_cast<double>(n_el)));
}

// local matrix entry (i, j) of element e: which = 0 mass h/6·[[2,1],[1,2]] (as h/3, h/6);
// which = 1: diff·g_i g_j h + adv·g_j h/2 + react·h·(1/3 | 1/6), g = ∓1/h (p1_stiffness; the two
// accumulations fused, as there)
__device__ __forceinline__ double local_1d(int which, int e, int i, int j, int n_el, double xa,
                                           double xb, double diff, double adv, double react) {
  const double h = __dadd_rn(node_x(e + 1, n_el, xa, xb), -node_x(e, n_el, xa, xb));
  if (which == 0) return i == j ? __ddiv_rn(h, 3.0) : __ddiv_rn(h, 6.0);
  const double gi = __ddiv_rn(i == 0 ? -1.0 : 1.0, h), gj = __ddiv_rn(j == 0 ? -1.0 : 1.0, h);
  double v = __dmul_rn(__dmul_rn(__dmul_rn(diff, gi), gj), h);
  v = __fma_rn(__dmul_rn(__dmul_rn(adv, gj), 0.5), h, v);
  v = __fma_rn(__dmul_rn(react, h), i == j ? 1.0 / 3.0 : 1.0 / 6.0, v);
  return v;
}

// column c of the tridiagonal matrix: rows c-1, c, c+1; the diagonal sums element
// c-1 then element c (the triplet order of the element loop)
__global__ void k_p1_interval(int n_el, double xa, double xb, int which, double diff, double adv,
                              double react, const i64* __restrict__ cp, double* __restrict__ v) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > n_el) return;
  i64 p = cp[c];
  if (c > 0) v[p++] = local_1d(which, c - 1, 0, 1, n_el, xa, xb, diff, adv, react);
  double d = 0.0;
  if (c > 0) d = local_1d(which, c - 1, 1, 1, n_el, xa, xb, diff, adv, react);
  if (c < n_el) {
    const double d1 = local_1d(which, c, 0, 0, n_el, xa, xb, diff, adv, react);
    d = c > 0 ? __dadd_rn(d, d1) : d1;
  }
  v[p++] = d;
  if (c < n_el) v[p++] = local_1d(which, c, 1, 0, n_el, xa, xb, diff, adv, react);
}

// Unit square, cells split along the lower-left → upper-right diagonal (mesh.hpp:140-147):
// per cell the triangles (v00, v10, v11) and (v00, v11, v01). Entry (r, c) sums, in
// cell-major then triangle order, the local entries of the triangles holding both nodes.
__device__ __forceinline__ double coord(int i, int nc) {
  return __ddiv_rn(static_cast<double>(i), static_cast<double>(nc));
}

__device__ double tri_entry(int which, const int* v, const double (*p)[2], int r, int c,
                            bool& found) {
  int il = -1, jl = -1;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    if (v[q] == r) il = q;
    if (v[q] == c) jl = q;
  }
  found = il >= 0 && jl >= 0;
  if (!found) return 0.0;
  const double det = __fma_rn(__dadd_rn(p[1][0], -p[0][0]), __dadd_rn(p[2][1], -p[0][1]),
                              -__dmul_rn(__dadd_rn(p[2][0], -p[0][0]), __dadd_rn(p[1][1], -p[0][1])));
  const double area = __dmul_rn(0.5, det);
  if (which == 0) return __dmul_rn(__ddiv_rn(area, 12.0), il == jl ? 2.0 : 1.0);
  double g[3][2];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int j = (i + 1) % 3, k = (i + 2) % 3;
    g[i][0] = __ddiv_rn(__dadd_rn(p[j][1], -p[k][1]), det);
    g[i][1] = __ddiv_rn(__dadd_rn(p[k][0], -p[j][0]), det);
  }
  // first product fused, as the host closed form (p1_laplace)
  return __dmul_rn(area, __fma_rn(g[il][0], g[jl][0], __dmul_rn(g[il][1], g[jl][1])));
}

__global__ void k_p1_square(int nc, int which, double scale, const i64* __restrict__ cp,
                            const i32* __restrict__ ri, double* __restrict__ v) {
  const int side = nc + 1;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= side * side) return;
  const int cx = c % side, cy = c / side;
  for (i64 q = cp[c]; q < cp[c + 1]; ++q) {
    const int r = ri[q];
    double acc = 0.0;
    bool any = false;
    // cells touching the column node, ascending (iy, ix)
    for (int iy = cy - 1; iy <= cy; ++iy)
      for (int ix = cx - 1; ix <= cx; ++ix) {
        if (ix < 0 || iy < 0 || ix >= nc || iy >= nc) continue;
        const int v00 = iy * side + ix, v10 = v00 + 1, v11 = v00 + side + 1, v01 = v00 + side;
        const double x0 = coord(ix, nc), y0 = coord(iy, nc), x1 = coord(ix + 1, nc),
                     y1 = coord(iy + 1, nc);
        const int t0[3] = {v00, v10, v11}, t1[3] = {v00, v11, v01};
        const double p0[3][2] = {{x0, y0}, {x1, y0}, {x1, y1}};
        const double p1[3][2] = {{x0, y0}, {x1, y1}, {x0, y1}};
        bool f;
        double e = tri_entry(which, t0, p0, r, c, f);
        if (f) {
          acc = any ? __dadd_rn(acc, e) : e;
          any = true;
        }
        e = tri_entry(which, t1, p1, r, c, f);
        if (f) {
          acc = any ? __dadd_rn(acc, e) : e;
          any = true;
        }
      }
    v[q] = which == 1 && scale != 1.0 ? __dmul_rn(acc, scale) : acc;
  }
}

// row sums of a symmetric CSC = column sums in row order (lumped_mass)
__global__ void k_lump_columns(int n, const i64* __restrict__ cp, const double* __restrict__ v,
                               double* __restrict__ d) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double s = 0.0;
  for (i64 p = cp[c]; p < cp[c + 1]; ++p) s = __dadd_rn(s, v[p]);
  d[c] = s;
}

// out[k] = src[k] >= 0 ? in[src[k]] : fill   (constraint folding with T = I)
__global__ void k_gather_values(i64 n, const i64* __restrict__ src, const double* __restrict__ in,
                                double fill, double* __restrict__ out) {
  const i64 k = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (k < n) out[k] = src[k] >= 0 ? in[src[k]] : fill;
}

Csc pattern_1d(i32 n_el) {
  Csc m;
  m.nr = m.nc = n_el + 1;
  m.cp.assign(1, 0);
  for (i32 c = 0; c <= n_el; ++c) {
    for (i32 r = std::max(0, c - 1); r <= std::min(n_el, c + 1); ++r) m.ri.push_back(r);
    m.cp.push_back(m.nnz());
  }
  m.v.assign(m.ri.size(), 0.0);
  return m;
}

Csc pattern_2d(i32 nc) {
  const i32 side = nc + 1;
  Csc m;
  m.nr = m.nc = side * side;
  m.cp.assign(1, 0);
  // neighbours sharing a triangle: (±1, 0), (0, ±1), (+1, +1), (-1, -1)
  const int dx[7] = {-1, 0, -1, 0, 1, 0, 1}, dy[7] = {-1, -1, 0, 0, 0, 1, 1};
  for (i32 cy = 0; cy < side; ++cy)
    for (i32 cx = 0; cx < side; ++cx) {
      for (int q = 0; q < 7; ++q) {
        const i32 x = cx + dx[q], y = cy + dy[q];
        if (x >= 0 && y >= 0 && x < side && y < side) m.ri.push_back(y * side + x);
      }
      m.cp.push_back(m.nnz());
    }
  m.v.assign(m.ri.size(), 0.0);
  return m;
}

constexpr int kT = 128;
inline unsigned blocks(i64 n) { return static_cast<unsigned>((n + kT - 1) / kT); }

}  // namespace

Csc p1_matrix_device(int dim, i32 n_el, double xa, double xb, int which, double diff, double adv,
                     double react, cudaStream_t st) {
  require(dim == 1 || dim == 2, kContract, "p1 assembly: dim must be 1 or 2");
  require(n_el >= 1, kContract, "p1 assembly: empty mesh");
  Csc m = dim == 1 ? pattern_1d(n_el) : pattern_2d(n_el);
  Tmp<i64> cp(m.cp.size());
  Tmp<i32> ri(m.ri.size());
  Tmp<double> v(m.v.size());
  ck(cudaMemcpyAsync(cp.p, m.cp.data(), m.cp.size() * 8, cudaMemcpyHostToDevice, st), "copy");
  ck(cudaMemcpyAsync(ri.p, m.ri.data(), m.ri.size() * 4, cudaMemcpyHostToDevice, st), "copy");
  if (dim == 1)
    k_p1_interval<<<blocks(m.nc), kT, 0, st>>>(n_el, xa, xb, which, diff, adv, react, cp.p, v.p);
  else
    k_p1_square<<<blocks(m.nc), kT, 0, st>>>(n_el, which, diff, cp.p, ri.p, v.p);
  ck(cudaGetLastError(), "p1 assembly launch");
  ck(cudaMemcpyAsync(m.v.data(), v.p, m.v.size() * 8, cudaMemcpyDeviceToHost, st), "copy");
  ck(cudaStreamSynchronize(st), "p1 assembly");
  return m;
}

SpatialOps spatial_ops_device(const Space1D& s, double diff, double adv, bool dirichlet,
                              cudaStream_t st) {
  SpatialOps o;
  o.n = s.n();
  o.mass = p1_matrix_device(1, s.n_el, s.xa, s.xb, 0, 0.0, 0.0, 0.0, st);
  o.lap = p1_matrix_device(1, s.n_el, s.xa, s.xb, 1, 1.0, 0.0, 0.0, st);
  o.op = p1_matrix_device(1, s.n_el, s.xa, s.xb, 1, diff, adv, 0.0, st);
  o.slack = dirichlet_mask(s, dirichlet);
  return o;
}

SpatialOps spatial_ops_device(const Space2D& s, double diff, cudaStream_t st) {
  SpatialOps o;
  o.n = s.n();
  o.mass = p1_matrix_device(2, s.n_cells, 0.0, 1.0, 0, 1.0, 0.0, 0.0, st);
  o.lap = p1_matrix_device(2, s.n_cells, 0.0, 1.0, 1, 1.0, 0.0, 0.0, st);
  o.op = p1_matrix_device(2, s.n_cells, 0.0, 1.0, 1, diff, 0.0, 0.0, st);  // laplace_operator(diff)
  o.slack.assign(o.n, 0);
  return o;
}

std::vector<double> lumped_mass_device(const Csc& m, cudaStream_t st) {
  Tmp<i64> cp(m.cp.size());
  Tmp<double> v(m.v.size()), d(m.nr);
  ck(cudaMemcpyAsync(cp.p, m.cp.data(), m.cp.size() * 8, cudaMemcpyHostToDevice, st), "copy");
  ck(cudaMemcpyAsync(v.p, m.v.data(), m.v.size() * 8, cudaMemcpyHostToDevice, st), "copy");
  k_lump_columns<<<blocks(m.nc), kT, 0, st>>>(m.nc, cp.p, v.p, d.p);
  ck(cudaGetLastError(), "lumped mass launch");
  std::vector<double> out(m.nr);
  ck(cudaMemcpyAsync(out.data(), d.p, out.size() * 8, cudaMemcpyDeviceToHost, st), "copy");
  ck(cudaStreamSynchronize(st), "lumped mass");
  for (double x : out) require(x > 0.0, kNumerical, "lumped mass: non-positive entry");
  return out;
}

Csc mask_constrained_device(const Csc& a, const std::vector<char>& mask, double diag,
                            cudaStream_t st) {
  // pattern and source map on the host (structure only), values on the device
  Csc m;
  m.nr = a.nr;
  m.nc = a.nc;
  m.cp.assign(1, 0);
  std::vector<i64> src;
  for (i32 j = 0; j < a.nc; ++j) {
    bool diag_done = !mask[j];
    for (i64 p = a.cp[j]; p < a.cp[j + 1]; ++p) {
      const i32 r = a.ri[p];
      if (mask[j]) {
        if (!diag_done && r >= j) {
          m.ri.push_back(j);
          src.push_back(-1);
          diag_done = true;
        }
        continue;
      }
      if (!mask[r]) {
        m.ri.push_back(r);
        src.push_back(p);
      }
    }
    if (!diag_done) {
      m.ri.push_back(j);
      src.push_back(-1);
    }
    m.cp.push_back(m.nnz());
  }
  m.v.assign(m.ri.size(), 0.0);
  Tmp<i64> ds(src.size());
  Tmp<double> in(a.v.size()), out(src.size());
  ck(cudaMemcpyAsync(ds.p, src.data(), src.size() * 8, cudaMemcpyHostToDevice, st), "copy");
  ck(cudaMemcpyAsync(in.p, a.v.data(), a.v.size() * 8, cudaMemcpyHostToDevice, st), "copy");
  k_gather_values<<<blocks(static_cast<i64>(src.size())), kT, 0, st>>>(
      static_cast<i64>(src.size()), ds.p, in.p, diag, out.p);
  ck(cudaGetLastError(), "constraint fold launch");
  ck(cudaMemcpyAsync(m.v.data(), out.p, m.v.size() * 8, cudaMemcpyDeviceToHost, st), "copy");
  ck(cudaStreamSynchronize(st), "constraint fold");
  return m;
}


FemDeviceScope::FemDeviceScope() {
  set_fem_hooks([](const Csc& m) { return lumped_mass_device(m); },
                [](const Csc& a, const std::vector<char>& k, double d) {
                  return mask_constrained_device(a, k, d);
                });
}
FemDeviceScope::~FemDeviceScope() { set_fem_hooks(nullptr, nullptr); }

}  // namespace gmrf
