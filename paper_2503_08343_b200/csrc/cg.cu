// Preconditioned conjugate gradients on the device (core/cg.hpp:39-95, the
// matrix-backed overload :98-105) and CG posterior sampling (sample_cg,
// gmrf.hpp:188-202): the matrix-free alternative to the factorization when L
// does not fit.
//
// Same recurrence, stopping rule and breakdown check as the reference:
// r = b − Qx0, target = max(rtol‖b‖, atol), z = r (or r ./ diag(Q) for
// Jacobi), p = z; per iteration α = rᵀz / pᵀQp (pᵀQp ≤ 0 raises), x += αp,
// r −= αq, stop when ‖r‖ ≤ target, β = r'ᵀz' / rᵀz, p = z + βp. The scalars
// live on the device: every kernel of an iteration reads them there, and once
// the stopping rule holds the remaining launched iterations are no-ops, so the
// host checks convergence only every kCgBatch iterations without changing
// where the iteration stops. Q·v is a row gather over a CSR copy of Q (the
// per-row accumulation order of matvec, sparse.hpp); dot products are a fixed
// two-stage tree (deterministic, not the reference's sequential sum).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "cg.hpp"
#include "factor.hpp"

namespace gmrf {

namespace {

constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 296;  // 2 per SM
constexpr int kCgBatch = 8;

// device-side CG scalars
struct CgState {
  double rz, pq, alpha, beta, rnorm, target;
  long long it, max_iter;
  int done, converged, breakdown;
};

__global__ void k_csr_spmv(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const double* __restrict__ v, const double* __restrict__ x,
                           double* __restrict__ y, const CgState* __restrict__ st) {
  if (st && st->done) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) s = __dadd_rn(s, __dmul_rn(v[p], x[ci[p]]));
    y[i] = s;
  }
}

__device__ __forceinline__ void block_sum_store(double s, double* out) {
  __shared__ double sh[kRedThreads];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = kRedThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// part[b] = Σ a_i c_i over block b's grid-stride slice
__global__ void __launch_bounds__(kRedThreads) k_dot_part(int n, const double* __restrict__ a,
                                                          const double* __restrict__ c,
                                                          double* __restrict__ part,
                                                          const CgState* __restrict__ st) {
  if (st && st->done) return;
  double s = 0.0;
  for (int i = blockIdx.x * kRedThreads + threadIdx.x; i < n; i += kRedBlocks * kRedThreads)
    s = __dadd_rn(s, __dmul_rn(a[i], c[i]));
  block_sum_store(s, part + blockIdx.x);
}

__device__ __forceinline__ double sum_parts(const double* part) {
  __shared__ double sh[512];
  const int t = threadIdx.x;
  sh[t] = t < kRedBlocks ? part[t] : 0.0;
  __syncthreads();
  for (int o = 256; o > 0; o >>= 1) {
    if (t < o) sh[t] = __dadd_rn(sh[t], sh[t + o]);
    __syncthreads();
  }
  return sh[0];
}

// r = b − q, z = precond(r)
__global__ void k_cg_init_r(int n, const double* __restrict__ b, const double* __restrict__ q,
                            const double* __restrict__ diag, double* __restrict__ r,
                            double* __restrict__ z, double* __restrict__ p) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double ri = __dadd_rn(b[i], -q[i]);
    const double zi = diag ? __ddiv_rn(ri, diag[i]) : ri;
    r[i] = ri;
    z[i] = zi;
    p[i] = zi;
  }
}

// which = 0: rz = Σ (initial); 1: pq → α (breakdown check); 2: ‖r‖ → stop rule;
// 3: rz' → β; 4: initial ‖r‖ → stop rule at iteration 0; 5: ‖b‖ → target
__global__ void k_cg_scalar(const double* __restrict__ part, CgState* __restrict__ st, int which,
                            double rtol, double atol) {
  if (which != 0 && which != 4 && which != 5 && st->done) return;
  const double s = sum_parts(part);
  if (threadIdx.x != 0) return;
  switch (which) {
    case 0: st->rz = s; break;
    case 1:
      st->pq = s;
      if (!(s > 0.0)) {
        st->breakdown = 1;
        st->done = 1;
      } else {
        st->alpha = __ddiv_rn(st->rz, s);
      }
      break;
    case 2:
      st->rnorm = sqrt(s);
      st->it += 1;
      if (st->rnorm <= st->target) {
        st->converged = 1;
        st->done = 1;
      } else if (st->it >= st->max_iter) {
        st->done = 1;
      }
      break;
    case 3: {
      st->beta = __ddiv_rn(s, st->rz);
      st->rz = s;
      break;
    }
    case 4:
      st->rnorm = sqrt(s);
      if (st->rnorm <= st->target) {
        st->converged = 1;
        st->done = 1;
      }
      break;
    case 5: st->target = fmax(rtol * sqrt(s), atol); break;
  }
}

// x += α p; r −= α q
__global__ void k_cg_update(int n, const double* __restrict__ p, const double* __restrict__ q,
                            double* __restrict__ x, double* __restrict__ r,
                            const CgState* __restrict__ st) {
  if (st->done) return;
  const double a = st->alpha;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(a, p[i]));
    r[i] = __dadd_rn(r[i], __dmul_rn(-a, q[i]));
  }
}

__global__ void k_cg_precond(int n, const double* __restrict__ r, const double* __restrict__ diag,
                             double* __restrict__ z, const CgState* __restrict__ st) {
  if (st->done) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    z[i] = diag ? __ddiv_rn(r[i], diag[i]) : r[i];
}

__global__ void k_cg_newp(int n, const double* __restrict__ z, double* __restrict__ p,
                          const CgState* __restrict__ st) {
  if (st->done) return;
  const double b = st->beta;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = __dadd_rn(z[i], __dmul_rn(b, p[i]));
}

__global__ void k_csr_diag(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const double* __restrict__ v, double* __restrict__ d) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] == i) s = v[p];
    d[i] = s;
  }
}

// CSC (nrows × ncols) → CSR, rows ascending columns (host)
void csc_to_csr(int nrows, int ncols, const int64_t* cp, const int32_t* ri, const double* v,
                std::vector<int64_t>& rp, std::vector<int32_t>& ci, std::vector<double>& vv) {
  const int64_t nnz = cp[ncols];
  rp.assign(nrows + 1, 0);
  for (int64_t p = 0; p < nnz; ++p) {
    require(ri[p] >= 0 && ri[p] < nrows, kStructural, "cg: row index out of range");
    rp[ri[p] + 1]++;
  }
  for (int i = 0; i < nrows; ++i) rp[i + 1] += rp[i];
  ci.resize(nnz);
  vv.resize(nnz);
  std::vector<int64_t> nx(rp.begin(), rp.end() - 1);
  for (int j = 0; j < ncols; ++j)
    for (int64_t p = cp[j]; p < cp[j + 1]; ++p) {
      const int64_t q = nx[ri[p]]++;
      ci[q] = j;
      vv[q] = v[p];
    }
}

inline int grid1(int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)));
}

}  // namespace

CgOutcome cg_solve_device(int n, const int64_t* cp, const int32_t* ri, const double* v,
                          const double* b, const double* x0, const CgOptions& opt, double* x,
                          cudaStream_t stream) {
  require(opt.rtol > 0.0, kContract, "cg: rtol must be positive");
  require(opt.max_iter >= 0, kContract, "cg: max_iter must be >= 1");
  CgOutcome res;
  if (n == 0) {
    res.converged = true;
    return res;
  }
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> vv;
  csc_to_csr(n, n, cp, ri, v, rp, ci, vv);
  DevBuf<int64_t> d_rp;
  DevBuf<int32_t> d_ci;
  DevBuf<double> d_v, d_b, d_x, d_r, d_z, d_p, d_q, d_diag, part;
  DevBuf<CgState> st;
  d_rp.upload(rp, stream);
  d_ci.upload(ci, stream);
  d_v.upload(vv, stream);
  for (DevBuf<double>* bf : {&d_b, &d_x, &d_r, &d_z, &d_p, &d_q}) bf->alloc(n);
  part.alloc(kRedBlocks);
  st.alloc(1);
  cuda_check(cudaMemcpyAsync(d_b.p, b, sizeof(double) * n, cudaMemcpyHostToDevice, stream), "b");
  if (x0) cuda_check(cudaMemcpyAsync(d_x.p, x0, sizeof(double) * n, cudaMemcpyHostToDevice, stream),
                     "x0");
  else cuda_check(cudaMemsetAsync(d_x.p, 0, sizeof(double) * n, stream), "x0");
  const double* diag = nullptr;
  const int g = grid1(n);
  if (opt.jacobi) {  // csc_diag(q) (sparse.hpp:113), as the matrix-backed overload
    d_diag.alloc(n);
    k_csr_diag<<<g, 256, 0, stream>>>(n, d_rp.p, d_ci.p, d_v.p, d_diag.p);
    diag = d_diag.p;
  }
  CgState h{};
  h.max_iter = opt.max_iter > 0 ? opt.max_iter : 10LL * n;
  cuda_check(cudaMemcpyAsync(st.p, &h, sizeof(CgState), cudaMemcpyHostToDevice, stream), "state");
  // r = b − Q x0, target, z, p, rz, ‖r‖
  k_csr_spmv<<<g, 256, 0, stream>>>(n, d_rp.p, d_ci.p, d_v.p, d_x.p, d_q.p, nullptr);
  k_cg_init_r<<<g, 256, 0, stream>>>(n, d_b.p, d_q.p, diag, d_r.p, d_z.p, d_p.p);
  k_dot_part<<<kRedBlocks, kRedThreads, 0, stream>>>(n, d_b.p, d_b.p, part.p, nullptr);
  k_cg_scalar<<<1, 512, 0, stream>>>(part.p, st.p, 5, opt.rtol, opt.atol);
  k_dot_part<<<kRedBlocks, kRedThreads, 0, stream>>>(n, d_r.p, d_z.p, part.p, nullptr);
  k_cg_scalar<<<1, 512, 0, stream>>>(part.p, st.p, 0, 0, 0);
  k_dot_part<<<kRedBlocks, kRedThreads, 0, stream>>>(n, d_r.p, d_r.p, part.p, nullptr);
  k_cg_scalar<<<1, 512, 0, stream>>>(part.p, st.p, 4, 0, 0);
  for (;;) {
    cuda_check(cudaMemcpyAsync(&h, st.p, sizeof(CgState), cudaMemcpyDeviceToHost, stream), "state");
    cuda_check(cudaStreamSynchronize(stream), "cg");
    if (h.done) break;
    for (int k = 0; k < kCgBatch; ++k) {
      k_csr_spmv<<<g, 256, 0, stream>>>(n, d_rp.p, d_ci.p, d_v.p, d_p.p, d_q.p, st.p);
      k_dot_part<<<kRedBlocks, kRedThreads, 0, stream>>>(n, d_p.p, d_q.p, part.p, st.p);
      k_cg_scalar<<<1, 512, 0, stream>>>(part.p, st.p, 1, 0, 0);
      k_cg_update<<<g, 256, 0, stream>>>(n, d_p.p, d_q.p, d_x.p, d_r.p, st.p);
      k_dot_part<<<kRedBlocks, kRedThreads, 0, stream>>>(n, d_r.p, d_r.p, part.p, st.p);
      k_cg_scalar<<<1, 512, 0, stream>>>(part.p, st.p, 2, 0, 0);
      k_cg_precond<<<g, 256, 0, stream>>>(n, d_r.p, diag, d_z.p, st.p);
      k_dot_part<<<kRedBlocks, kRedThreads, 0, stream>>>(n, d_r.p, d_z.p, part.p, st.p);
      k_cg_scalar<<<1, 512, 0, stream>>>(part.p, st.p, 3, 0, 0);
      k_cg_newp<<<g, 256, 0, stream>>>(n, d_z.p, d_p.p, st.p);
    }
    cuda_check(cudaGetLastError(), "cg launch");
  }
  if (h.breakdown)
    fail(kNumerical, "cg: non-positive curvature, operator not SPD (pᵀQp = " +
                         std::to_string(h.pq) + ")");
  cuda_check(cudaMemcpyAsync(x, d_x.p, sizeof(double) * n, cudaMemcpyDeviceToHost, stream), "x");
  cuda_check(cudaStreamSynchronize(stream), "cg result");
  res.iterations = h.it;
  res.final_residual = h.rnorm;
  res.converged = h.converged != 0;
  return res;
}

void sample_cg_device(int n, const int64_t* qcp, const int32_t* qri, const double* qv, int m,
                      const int64_t* scp, const int32_t* sri, const double* sv,
                      const double* mean, const double* z, const CgOptions& opt, double* out,
                      cudaStream_t stream) {
  // b = S z (matvec, sparse.hpp) as a row gather over CSR(S)
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> vv;
  csc_to_csr(n, m, scp, sri, sv, rp, ci, vv);
  DevBuf<int64_t> d_rp;
  DevBuf<int32_t> d_ci;
  DevBuf<double> d_v, d_z, d_b;
  d_rp.upload(rp, stream);
  d_ci.upload(ci, stream);
  d_v.upload(vv, stream);
  d_z.alloc(std::max(m, 1));
  d_b.alloc(std::max(n, 1));
  if (m) cuda_check(cudaMemcpyAsync(d_z.p, z, sizeof(double) * m, cudaMemcpyHostToDevice, stream), "z");
  k_csr_spmv<<<grid1(n), 256, 0, stream>>>(n, d_rp.p, d_ci.p, d_v.p, d_z.p, d_b.p, nullptr);
  std::vector<double> b(n), x(n);
  cuda_check(cudaMemcpyAsync(b.data(), d_b.p, sizeof(double) * n, cudaMemcpyDeviceToHost, stream),
             "b");
  cuda_check(cudaStreamSynchronize(stream), "sample_cg");
  CgOutcome r = cg_solve_device(n, qcp, qri, qv, b.data(), nullptr, opt, x.data(), stream);
  if (!r.converged)
    fail(kNumerical, "sample_cg: CG did not reach tolerance after " + std::to_string(r.iterations) +
                         " iterations (residual " + std::to_string(r.final_residual) + ")");
  for (int i = 0; i < n; ++i) out[i] = mean[i] + x[i];  // vec_add (gmrf.hpp:201)
}

}  // namespace gmrf
