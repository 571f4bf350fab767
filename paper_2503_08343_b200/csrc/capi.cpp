// C-ABI entry points (include/gmrf_b200.h).
#include "../../include/gmrf_b200.h"

#include <algorithm>
#include <cstddef>
#include <cstring>
#include <memory>
#include <string>
#include <tuple>

#include "cg.hpp"
#include "factor.hpp"
#include "partition.hpp"
#include "rng.hpp"
#include "gram.hpp"
#include "regression.hpp"
#include "update_system.hpp"
#include "spacetime.hpp"

static_assert(sizeof(gmrf_msg_t) == sizeof(gmrf::XferMsg), "gmrf_msg_t layout");
static_assert(offsetof(gmrf_msg_t, dptr) == offsetof(gmrf::XferMsg, dptr), "gmrf_msg_t layout");
static_assert(offsetof(gmrf_msg_t, count) == offsetof(gmrf::XferMsg, count), "gmrf_msg_t layout");
#include "symbolic.hpp"

struct gmrf_symbolic {
  std::shared_ptr<const gmrf::Symbolic> s;
};
struct gmrf_factor {
  std::shared_ptr<const gmrf::Symbolic> s;
  std::unique_ptr<gmrf::DeviceFactor> f;
};
struct gmrf_gram {
  std::shared_ptr<const gmrf::Symbolic> s;
  std::unique_ptr<gmrf::GramPlan> g;
  gmrf::i32 m = 0;
  gmrf::DevBuf<double> a, w, base, out;
};
struct gmrf_regression {
  std::unique_ptr<gmrf::RegressionPosterior> p;
  gmrf_factor wrap;  // borrowed view of p's factor for the gmrf_factor_* entry points
};
struct gmrf_update_system {
  std::unique_ptr<gmrf::UpdateSystem> u;
  gmrf_symbolic sym;  // views
  gmrf_factor fac;
};
struct gmrf_spacetime {
  gmrf::GnConfig cfg;
  std::unique_ptr<gmrf::SpaceTimePosterior> p;
  gmrf::DevBuf<double> tmp;
};

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& fn) {
  try {
    fn();
    return GMRF_OK;
  } catch (const gmrf::Error& e) {
    g_err = e.what();
    return e.status;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GMRF_ERR_NUMERICAL;
  }
}
}  // namespace

extern "C" {

const char* gmrf_last_error(void) { return g_err.c_str(); }
int gmrf_version(void) { return 1; }

int gmrf_nd_order(int32_t n, const int64_t* cp, const int32_t* ri, int32_t* perm) {
  return guard([&] {
    auto p = gmrf::nd_order(n, cp, ri);
    std::memcpy(perm, p.data(), sizeof(int32_t) * n);
  });
}

int gmrf_symbolic_analyze(int32_t n, const int64_t* cp, const int32_t* ri, const int32_t* perm,
                          gmrf_symbolic_t** out) {
  return guard([&] {
    auto h = std::make_unique<gmrf_symbolic>();
    h->s = std::make_shared<const gmrf::Symbolic>(gmrf::analyze(n, cp, ri, perm));
    *out = h.release();
  });
}

int gmrf_symbolic_info(const gmrf_symbolic_t* h, gmrf_symbolic_info_t* info) {
  return guard([&] {
    const gmrf::Symbolic& s = *h->s;
    info->n = s.n;
    info->nnz_q = static_cast<int64_t>(s.qri.size());
    info->nnz_l = s.nnz_l;
    info->nnz_l_padded = s.nnz_l_padded;
    info->update_entries = s.uptr.empty() ? 0 : s.uptr[s.ns];
    info->n_supernodes = s.ns;
    info->n_levels = s.n_levels;
    info->etree_height = s.etree_height;
    int mf = 0;
    for (int k = 0; k < s.ns; ++k) mf = std::max(mf, s.rows(k));
    info->max_front = mf;
    info->flops_ref = s.flops_ref;
    info->flops_sn = s.flops_sn;
  });
}

int gmrf_symbolic_export(const gmrf_symbolic_t* h, int32_t* perm, int32_t* parent,
                         int64_t* cpl) {
  return guard([&] {
    const gmrf::Symbolic& s = *h->s;
    if (perm) std::memcpy(perm, s.perm.data(), sizeof(int32_t) * s.n);
    if (parent) std::memcpy(parent, s.parent.data(), sizeof(int32_t) * s.n);
    if (cpl) std::memcpy(cpl, s.colptr_l.data(), sizeof(int64_t) * (s.n + 1));
  });
}

void gmrf_symbolic_free(gmrf_symbolic_t* h) { delete h; }

int gmrf_symbolic_supernodes(const gmrf_symbolic_t* h, int32_t* first, int32_t* rows,
                             int32_t* level, int32_t* parent) {
  return guard([&] {
    const gmrf::Symbolic& s = *h->s;
    for (int k = 0; k < s.ns; ++k) {
      if (first) first[k] = s.sn_first[k];
      if (rows) rows[k] = s.rows(k);
      if (level) level[k] = s.sn_level[k];
      if (parent) parent[k] = s.sn_parent[k];
    }
    if (first) first[s.ns] = s.n;
  });
}

int gmrf_factor_create(const gmrf_symbolic_t* h, gmrf_factor_t** out) {
  return guard([&] {
    auto f = std::make_unique<gmrf_factor>();
    f->s = h->s;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      gmrf::fail(gmrf::kCuda, "no CUDA device: libgmrf_b200 has no CPU fallback");
    f->f = std::make_unique<gmrf::DeviceFactor>(h->s);
    *out = f.release();
  });
}

static gmrf::CgOptions cg_opts(const gmrf_cg_config_t* c) {
  gmrf::CgOptions o;
  if (c) {
    o.rtol = c->rtol;
    o.atol = c->atol;
    o.max_iter = c->max_iter;
    gmrf::require(c->preconditioner == 0 || c->preconditioner == 1, gmrf::kContract,
                  "cg: unknown preconditioner");
    o.jacobi = c->preconditioner == 1;
  }
  return o;
}

static void need_device() {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    gmrf::fail(gmrf::kCuda, "no CUDA device: libgmrf_b200 has no CPU fallback");
}

int gmrf_cg_solve(int32_t n, const int64_t* cp, const int32_t* ri, const double* v,
                  const double* b, const double* x0, const gmrf_cg_config_t* cfg, double* x,
                  gmrf_cg_result_t* res) {
  return guard([&] {
    need_device();
    gmrf::CgOutcome r = gmrf::cg_solve_device(n, cp, ri, v, b, x0, cg_opts(cfg), x);
    if (res) *res = {r.iterations, r.final_residual, r.converged ? 1 : 0};
  });
}

int gmrf_sample_cg(int32_t n, const int64_t* qcp, const int32_t* qri, const double* qv,
                   int32_t m, const int64_t* scp, const int32_t* sri, const double* sv,
                   const double* mean, const double* z, const gmrf_cg_config_t* cfg,
                   double* out) {
  return guard([&] {
    need_device();
    gmrf::sample_cg_device(n, qcp, qri, qv, m, scp, sri, sv, mean, z, cg_opts(cfg), out);
  });
}

int gmrf_partition_owners(const gmrf_symbolic_t* h, int32_t nranks, int32_t* owner) {
  return guard([&] {
    gmrf::require(nranks >= 1, gmrf::kContract, "partition: nranks < 1");
    auto o = gmrf::partition_owners(*h->s, nranks);
    std::copy(o.begin(), o.end(), owner);
  });
}

int gmrf_partition_schedule(const gmrf_symbolic_t* h, const int32_t* owner, int64_t* rows,
                            int64_t* n_rows) {
  return guard([&] {
    const gmrf::Symbolic& s = *h->s;
    std::vector<int32_t> o(owner, owner + s.ns);
    auto e = gmrf::partition_schedule(s, o);
    if (n_rows) *n_rows = static_cast<int64_t>(e.size());
    if (rows)
      for (size_t i = 0; i < e.size(); ++i) {
        int64_t* r = rows + 6 * i;
        r[0] = e[i].phase;
        r[1] = e[i].point;
        r[2] = e[i].src;
        r[3] = e[i].dst;
        r[4] = e[i].sn;
        r[5] = e[i].count;
      }
  });
}

int gmrf_factor_set_selinv_inplace(gmrf_factor_t* f, int32_t on) {
  return guard([&] { f->f->set_selinv_inplace(on != 0); });
}

int gmrf_partition_memory(const gmrf_symbolic_t* s, int32_t nranks, const int32_t* owner,
                          int64_t* rows) {
  return guard([&] {
    gmrf::require(nranks >= 1, gmrf::kContract, "partition: nranks >= 1");
    std::vector<int32_t> own = owner ? std::vector<int32_t>(owner, owner + s->s->ns)
                                     : gmrf::partition_owners(*s->s, nranks);
    const auto mem = gmrf::partition_memory(*s->s, own, nranks);
    for (int r = 0; r < nranks; ++r) {
      const gmrf::RankMemory& m = mem[r];
      const int64_t v[7] = {m.l_panels, m.sigma_panels, m.u_arena_factor, m.u_arena_selinv,
                            m.replicated, m.total(), m.supernodes};
      std::memcpy(rows + 7 * r, v, sizeof(v));
    }
  });
}

int gmrf_factor_create_partitioned(const gmrf_symbolic_t* h, int32_t nranks, int32_t rank,
                                   const int32_t* owner, gmrf_exchange_fn fn, void* ctx,
                                   gmrf_factor_t** out) {
  return guard([&] {
    auto f = std::make_unique<gmrf_factor>();
    f->s = h->s;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      gmrf::fail(gmrf::kCuda, "no CUDA device: libgmrf_b200 has no CPU fallback");
    gmrf::PartitionSpec ps;
    ps.nranks = nranks;
    ps.rank = rank;
    if (owner) ps.owner.assign(owner, owner + h->s->ns);
    ps.fn = reinterpret_cast<gmrf::ExchangeFn>(fn);
    ps.ctx = ctx;
    f->f = std::make_unique<gmrf::DeviceFactor>(h->s, nullptr, &ps);
    *out = f.release();
  });
}

int gmrf_factor_set_stream(gmrf_factor_t* f, void* stream) {
  return guard([&] { f->f->set_stream(static_cast<cudaStream_t>(stream)); });
}

static int numeric_impl(gmrf_factor_t* f, const double* q, bool dev, int32_t* bad) {
  int32_t b = -1;
  int rc = guard([&] { b = f->f->numeric(q, dev); });
  if (bad) *bad = b;
  if (rc != GMRF_OK) return rc;
  if (b >= 0) {
    g_err = "cholesky: non-positive pivot at index " + std::to_string(b);
    return GMRF_ERR_NOT_SPD;
  }
  return GMRF_OK;
}

int gmrf_factor_numeric(gmrf_factor_t* f, const double* q, int32_t* bad) {
  return numeric_impl(f, q, false, bad);
}
int gmrf_factor_numeric_device(gmrf_factor_t* f, const double* q, int32_t* bad) {
  return numeric_impl(f, q, true, bad);
}

int gmrf_solve(gmrf_factor_t* f, int mode, int32_t nrhs, const double* b, double* x) {
  return guard([&] { f->f->solve(mode, nrhs, b, x, false); });
}
int gmrf_solve_device(gmrf_factor_t* f, int mode, int32_t nrhs, const double* b, double* x) {
  return guard([&] { f->f->solve(mode, nrhs, b, x, true); });
}

int gmrf_selinv_diag(gmrf_factor_t* f, double* d) {
  return guard([&] { f->f->selinv(d, false); });
}
int gmrf_selinv_diag_device(gmrf_factor_t* f, double* d) {
  return guard([&] { f->f->selinv(d, true); });
}

int gmrf_sample_direct(gmrf_factor_t* f, const double* mean, int32_t ns, uint64_t seed,
                       double* out) {
  return guard([&] {
    const int n = f->s->n;
    gmrf::require(ns >= 0, gmrf::kContract, "sample_direct: negative sample count");
    if (n == 0 || ns == 0) return;
    gmrf::DevBuf<double> m, o;
    m.alloc(n);
    o.alloc(static_cast<size_t>(n) * ns);
    gmrf::cuda_check(cudaMemcpy(m.p, mean, sizeof(double) * n, cudaMemcpyHostToDevice), "mean");
    f->f->sample_direct(m.p, ns, seed, o.p);
    gmrf::cuda_check(cudaMemcpy(out, o.p, sizeof(double) * n * static_cast<size_t>(ns),
                                cudaMemcpyDeviceToHost), "samples");
  });
}

int gmrf_rbmc_variance(gmrf_factor_t* f, const double* qv, const double* mean, int32_t ns,
                       uint64_t seed, double* var) {
  return guard([&] {
    const int n = f->s->n;
    gmrf::require(ns >= 2, gmrf::kContract, "rbmc_variance: need at least 2 samples");
    if (n == 0) return;
    const size_t nnz = f->s->qri.size();
    gmrf::DevBuf<double> q, m, v;
    q.alloc(std::max<size_t>(nnz, 1));
    m.alloc(n);
    v.alloc(n);
    gmrf::cuda_check(cudaMemcpy(q.p, qv, sizeof(double) * nnz, cudaMemcpyHostToDevice), "Q");
    gmrf::cuda_check(cudaMemcpy(m.p, mean, sizeof(double) * n, cudaMemcpyHostToDevice), "mean");
    f->f->rbmc_variance(q.p, m.p, ns, seed, v.p);
    gmrf::cuda_check(cudaMemcpy(var, v.p, sizeof(double) * n, cudaMemcpyDeviceToHost), "var");
  });
}

// Value of the lower-triangular panel entry (i, j), i >= j, internal order.
static double panel_at(const gmrf::Symbolic& s, const std::vector<double>& pan, int i, int j) {
  const int k = s.col2sn[j];
  const int32_t* b = s.sn_rows.data() + s.sn_rptr[k];
  const int32_t* e = s.sn_rows.data() + s.sn_rptr[k + 1];
  const int32_t* it = std::lower_bound(b, e, i);
  if (it == e || *it != i) gmrf::fail(gmrf::kStructural, "panel entry outside structure");
  return pan[s.lptr[k] + static_cast<int64_t>(j - s.sn_first[k]) * s.rows(k) + (it - b)];
}

int gmrf_selinv_pattern_nnz(gmrf_factor_t* f, int64_t* nnz) {
  return guard([&] {
    const gmrf::Symbolic& s = *f->s;
    *nnz = 2 * s.nnz_l - s.n;
  });
}

int gmrf_selinv_pattern(gmrf_factor_t* f, int64_t* cp, int32_t* ri, double* v) {
  return guard([&] {
    gmrf::require(f->f->has_selinv(), gmrf::kContract, "selinv_pattern: run selinv first");
    gmrf::require(!f->f->partitioned(), gmrf::kContract, "selinv_pattern: partitioned factor");
    const gmrf::Symbolic& s = *f->s;
    std::vector<double> sig;
    f->f->copy_sig_panels(sig);
    std::vector<int32_t> lrows = gmrf::exact_l_rows(s);
    std::vector<std::tuple<int32_t, int32_t, double>> t;
    t.reserve(2 * s.nnz_l);
    for (int j = 0; j < s.n; ++j)
      for (int64_t p = s.colptr_l[j]; p < s.colptr_l[j + 1]; ++p) {
        int i = lrows[p];
        double val = panel_at(s, sig, i, j);
        t.emplace_back(s.perm[j], s.perm[i], val);  // (col, row, value)
        if (i != j) t.emplace_back(s.perm[i], s.perm[j], val);
      }
    std::sort(t.begin(), t.end(), [](const auto& a, const auto& b) {
      return std::tie(std::get<0>(a), std::get<1>(a)) < std::tie(std::get<0>(b), std::get<1>(b));
    });
    std::fill(cp, cp + s.n + 1, 0);
    for (size_t q = 0; q < t.size(); ++q) {
      cp[std::get<0>(t[q]) + 1]++;
      ri[q] = std::get<1>(t[q]);
      v[q] = std::get<2>(t[q]);
    }
    for (int j = 0; j < s.n; ++j) cp[j + 1] += cp[j];
  });
}

int gmrf_factor_l(gmrf_factor_t* f, int64_t* cp, int32_t* ri, double* v, int32_t* perm) {
  return guard([&] {
    gmrf::require(f->f->factored(), gmrf::kContract, "factor_l: factor not computed");
    gmrf::require(!f->f->partitioned(), gmrf::kContract, "factor_l: partitioned factor");
    const gmrf::Symbolic& s = *f->s;
    std::vector<double> pan;
    f->f->copy_l_panels(pan);
    std::vector<int32_t> lrows = gmrf::exact_l_rows(s);
    for (int j = 0; j <= s.n; ++j) cp[j] = s.colptr_l[j];
    for (int j = 0; j < s.n; ++j)
      for (int64_t p = s.colptr_l[j]; p < s.colptr_l[j + 1]; ++p) {
        ri[p] = lrows[p];
        v[p] = panel_at(s, pan, lrows[p], j);
      }
    if (perm) std::memcpy(perm, s.perm.data(), sizeof(int32_t) * s.n);
  });
}

int gmrf_factor_stats(const gmrf_factor_t* f, gmrf_factor_stats_t* st) {
  return guard([&] {
    st->device_bytes = f->f->device_bytes();
    st->launches_numeric = f->f->launches_numeric();
    st->launches_solve = f->f->launches_solve();
    st->launches_selinv = f->f->launches_selinv();
  });
}

void gmrf_factor_free(gmrf_factor_t* f) { delete f; }

int gmrf_rng_draw(uint64_t seed, int64_t nu, int64_t nn, double* out) {
  return guard([&] {
    gmrf::require(nu >= 0 && nn >= 0, gmrf::kContract, "rng_draw: negative count");
    gmrf::HostRng r(seed);
    for (int64_t i = 0; i < nu; ++i) out[i] = r.uniform();
    for (int64_t i = 0; i < nn; ++i) out[nu + i] = r.normal();
  });
}

int gmrf_rng_fill(uint64_t seed, int32_t kind, int64_t n, double* out) {
  return guard([&] {
    gmrf::require(kind == 0 || kind == 1, gmrf::kContract, "rng_fill: kind must be 0 or 1");
    gmrf::HostRng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = kind == 0 ? r.uniform() : r.normal();
  });
}

int gmrf_bench_fp64(double* a, double* b) {
  return guard([&] { gmrf::bench_fp64(a, b); });
}

static gmrf::SpaceTimeSpec spacetime_spec(const gmrf_spacetime_config_t* c) {
    gmrf::SpaceTimeSpec s;
    s.n_el = c->n_el;
    s.xa = c->xa;
    s.xb = c->xb;
    s.n_t = c->n_t;
    s.t_end = c->t_end;
    s.diffusion = c->diffusion;
    s.advection = c->advection;
    s.noise = {c->noise_kappa, c->noise_alpha, c->noise_tau};
    s.init = {c->init_kappa, c->init_alpha, c->init_tau};
    s.tau = c->tau;
    s.eps = c->eps;
    s.dirichlet = c->dirichlet != 0;
    s.ic_noise_prec = c->ic_noise_prec;
    s.residual = c->residual;
    s.pde_noise_prec = c->pde_noise_prec;
    s.dim = c->dim == 0 ? 1 : c->dim;
    return s;
}

int gmrf_spacetime_symbolic(const gmrf_spacetime_config_t* c, gmrf_symbolic_t** out) {
  return guard([&] {
    auto h = std::make_unique<gmrf_symbolic>();
    h->s = gmrf::SpaceTimePosterior::host_symbolic(spacetime_spec(c));
    *out = h.release();
  });
}

static int spacetime_create(const gmrf_spacetime_config_t* c, const gmrf::PartitionSpec* part,
                            gmrf_spacetime_t** out) {
  return guard([&] {
    const gmrf::SpaceTimeSpec s = spacetime_spec(c);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      gmrf::fail(gmrf::kCuda, "no CUDA device: libgmrf_b200 has no CPU fallback");
    auto h = std::make_unique<gmrf_spacetime>();
    h->cfg.max_iters = c->gn_max_iters;
    h->cfg.decrement_tol = c->gn_decrement_tol;
    h->cfg.armijo_c = c->gn_armijo_c;
    h->cfg.shrink = c->gn_shrink;
    h->cfg.max_backtracks = c->gn_max_backtracks;
    h->p = std::make_unique<gmrf::SpaceTimePosterior>(s, nullptr, part);
    *out = h.release();
  });
}

int gmrf_spacetime_create(const gmrf_spacetime_config_t* c, gmrf_spacetime_t** out) {
  return spacetime_create(c, nullptr, out);
}

int gmrf_spacetime_create_partitioned(const gmrf_spacetime_config_t* c, int32_t nranks,
                                      int32_t rank, gmrf_exchange_fn fn, void* ctx,
                                      gmrf_spacetime_t** out) {
  gmrf::PartitionSpec ps;
  ps.nranks = nranks;
  ps.rank = rank;
  ps.fn = reinterpret_cast<gmrf::ExchangeFn>(fn);
  ps.ctx = ctx;
  return spacetime_create(c, &ps, out);
}

int gmrf_spacetime_run(gmrf_spacetime_t* h, const double* u0, int32_t want_var, double* mean,
                       double* var, gmrf_gn_iter_t* trace, int32_t max_trace, int32_t* n_trace,
                       int32_t* converged) {
  int rc = guard([&] {
    h->p->run(u0, h->cfg, want_var != 0);
    const int n = h->p->n();
    if (mean)
      gmrf::cuda_check(cudaMemcpy(mean, h->p->d_mean(), n * sizeof(double), cudaMemcpyDeviceToHost),
                       "mean");
    if (var && want_var)
      gmrf::cuda_check(cudaMemcpy(var, h->p->d_var(), n * sizeof(double), cudaMemcpyDeviceToHost),
                       "var");
  });
  // the trace is complete on the error path too (line-search stagnation)
  const std::vector<gmrf::GnIter>& tr = h->p->last_trace();
  if (n_trace) *n_trace = static_cast<int32_t>(tr.size());
  if (trace)
    for (size_t i = 0; i < tr.size() && static_cast<int32_t>(i) < max_trace; ++i)
      trace[i] = {tr[i].iter, tr[i].objective, tr[i].decrement, tr[i].step_size, tr[i].backtracks};
  if (converged) *converged = h->p->converged() ? 1 : 0;
  return rc;
}

int gmrf_spacetime_info(const gmrf_spacetime_t* h, gmrf_spacetime_info_t* info) {
  return guard([&] {
    const auto& t = h->p->times();
    const auto& s = h->p->symbolic();
    info->setup_host_ms = t.setup_host_ms;
    info->init_ms = t.init_ms;
    info->assemble_ms = t.assemble_ms;
    info->condition_ms = t.condition_ms;
    info->gn_ms = t.gn_ms;
    info->laplace_ms = t.laplace_ms;
    info->selinv_ms = t.selinv_ms;
    info->numeric_ms = t.numeric_ms;
    info->n_factorizations = t.n_factorizations;
    info->numeric_pure_ms = t.numeric_pure_ms;
    info->n_pure_factorizations = t.n_pure_factorizations;
    info->kernel_launches = t.kernel_launches;
    info->n = h->p->n();
    info->n_space = h->p->n_space();
    info->n_res = h->p->n_res();
    info->nnz_pattern = static_cast<int64_t>(s.qri.size());
    info->nnz_l = s.nnz_l;
    info->nnz_l_padded = s.nnz_l_padded;
    info->flops_ref = s.flops_ref;
    info->flops_sn = s.flops_sn;
    info->factor_device_bytes = const_cast<gmrf_spacetime_t*>(h)->p->factor().device_bytes();
  });
}

int gmrf_spacetime_device_results(const gmrf_spacetime_t* h, const double** m, const double** v) {
  return guard([&] {
    if (m) *m = h->p->d_mean();
    if (v) *v = h->p->d_var();
  });
}

int gmrf_spacetime_pattern(const gmrf_spacetime_t* h, int64_t* cp, int32_t* ri, double* qc,
                           double* qe) {
  return guard([&] {
    std::vector<int64_t> c;
    std::vector<int32_t> r;
    std::vector<double> a, b;
    h->p->copy_pattern(c, r);
    h->p->copy_values(a, b);
    if (cp) std::copy(c.begin(), c.end(), cp);
    if (ri) std::copy(r.begin(), r.end(), ri);
    if (qc) std::copy(a.begin(), a.end(), qc);
    if (qe) std::copy(b.begin(), b.end(), qe);
  });
}

static void upload_state(gmrf_spacetime_t* h, const double* u) {
  h->tmp.alloc(h->p->n());
  gmrf::cuda_check(cudaMemcpy(h->tmp.p, u, h->p->n() * sizeof(double), cudaMemcpyHostToDevice),
                   "state");
}

int gmrf_spacetime_residual(gmrf_spacetime_t* h, const double* u, double* f) {
  return guard([&] {
    upload_state(h, u);
    gmrf::DevBuf<double> out;
    out.alloc(std::max(h->p->n_res(), 1));
    h->p->residual(h->tmp.p, out.p);
    gmrf::cuda_check(cudaMemcpy(f, out.p, h->p->n_res() * sizeof(double), cudaMemcpyDeviceToHost),
                     "f");
  });
}

int gmrf_spacetime_jacobian_nnz(const gmrf_spacetime_t* h, int64_t* nnz) {
  return guard([&] {
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> v;
    gmrf::DevBuf<double> z;
    z.alloc(std::max(h->p->n(), 1));
    gmrf::cuda_check(cudaMemset(z.p, 0, h->p->n() * sizeof(double)), "z");
    const_cast<gmrf_spacetime_t*>(h)->p->jacobian_csr(z.p, rp, ci, v);
    *nnz = static_cast<int64_t>(ci.size());
  });
}

int gmrf_spacetime_jacobian(gmrf_spacetime_t* h, const double* u, int64_t* rp_out,
                            int32_t* ci_out, double* v_out) {
  return guard([&] {
    upload_state(h, u);
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> v;
    h->p->jacobian_csr(h->tmp.p, rp, ci, v);
    std::copy(rp.begin(), rp.end(), rp_out);
    std::copy(ci.begin(), ci.end(), ci_out);
    std::copy(v.begin(), v.end(), v_out);
  });
}

void gmrf_spacetime_free(gmrf_spacetime_t* h) { delete h; }

// ---- fixed-pattern Gram update ----------------------------------------------
int gmrf_gram_create(const gmrf_symbolic_t* s, int32_t m, const int64_t* arp, const int32_t* aci,
                     gmrf_gram_t** out) {
  return guard([&] {
    gmrf::require(m >= 0, gmrf::kDimension, "gram: negative row count");
    auto h = std::make_unique<gmrf_gram>();
    h->s = s->s;
    h->m = m;
    const gmrf::Symbolic& sy = *s->s;
    h->g = std::make_unique<gmrf::GramPlan>(sy.n, sy.qcp.data(), sy.qri.data(), m, arp, aci,
                                            nullptr, nullptr);
    *out = h.release();
  });
}

void gmrf_gram_free(gmrf_gram_t* g) { delete g; }

namespace {
// host arrays → the plan's device staging buffers
void gram_stage(gmrf_gram_t* g, const double* base, const double* a, const double* w,
                cudaStream_t st) {
  const int64_t np = g->g->nnz_pattern(), na = g->g->nnz_a();
  auto up = [&](gmrf::DevBuf<double>& b, const double* src, int64_t n) {
    b.alloc(std::max<int64_t>(n, 1));
    if (n) gmrf::cuda_check(cudaMemcpyAsync(b.p, src, n * 8, cudaMemcpyHostToDevice, st), "stage");
  };
  up(g->a, a, na);
  if (w) up(g->w, w, g->m);
  if (base) up(g->base, base, np);
}
}  // namespace

int gmrf_gram_apply(gmrf_gram_t* g, const double* base, const double* a, const double* w, double c,
                    double* out) {
  return guard([&] {
    gram_stage(g, base, a, w, nullptr);
    g->out.alloc(std::max<int64_t>(g->g->nnz_pattern(), 1));
    g->g->apply(g->a.p, w ? g->w.p : nullptr, c, base ? g->base.p : nullptr, g->out.p, nullptr,
                nullptr, nullptr);
    gmrf::cuda_check(cudaMemcpy(out, g->out.p, g->g->nnz_pattern() * 8, cudaMemcpyDeviceToHost),
                     "gram out");
  });
}

namespace {
int update_fixed(gmrf_factor_t* f, gmrf_gram_t* g, const double* base, const double* a,
                 const double* w, double c, int32_t* bad) {
  int32_t b = -1;
  const int rc = guard([&] {
    gmrf::require(f->s.get() == g->s.get(), gmrf::kStructural,
                  "update_fixed_pattern: plan built for another symbolic");
    f->f->begin_numeric();
    g->g->apply(a, w, c, base, nullptr, f->f->d_qmap(), f->f->d_l(), f->f->stream());
    b = f->f->factor_panels();
  });
  if (bad) *bad = b;
  if (rc == GMRF_OK && b >= 0) {
    g_err = "cholesky: non-positive pivot at index " + std::to_string(b);
    return GMRF_ERR_NOT_SPD;
  }
  return rc;
}
}  // namespace

int gmrf_factor_update_fixed_pattern(gmrf_factor_t* f, gmrf_gram_t* g, const double* base,
                                     const double* a, const double* w, double c, int32_t* bad) {
  const int rc = guard([&] { gram_stage(g, base, a, w, f->f->stream()); });
  if (rc != GMRF_OK) return rc;
  return update_fixed(f, g, base ? g->base.p : nullptr, g->a.p, w ? g->w.p : nullptr, c, bad);
}

int gmrf_factor_update_fixed_pattern_device(gmrf_factor_t* f, gmrf_gram_t* g, const double* base,
                                            const double* a, const double* w, double c,
                                            int32_t* bad) {
  return update_fixed(f, g, base, a, w, c, bad);
}

// ---- update system ------------------------------------------------------------------
int gmrf_update_system_create(int32_t n, int32_t kind, int32_t bcols, const int64_t* bcp,
                              const int32_t* bri, const double* bv, int32_t m, const int64_t* acp,
                              const int32_t* ari, const int32_t* perm,
                              gmrf_update_system_t** out) {
  return guard([&] {
    auto h = std::make_unique<gmrf_update_system>();
    h->u = std::make_unique<gmrf::UpdateSystem>(n, kind, bcols, bcp, bri, bv, m, acp, ari, perm);
    *out = h.release();
  });
}

int gmrf_update_system_same_operator(const gmrf_update_system_t* h, int32_t m, const int64_t* acp,
                                     const int32_t* ari) {
  return h->u->same_operator(m, acp, ari) ? 1 : 0;
}

int gmrf_update_system_refactor(gmrf_update_system_t* h, const double* a, const double* w,
                                int32_t* bad) {
  int32_t b = -1;
  const int rc = guard([&] {
    b = h->u->refactor(a, w);
    if (!h->fac.f) {  // views of the factor created by the first refactor
      h->sym.s = h->u->symbolic();
      h->fac.s = h->u->symbolic();
      h->fac.f.reset(&h->u->factor());
    }
  });
  if (bad) *bad = b;
  if (rc == GMRF_OK && b >= 0) {
    g_err = "cholesky: non-positive pivot at index " + std::to_string(b);
    return GMRF_ERR_NOT_SPD;
  }
  return rc;
}

int gmrf_update_system_refactor_solve(gmrf_update_system_t* h, const double* a, const double* w,
                                      const double* b, double* x, int32_t* bad) {
  int32_t bi = -1;
  const int rc = guard([&] {
    bi = h->u->refactor(a, w, b);
    if (!h->fac.f) {
      h->sym.s = h->u->symbolic();
      h->fac.s = h->u->symbolic();
      h->fac.f.reset(&h->u->factor());
    }
    if (bi < 0) h->u->solve_pending(x);
  });
  if (bad) *bad = bi;
  if (rc == GMRF_OK && bi >= 0) {
    g_err = "cholesky: non-positive pivot at index " + std::to_string(bi);
    return GMRF_ERR_NOT_SPD;
  }
  return rc;
}

int gmrf_update_system_assemble(gmrf_update_system_t* h, const double* a, const double* w, double c,
                                double* v) {
  return guard([&] {
    h->u->assemble(a, w, c);
    if (v) h->u->copy_values(v);
  });
}

int gmrf_update_system_matrix(const gmrf_update_system_t* h, int64_t* cp, int32_t* ri, double* v) {
  return guard([&] {
    const auto& c = h->u->col_ptr();
    if (cp) std::memcpy(cp, c.data(), c.size() * sizeof(int64_t));
    if (ri) std::memcpy(ri, h->u->row_idx().data(), h->u->row_idx().size() * sizeof(int32_t));
    if (v) h->u->copy_values(v);
  });
}

const gmrf_symbolic_t* gmrf_update_system_symbolic(const gmrf_update_system_t* h) {
  return h->sym.s ? &h->sym : nullptr;  // after the first refactor
}

gmrf_factor_t* gmrf_update_system_factor(gmrf_update_system_t* h) {
  return h->fac.f ? &h->fac : nullptr;
}

void gmrf_update_system_free(gmrf_update_system_t* h) {
  if (h) h->fac.f.release();  // borrowed view of the system's factor
  delete h;
}

// ---- Matérn regression ----------------------------------------------------------
namespace {
gmrf::MeshSpec mesh_of(const gmrf_matern_config_t* c) {
  gmrf::MeshSpec m;
  m.dim = c->dim;
  m.n_el = c->n_el;
  m.xa = c->dim == 1 ? c->xa : 0.0;
  m.xb = c->dim == 1 ? c->xb : 1.0;
  gmrf::require(m.dim == 1 || m.dim == 2, gmrf::kContract, "mesh: dim must be 1 or 2");
  gmrf::require(m.n_el >= 1, gmrf::kContract, "mesh: need at least one element");
  gmrf::require(m.dim == 2 || m.xa < m.xb, gmrf::kContract, "build_interval_mesh: need a < b");
  return m;
}
}  // namespace

int gmrf_point_operator(const gmrf_matern_config_t* mesh, int32_t m, const double* pts,
                        int64_t* rp, int32_t* ci, double* v) {
  return guard([&] {
    std::vector<int64_t> r;
    std::vector<int32_t> c;
    std::vector<double> x;
    gmrf::point_operator(mesh_of(mesh), m, pts, r, c, x);
    if (rp) std::memcpy(rp, r.data(), r.size() * sizeof(int64_t));
    if (ci) std::memcpy(ci, c.data(), c.size() * sizeof(int32_t));
    if (v) std::memcpy(v, x.data(), x.size() * sizeof(double));
  });
}

static int fem_assemble(bool device, const gmrf_matern_config_t* cfg, int32_t which, double diff,
                        double adv, double react, int32_t dirichlet, double cdiag, int32_t* n,
                        int64_t* cp, int32_t* ri, double* v, double* lumped) {
  return guard([&] {
    gmrf::require(cfg && n && cp, gmrf::kContract, "fem_assemble: null argument");
    gmrf::require(cfg->dim == 1 || cfg->dim == 2, gmrf::kContract, "fem_assemble: dim must be 1 or 2");
    gmrf::require(which == 0 || which == 1, gmrf::kContract, "fem_assemble: which must be 0 or 1");
    gmrf::require(!dirichlet || cfg->dim == 1, gmrf::kContract,
                  "fem_assemble: Dirichlet folding is for the interval mesh");
    gmrf::Csc m;
    if (device) {
      m = gmrf::p1_matrix_device(cfg->dim, cfg->n_el, cfg->xa, cfg->xb, which, diff, adv, react);
    } else if (cfg->dim == 1) {
      const gmrf::Space1D s{cfg->n_el, cfg->xa, cfg->xb};
      m = which == 0 ? gmrf::p1_mass(s) : gmrf::p1_stiffness(s, diff, adv, react);
    } else {
      const gmrf::Space2D s{cfg->n_el};
      m = which == 0 ? gmrf::p1_mass(s) : gmrf::scale(gmrf::p1_laplace(s), diff);
    }
    if (dirichlet) {
      const auto mask = gmrf::dirichlet_mask(gmrf::Space1D{cfg->n_el, cfg->xa, cfg->xb}, true);
      m = device ? gmrf::mask_constrained_device(m, mask, cdiag)
                 : gmrf::mask_constrained_host(m, mask, cdiag);
    }
    *n = m.nr;
    for (size_t i = 0; i < m.cp.size(); ++i) cp[i] = m.cp[i];
    if (!ri) return;
    gmrf::require(v != nullptr, gmrf::kContract, "fem_assemble: values missing");
    for (size_t i = 0; i < m.ri.size(); ++i) {
      ri[i] = m.ri[i];
      v[i] = m.v[i];
    }
    if (lumped) {
      const std::vector<double> l = device ? gmrf::lumped_mass_device(m) : gmrf::lumped_mass_host(m);
      for (size_t i = 0; i < l.size(); ++i) lumped[i] = l[i];
    }
  });
}
int gmrf_fem_assemble(const gmrf_matern_config_t* cfg, int32_t which, double diff, double adv,
                      double react, int32_t dirichlet, double cdiag, int32_t* n, int64_t* cp,
                      int32_t* ri, double* v, double* lumped) {
  return fem_assemble(true, cfg, which, diff, adv, react, dirichlet, cdiag, n, cp, ri, v, lumped);
}
int gmrf_fem_assemble_host(const gmrf_matern_config_t* cfg, int32_t which, double diff, double adv,
                           double react, int32_t dirichlet, double cdiag, int32_t* n, int64_t* cp,
                           int32_t* ri, double* v, double* lumped) {
  return fem_assemble(false, cfg, which, diff, adv, react, dirichlet, cdiag, n, cp, ri, v, lumped);
}

int gmrf_matern_prior(const gmrf_matern_config_t* cfg, int32_t* n, int64_t* cp, int32_t* ri,
                      double* v) {
  return guard([&] {
    gmrf::RegressionPosterior p(mesh_of(cfg), gmrf::MaternSpec{cfg->kappa, cfg->alpha, cfg->tau},
                                0, nullptr, nullptr);
    std::vector<int64_t> c;
    std::vector<int32_t> r;
    std::vector<double> q, qp;
    p.copy_precisions(c, r, q, qp);
    if (n) *n = p.n();
    if (cp) std::memcpy(cp, c.data(), c.size() * sizeof(int64_t));
    if (ri) std::memcpy(ri, r.data(), r.size() * sizeof(int32_t));
    if (v) std::memcpy(v, q.data(), q.size() * sizeof(double));
  });
}

int gmrf_regression_create(const gmrf_matern_config_t* cfg, int32_t m, const double* pts,
                           const int32_t* perm, gmrf_regression_t** out) {
  return guard([&] {
    auto h = std::make_unique<gmrf_regression>();
    h->p = std::make_unique<gmrf::RegressionPosterior>(
        mesh_of(cfg), gmrf::MaternSpec{cfg->kappa, cfg->alpha, cfg->tau}, m, pts, perm);
    h->wrap.s = h->p->symbolic_ptr();
    h->wrap.f.reset(&h->p->factor());
    *out = h.release();
  });
}

int gmrf_regression_run(gmrf_regression_t* h, const double* y, const double* lam, int32_t want_var,
                        int32_t ns, uint64_t seed, double* mean, double* var, double* samples) {
  return guard([&] {
    h->p->run(y, lam, want_var != 0, ns, seed);
    const size_t n = static_cast<size_t>(h->p->n());
    if (mean) gmrf::cuda_check(cudaMemcpy(mean, h->p->d_mean(), n * 8, cudaMemcpyDeviceToHost), "mean");
    if (var && want_var)
      gmrf::cuda_check(cudaMemcpy(var, h->p->d_var(), n * 8, cudaMemcpyDeviceToHost), "var");
    if (samples && ns > 0)
      gmrf::cuda_check(
          cudaMemcpy(samples, h->p->d_samples(), n * ns * 8, cudaMemcpyDeviceToHost), "samples");
  });
}

int gmrf_regression_info(const gmrf_regression_t* h, gmrf_regression_info_t* info) {
  return guard([&] {
    const auto& s = h->p->symbolic();
    info->n = h->p->n();
    info->m = h->p->m();
    info->nnz_pattern = static_cast<int64_t>(s.qri.size());
    info->nnz_l = s.nnz_l;
    info->setup_host_ms = h->p->times().setup_host_ms;
    info->run_ms = h->p->times().total_ms;
    info->flops_ref = s.flops_ref;
    info->kernel_launches = h->p->times().kernel_launches;
  });
}

int gmrf_regression_precisions(const gmrf_regression_t* h, int64_t* cp, int32_t* ri, double* qpr,
                               double* qpo) {
  return guard([&] {
    std::vector<int64_t> c;
    std::vector<int32_t> r;
    std::vector<double> a, b;
    h->p->copy_precisions(c, r, a, b);
    if (cp) std::memcpy(cp, c.data(), c.size() * sizeof(int64_t));
    if (ri) std::memcpy(ri, r.data(), r.size() * sizeof(int32_t));
    if (qpr) std::memcpy(qpr, a.data(), a.size() * 8);
    if (qpo) std::memcpy(qpo, b.data(), b.size() * 8);
  });
}

gmrf_factor_t* gmrf_regression_factor(gmrf_regression_t* h) {
  return nullptr == h ? nullptr : &h->wrap;
}

void gmrf_regression_free(gmrf_regression_t* h) {
  if (h) h->wrap.f.release();  // borrowed: owned by the posterior
  delete h;
}

int gmrf_spacetime_set_profile(gmrf_spacetime_t* h, int32_t on) {
  return guard([&] {
    h->p->prof_.reset();
    h->p->prof_.on = on != 0;
    h->p->prof_.level_detail = on == 2;  // 2: per-level kernel classes
  });
}

int gmrf_spacetime_kernel_stats(gmrf_spacetime_t* h, gmrf_kernel_stat_t* out, int32_t max,
                                int32_t* n) {
  return guard([&] {
    h->p->prof_.flush();
    int32_t i = 0;
    for (const auto& kv : h->p->prof_.stats) {
      if (i < max && out) {
        gmrf_kernel_stat_t& o = out[i];
        std::memset(o.name, 0, sizeof(o.name));
        std::strncpy(o.name, kv.first.c_str(), sizeof(o.name) - 1);
        o.launches = kv.second.launches;
        o.ms = kv.second.ms;
        o.flops = kv.second.flops;
        o.bytes = kv.second.bytes;
      }
      ++i;
    }
    if (n) *n = i;
  });
}

}  // extern "C"
