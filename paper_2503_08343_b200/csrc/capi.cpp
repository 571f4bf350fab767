// C-ABI entry points (include/gmrf_b200.h).
#include "../../include/gmrf_b200.h"

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <tuple>

#include "factor.hpp"
#include "symbolic.hpp"

struct gmrf_symbolic {
  std::shared_ptr<const gmrf::Symbolic> s;
};
struct gmrf_factor {
  std::shared_ptr<const gmrf::Symbolic> s;
  std::unique_ptr<gmrf::DeviceFactor> f;
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

int gmrf_bench_fp64(double* a, double* b) {
  return guard([&] { gmrf::bench_fp64(a, b); });
}

}  // extern "C"
