// Fixed-pattern weighted Gram update (gram.hpp).
#include "gram.hpp"

#include <memory>

#include <algorithm>
#include <string>

namespace gmrf {

namespace {

// wa = w[row] · a  (scale_rows, core/sparse.hpp)
__global__ void k_gram_weight(i64 na, const i32* __restrict__ arow, const double* __restrict__ w,
                              const double* __restrict__ a, double* __restrict__ wa) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < na;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    wa[i] = w[arow[i]] * a[i];
}

// One thread per computed entry; pairs (x, y) = (A_kR, A_kC) value indices,
// ascending k. s1 is the (R, C) product, s2 the (C, R) one; their average
// with the base is the reference's symmetrize(add(base, c·AᵀWA)).
__global__ void k_gram(i64 ne, const i64* __restrict__ ent, const i64* __restrict__ off,
                       const int2* __restrict__ pairs, const double* __restrict__ a,
                       const double* __restrict__ wa, double c, const double* __restrict__ base,
                       const i64* __restrict__ tpos, double* __restrict__ out,
                       const i64* __restrict__ qmap, double* __restrict__ L) {
  for (i64 t = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; t < ne;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 p = ent ? ent[t] : t;
    double s1 = 0.0, s2 = 0.0;
    const i64 k1 = off[t + 1];
    for (i64 k = off[t]; k < k1; ++k) {
      const int2 xy = pairs[k];
      const double ax = a[xy.x], ay = a[xy.y];
      s1 += ax * wa[xy.y];
      s2 += ay * wa[xy.x];
    }
    const double b = base ? base[p] : 0.0;
    const double bt = base && tpos ? base[tpos[t]] : b;
    const double v = 0.5 * (b + c * s1) + 0.5 * (bt + c * s2);
    if (out) out[p] = v;
    if (L) {
      const i64 o = qmap[p];
      if (o >= 0) L[o] = v;
    }
  }
}

int grid_of(i64 n) {
  return static_cast<int>(std::max<i64>(1, std::min<i64>((n + 255) / 256, 148 * 16)));
}

}  // namespace

GramPlan::GramPlan(i32 n, const i64* pcp, const i32* pri, i32 m, const i64* arp, const i32* aci,
                   const std::vector<char>* need, cudaStream_t stream, const i64* vmap,
                   bool base_transpose) {
  m_ = m;
  np_ = pcp[n];
  na_ = arp[m];
  // A by columns: (row k, CSR value index), rows ascending
  std::vector<i64> acp(static_cast<size_t>(n) + 1, 0);
  for (i64 i = 0; i < na_; ++i) {
    require(aci[i] >= 0 && aci[i] < n, kDimension, "gram: operator column out of range");
    acp[aci[i] + 1]++;
  }
  for (i32 j = 0; j < n; ++j) acp[j + 1] += acp[j];
  std::vector<i32> ak(na_);
  std::vector<i32> av(na_);
  std::vector<i32> arow(na_);
  {
    std::vector<i64> nx(acp.begin(), acp.end() - 1);
    for (i32 k = 0; k < m; ++k)
      for (i64 i = arp[k]; i < arp[k + 1]; ++i) {
        require(i == arp[k] || aci[i] > aci[i - 1], kStructural,
                "gram: operator columns must be strictly ascending per row");
        const i64 q = nx[aci[i]]++;
        const i64 vi = vmap ? vmap[i] : i;
        require(vi >= 0 && vi < na_, kDimension, "gram: value map out of range");
        ak[q] = k;
        av[q] = static_cast<i32>(vi);
        arow[vi] = k;
      }
  }
  require(na_ < (1ll << 31), kContract, "gram: operator nnz exceeds int32 value indices");
  // product map over the computed entries: count the shared rows of every
  // pattern entry, prefix-sum, then fill — both merge passes run over column
  // ranges on the host threads (the map of config 4's S Sᵀ has 2e8 pairs, the
  // config-5 shapes' 2e9)
  const i64 npat = pcp[n];
  std::vector<i32> cnt(static_cast<size_t>(npat), 0);
  std::vector<i64> cov(parallel_threads(n), 0);
  parallel_ranges(n, [&](int64_t c0, int64_t c1, int t) {
    i64 covered_t = 0;
    for (i32 C = static_cast<i32>(c0); C < static_cast<i32>(c1); ++C)
      for (i64 p = pcp[C]; p < pcp[C + 1]; ++p) {
        const i32 R = pri[p];
        i64 x = acp[R], xe = acp[R + 1], y = acp[C], ye = acp[C + 1];
        i32 c = 0;
        while (x < xe && y < ye) {
          if (ak[x] < ak[y]) {
            ++x;
          } else if (ak[y] < ak[x]) {
            ++y;
          } else {
            ++c;
            ++x;
            ++y;
          }
        }
        cnt[p] = c;
        covered_t += c;
      }
    cov[t] = covered_t;
  });
  i64 covered = 0;
  for (i64 c : cov) covered += c;
  std::vector<i64> ent, off(1, 0), tpos;
  std::vector<i64> slot(static_cast<size_t>(npat), -1);  // pattern entry → computed-entry index
  for (i64 p = 0; p < npat; ++p) {
    if (need && !(*need)[p]) continue;
    slot[p] = static_cast<i64>(off.size()) - 1;
    if (need) ent.push_back(p);
    off.push_back(off.back() + cnt[p]);
  }
  const i64 npr = off.back();
  std::unique_ptr<int2[]> pr(new int2[std::max<i64>(npr, 1)]);  // uninitialised: filled below
  if (base_transpose) tpos.assign(off.size() - 1, 0);
  parallel_ranges(n, [&](int64_t c0, int64_t c1, int) {
    for (i32 C = static_cast<i32>(c0); C < static_cast<i32>(c1); ++C)
      for (i64 p = pcp[C]; p < pcp[C + 1]; ++p) {
        const i64 e = slot[p];
        if (e < 0) continue;
        const i32 R = pri[p];
        i64 x = acp[R], xe = acp[R + 1], y = acp[C], ye = acp[C + 1];
        int2* out = pr.get() + off[e];
        while (x < xe && y < ye) {
          if (ak[x] < ak[y]) {
            ++x;
          } else if (ak[y] < ak[x]) {
            ++y;
          } else {
            *out++ = make_int2(av[x], av[y]);
            ++x;
            ++y;
          }
        }
        if (base_transpose) {  // position of (C, R): binary search in column R
          const i32* b0 = pri + pcp[R];
          const i32* b1 = pri + pcp[R + 1];
          const i32* f = std::lower_bound(b0, b1, C);
          require(f != b1 && *f == C, kStructural, "gram: pattern is not symmetric");
          tpos[e] = pcp[R] + (f - b0);
        }
      }
  });
  // every product A_kR A_kC must have a home in the pattern
  i64 total = 0;
  for (i32 k = 0; k < m; ++k) total += (arp[k + 1] - arp[k]) * (arp[k + 1] - arp[k]);
  require(covered == total, kStructural,
          "gram: pattern does not contain the operator's product pattern (" +
              std::to_string(covered) + " of " + std::to_string(total) + " products)");
  npairs_ = npr;
  off_.upload(off, stream);
  pairs_.alloc(static_cast<size_t>(std::max<i64>(npr, 1)));
  if (npr)
    cuda_check(cudaMemcpyAsync(pairs_.p, pr.get(), static_cast<size_t>(npr) * sizeof(int2),
                               cudaMemcpyHostToDevice, stream),
               "gram pairs upload");
  arow_.upload(arow, stream);
  wa_.alloc(std::max<i64>(na_, 1));
  if (base_transpose) tpos_.upload(tpos, stream);
  if (need) {
    ent_.upload(ent, stream);
    ne_ = static_cast<i64>(ent.size());
  } else {
    ne_ = np_;
  }
  cuda_check(cudaStreamSynchronize(stream), "gram plan upload");
}

void GramPlan::apply(const double* d_a, const double* d_w, double c, const double* d_base,
                     double* d_out, const i64* d_qmap, double* d_L, cudaStream_t stream) {
  const double* wa = d_a;
  if (d_w && na_ > 0) {
    k_gram_weight<<<grid_of(na_), 256, 0, stream>>>(na_, arow_.p, d_w, d_a, wa_.p);
    wa = wa_.p;
  }
  if (ne_ > 0)
    k_gram<<<grid_of(ne_), 256, 0, stream>>>(ne_, ent_.p, off_.p, pairs_.p, d_a, wa, c, d_base,
                                             tpos_.p, d_out, d_qmap, d_L);
  cuda_check(cudaGetLastError(), "gram apply");
}

void gram_pattern(i32 n, i32 m, const i64* arp, const i32* aci, std::vector<i64>& cp,
                  std::vector<i32>& ri) {
  // columns of A: rows k touching column j
  std::vector<i64> acp(static_cast<size_t>(n) + 1, 0);
  for (i64 p = 0; p < arp[m]; ++p) acp[aci[p] + 1]++;
  for (i32 j = 0; j < n; ++j) acp[j + 1] += acp[j];
  std::vector<i32> ak(acp[n]);
  {
    std::vector<i64> nx(acp.begin(), acp.end() - 1);
    for (i32 k = 0; k < m; ++k)
      for (i64 p = arp[k]; p < arp[k + 1]; ++p) ak[nx[aci[p]]++] = k;
  }
  cp.assign(static_cast<size_t>(n) + 1, 0);
  ri.clear();
  std::vector<i32> mark(n, -1), col;
  for (i32 j = 0; j < n; ++j) {
    col.clear();
    mark[j] = j;
    col.push_back(j);  // the diagonal is always stored
    for (i64 q = acp[j]; q < acp[j + 1]; ++q) {
      const i32 k = ak[q];
      for (i64 p = arp[k]; p < arp[k + 1]; ++p)
        if (mark[aci[p]] != j) {
          mark[aci[p]] = j;
          col.push_back(aci[p]);
        }
    }
    std::sort(col.begin(), col.end());
    ri.insert(ri.end(), col.begin(), col.end());
    cp[j + 1] = static_cast<i64>(ri.size());
  }
}

void pattern_union(i32 n, const std::vector<i64>& acp, const std::vector<i32>& ari,
                   const std::vector<i64>& bcp, const std::vector<i32>& bri, std::vector<i64>& cp,
                   std::vector<i32>& ri) {
  cp.assign(static_cast<size_t>(n) + 1, 0);
  ri.clear();
  ri.reserve(ari.size() + bri.size());
  for (i32 j = 0; j < n; ++j) {
    i64 a = acp[j], b = bcp[j];
    while (a < acp[j + 1] || b < bcp[j + 1]) {
      const i32 ra = a < acp[j + 1] ? ari[a] : n, rb = b < bcp[j + 1] ? bri[b] : n;
      ri.push_back(std::min(ra, rb));
      if (ra <= rb) ++a;
      if (rb <= ra) ++b;
    }
    cp[j + 1] = static_cast<i64>(ri.size());
  }
}

int GramPlan::launches(bool weighted) const { return (weighted && na_ > 0 ? 1 : 0) + (ne_ > 0); }

double GramPlan::bytes(bool base, bool out, bool panels) const {
  // A values (+ weights / scaled copy) once, offsets, pairs, entry list, base,
  // outputs, map
  double b = 16.0 * na_ + 8.0 * (ne_ + 1) + 8.0 * npairs_;
  if (ne_ != np_) b += 8.0 * ne_;
  if (base) b += 8.0 * ne_;
  if (out) b += 8.0 * ne_;
  if (panels) b += 16.0 * ne_;
  return b;
}

}  // namespace gmrf
