// Fixed-pattern weighted Gram update (gram.hpp).
#include "gram.hpp"

#include <cub/cub.cuh>

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

// ---- product map, built on the device -------------------------------------------
// For pattern entry p = (R, C): the rows k shared by columns R and C of A (both
// lists ascending) — counted (pass 1), then written as (value index of A_kR,
// value index of A_kC) pairs at the entry's offset (pass 2). One thread per
// pattern column walks its entries; masked entries are not computed.
__global__ void k_gram_count(i32 n, const i64* __restrict__ pcp, const i32* __restrict__ pri,
                             const i64* __restrict__ acp, const i32* __restrict__ ak,
                             const char* __restrict__ need, i64* __restrict__ cnt,
                             unsigned long long* __restrict__ covered) {
  unsigned long long cov = 0;
  for (i32 C = blockIdx.x * blockDim.x + threadIdx.x; C < n; C += gridDim.x * blockDim.x)
    for (i64 p = pcp[C]; p < pcp[C + 1]; ++p) {
      const i32 R = pri[p];
      i64 x = acp[R], y = acp[C];
      const i64 xe = acp[R + 1], ye = acp[C + 1];
      i64 c = 0;
      while (x < xe && y < ye) {
        const i32 kx = ak[x], ky = ak[y];
        c += kx == ky;
        x += kx <= ky;
        y += ky <= kx;
      }
      cov += static_cast<unsigned long long>(c);
      cnt[p] = (!need || need[p]) ? c : 0;
    }
  if (cov) atomicAdd(covered, cov);  // integer: order does not matter
}

__global__ void k_gram_fill(i32 n, const i64* __restrict__ pcp, const i32* __restrict__ pri,
                            const i64* __restrict__ acp, const i32* __restrict__ ak,
                            const i32* __restrict__ av, const char* __restrict__ need,
                            const i64* __restrict__ poff, int2* __restrict__ pairs) {
  for (i32 C = blockIdx.x * blockDim.x + threadIdx.x; C < n; C += gridDim.x * blockDim.x)
    for (i64 p = pcp[C]; p < pcp[C + 1]; ++p) {
      if (need && !need[p]) continue;
      const i32 R = pri[p];
      i64 x = acp[R], y = acp[C];
      const i64 xe = acp[R + 1], ye = acp[C + 1];
      int2* out = pairs + poff[p];
      while (x < xe && y < ye) {
        const i32 kx = ak[x], ky = ak[y];
        if (kx == ky) *out++ = make_int2(av[x], av[y]);
        x += kx <= ky;
        y += ky <= kx;
      }
    }
}

// off[e] (computed entries only, compacted) from the per-pattern-entry offsets
__global__ void k_gram_compact(i64 ne, const i64* __restrict__ ent, const i64* __restrict__ poff,
                               i64 total, i64* __restrict__ off) {
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e <= ne;
       e += static_cast<i64>(gridDim.x) * blockDim.x)
    off[e] = e < ne ? poff[ent[e]] : total;
}

// position of the transposed entry (C, R) of every computed entry (R, C)
__global__ void k_gram_tpos(i32 n, const i64* __restrict__ pcp, const i32* __restrict__ pri,
                            const i64* __restrict__ slot, i64* __restrict__ tpos,
                            int* __restrict__ bad) {
  for (i32 C = blockIdx.x * blockDim.x + threadIdx.x; C < n; C += gridDim.x * blockDim.x)
    for (i64 p = pcp[C]; p < pcp[C + 1]; ++p) {
      const i64 e = slot ? slot[p] : p;
      if (e < 0) continue;
      const i32 R = pri[p];
      i64 lo = pcp[R], hi = pcp[R + 1];
      while (lo < hi) {
        const i64 mid = (lo + hi) >> 1;
        if (pri[mid] < C) lo = mid + 1; else hi = mid;
      }
      if (lo < pcp[R + 1] && pri[lo] == C) tpos[e] = lo;
      else *bad = 1;
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
  // product map over the computed entries, built on the device: count the
  // shared rows of every pattern entry, exclusive scan, fill (config 4's S Sᵀ
  // map has 2e8 pairs, the config-5 shapes' 2e9 — seconds to a minute of host
  // merging plus a pageable upload otherwise)
  const i64 npat = pcp[n];
  DevBuf<i64> d_pcp, d_acp, d_cnt, d_poff, d_slot;
  DevBuf<i32> d_pri, d_ak, d_av;
  DevBuf<char> d_need;
  DevBuf<unsigned long long> d_cov;
  DevBuf<int> d_bad;
  d_pcp.alloc(static_cast<size_t>(n) + 1);
  d_pri.alloc(static_cast<size_t>(std::max<i64>(npat, 1)));
  cuda_check(cudaMemcpyAsync(d_pcp.p, pcp, (static_cast<size_t>(n) + 1) * sizeof(i64),
                             cudaMemcpyHostToDevice, stream), "copy pattern");
  if (npat)
    cuda_check(cudaMemcpyAsync(d_pri.p, pri, static_cast<size_t>(npat) * sizeof(i32),
                               cudaMemcpyHostToDevice, stream), "copy pattern");
  d_acp.upload(acp, stream);
  d_ak.upload(ak, stream);
  d_av.upload(av, stream);
  if (need) d_need.upload(*need, stream);
  cuda_check(cudaStreamSynchronize(stream), "gram plan inputs");
  d_cnt.alloc(static_cast<size_t>(npat) + 1);
  d_poff.alloc(static_cast<size_t>(npat) + 1);
  d_cov.alloc(1);
  cuda_check(cudaMemsetAsync(d_cov.p, 0, sizeof(unsigned long long), stream), "memset");
  cuda_check(cudaMemsetAsync(d_cnt.p + npat, 0, sizeof(i64), stream), "memset");
  const int gc = grid_of(n);
  k_gram_count<<<gc, 256, 0, stream>>>(n, d_pcp.p, d_pri.p, d_acp.p, d_ak.p,
                                       need ? d_need.p : nullptr, d_cnt.p, d_cov.p);
  {
    size_t tmp_bytes = 0;
    cuda_check(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_cnt.p, d_poff.p, npat + 1, stream),
               "scan size");
    DevBuf<char> tmp;
    tmp.alloc(tmp_bytes + 1);
    cuda_check(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, d_cnt.p, d_poff.p, npat + 1, stream),
               "scan");
    cuda_check(cudaStreamSynchronize(stream), "gram plan scan");
  }
  i64 npr = 0;
  unsigned long long covered_u = 0;
  cuda_check(cudaMemcpyAsync(&npr, d_poff.p + npat, sizeof(i64), cudaMemcpyDeviceToHost, stream), "copy");
  cuda_check(cudaMemcpyAsync(&covered_u, d_cov.p, sizeof(covered_u), cudaMemcpyDeviceToHost, stream),
             "copy");
  cuda_check(cudaStreamSynchronize(stream), "gram plan counts");
  const i64 covered = static_cast<i64>(covered_u);
  pairs_.alloc(static_cast<size_t>(std::max<i64>(npr, 1)));
  k_gram_fill<<<gc, 256, 0, stream>>>(n, d_pcp.p, d_pri.p, d_acp.p, d_ak.p, d_av.p,
                                      need ? d_need.p : nullptr, d_poff.p, pairs_.p);
  // computed-entry list (host: a pass over the mask) and compacted offsets
  std::vector<i64> ent;
  if (need) {
    for (i64 p = 0; p < npat; ++p)
      if ((*need)[p]) ent.push_back(p);
    ent_.upload(ent, stream);
    ne_ = static_cast<i64>(ent.size());
    off_.alloc(static_cast<size_t>(ne_) + 1);
    k_gram_compact<<<grid_of(ne_ + 1), 256, 0, stream>>>(ne_, ent_.p, d_poff.p, npr, off_.p);
  } else {
    ne_ = np_;
    off_.alloc(static_cast<size_t>(npat) + 1);
    cuda_check(cudaMemcpyAsync(off_.p, d_poff.p, (static_cast<size_t>(npat) + 1) * sizeof(i64),
                               cudaMemcpyDeviceToDevice, stream),
               "copy offsets");
  }
  std::vector<i64> slot;
  if (base_transpose) {
    tpos_.alloc(static_cast<size_t>(std::max<i64>(ne_, 1)));
    d_bad.alloc(1);
    cuda_check(cudaMemsetAsync(d_bad.p, 0, sizeof(int), stream), "memset");
    if (need) {  // pattern entry → computed-entry index
      slot.assign(static_cast<size_t>(npat), -1);
      for (i64 e = 0; e < ne_; ++e) slot[ent[e]] = e;
      d_slot.upload(slot, stream);
    }
    k_gram_tpos<<<gc, 256, 0, stream>>>(n, d_pcp.p, d_pri.p, need ? d_slot.p : nullptr, tpos_.p,
                                        d_bad.p);
    int bad = 0;
    cuda_check(cudaMemcpyAsync(&bad, d_bad.p, sizeof(int), cudaMemcpyDeviceToHost, stream), "copy");
    cuda_check(cudaStreamSynchronize(stream), "gram plan transpose map");
    require(bad == 0, kStructural, "gram: pattern is not symmetric");
  }
  // every product A_kR A_kC must have a home in the pattern
  i64 total = 0;
  for (i32 k = 0; k < m; ++k) total += (arp[k + 1] - arp[k]) * (arp[k + 1] - arp[k]);
  require(covered == total, kStructural,
          "gram: pattern does not contain the operator's product pattern (" +
              std::to_string(covered) + " of " + std::to_string(total) + " products)");
  npairs_ = npr;
  arow_.upload(arow, stream);
  wa_.alloc(std::max<i64>(na_, 1));
  cuda_check(cudaGetLastError(), "gram plan kernels");
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
