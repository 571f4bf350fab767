// Supernode ownership and exchange schedule of the partitioned factorization
// (partition.hpp). Host code, no device calls: tests query it on CPU.
#include "partition.hpp"

#include <algorithm>
#include <functional>
#include <map>

#include "kernels.cuh"

namespace gmrf {

void chunk_levels(const Symbolic& s, std::vector<int>& lvl0, std::vector<int>& last, int& nlev,
                  int small_rows) {
  lvl0.assign(s.ns, 0);
  last.assign(s.ns, 0);
  nlev = 0;
  for (int k = 0; k < s.ns; ++k) {
    int l = 0;
    for (int q = s.ch_ptr[k]; q < s.ch_ptr[k + 1]; ++q) l = std::max(l, last[s.ch_list[q]] + 1);
    lvl0[k] = l;
    const int nch = (s.w(k) + kNB - 1) / kNB;
    last[k] = s.rows(k) <= small_rows ? l : l + nch - 1;
    nlev = std::max(nlev, last[k] + 1);
  }
}

std::vector<i32> partition_owners(const Symbolic& s, int nranks) {
  std::vector<i32> owner(s.ns, 0);
  if (nranks <= 1 || s.ns == 0) return owner;
  // subtree work = Σ over the subtree's panel columns of c² (children precede
  // their parent in the supernode numbering)
  std::vector<double> work(s.ns, 0.0);
  for (int k = 0; k < s.ns; ++k) {
    const double rows = s.rows(k);
    for (int j = 0; j < s.w(k); ++j) work[k] += (rows - j) * (rows - j);
    if (s.sn_parent[k] >= 0) work[s.sn_parent[k]] += work[k];
  }
  auto fill = [&](int root, int r) {
    std::vector<int> st{root};
    while (!st.empty()) {
      const int k = st.back();
      st.pop_back();
      owner[k] = r;
      for (int q = s.ch_ptr[k]; q < s.ch_ptr[k + 1]; ++q) st.push_back(s.ch_list[q]);
    }
  };
  // (roots, rank range) work list: a single root is a separator, owned by the
  // lowest rank of its range, and its children inherit the range; several roots
  // are split into two groups (largest subtree first onto the lighter group,
  // per rank) for the two halves of the range.
  struct Item {
    std::vector<int> roots;
    int r0, r1;
  };
  std::vector<Item> todo;
  {
    Item top{{}, 0, nranks};
    for (int k = 0; k < s.ns; ++k)
      if (s.sn_parent[k] < 0) top.roots.push_back(k);
    todo.push_back(std::move(top));
  }
  // separators (single roots over a rank range) go to the rank of their range
  // holding the fewest separator panel bytes so far, top-down (breadth first):
  // the big top fronts spread over the ranks instead of stacking on the lowest
  // rank of every range (per-rank memory plan, gmrf_partition_memory)
  std::vector<double> sep_bytes(nranks, 0.0);
  for (size_t head = 0; head < todo.size(); ++head) {
    Item it = std::move(todo[head]);
    if (it.roots.empty()) continue;
    if (it.r1 - it.r0 == 1) {
      for (int k : it.roots) fill(k, it.r0);
      continue;
    }
    if (it.roots.size() == 1) {
      const int k = it.roots[0];
      int best = it.r0;
      for (int r = it.r0 + 1; r < it.r1; ++r)
        if (sep_bytes[r] < sep_bytes[best]) best = r;
      owner[k] = best;
      sep_bytes[best] += static_cast<double>(s.rows(k)) * s.w(k);
      Item ch{{}, it.r0, it.r1};
      for (int q = s.ch_ptr[k]; q < s.ch_ptr[k + 1]; ++q) ch.roots.push_back(s.ch_list[q]);
      todo.push_back(std::move(ch));
      continue;
    }
    std::vector<int> rs = it.roots;
    std::stable_sort(rs.begin(), rs.end(), [&](int a, int b) { return work[a] > work[b]; });
    const int mid = it.r0 + (it.r1 - it.r0) / 2;
    const double na = mid - it.r0, nb = it.r1 - mid;
    Item a{{}, it.r0, mid}, b{{}, mid, it.r1};
    double la = 0.0, lb = 0.0;
    for (int k : rs) {
      if ((la + work[k]) / na <= (lb + work[k]) / nb) {
        a.roots.push_back(k);
        la += work[k];
      } else {
        b.roots.push_back(k);
        lb += work[k];
      }
    }
    std::sort(a.roots.begin(), a.roots.end());
    std::sort(b.roots.begin(), b.roots.end());
    todo.push_back(std::move(a));
    todo.push_back(std::move(b));
  }
  return owner;
}

std::vector<XEdge> partition_schedule(const Symbolic& s, const std::vector<i32>& owner) {
  require(static_cast<i32>(owner.size()) == s.ns, kContract, "partition: owner size != supernodes");
  std::vector<int> fl0, flast, sl0, slast;
  int fn = 0, sn = 0;
  chunk_levels(s, fl0, flast, fn, kSmallRows);
  chunk_levels(s, sl0, slast, sn, 0);
  std::vector<XEdge> e;
  for (int k = 0; k < s.ns; ++k) {
    const int p = s.sn_parent[k];
    if (p < 0 || owner[k] == owner[p]) continue;
    const i64 r = s.r(k);
    e.push_back({kXFactor, flast[k], owner[k], owner[p], k, r * r});
    e.push_back({kXFsolve, s.sn_level[k], owner[k], owner[p], k, r});
    e.push_back({kXBsolve, s.sn_level[p], owner[p], owner[k], k, r});
    e.push_back({kXSelinv, sl0[p], owner[p], owner[k], k, r * r});
  }
  std::sort(e.begin(), e.end(), [](const XEdge& a, const XEdge& b) {
    if (a.phase != b.phase) return a.phase < b.phase;
    if (a.point != b.point) return a.point < b.point;
    return a.sn < b.sn;
  });
  return e;
}

// Lifetime-packed update-matrix storage, per phase. Factorization: U_k lives
// from its supernode's first chunk level (extend-add, zeroing) to the parent's
// first chunk level (the parent's extend-add reads it); a Schur complement
// received from another rank from the exchange after the child's last level.
// Selected inversion (levels top-down): Σ_RR(k) lives from its gather (or
// receipt) to the last of its readers — k's own chunks and its children's
// gathers. Regions are reused first-fit once their interval has ended, so the
// buffer holds the live matrices of a level front, not Σ_s r_s² (C4: see
// gmrf_factor_stats device_bytes). GMRF_U_STATIC=1: one slot per supernode.
std::vector<i64> plan_arena(const std::vector<i64>& size, const std::vector<int>& start,
                                   const std::vector<int>& end, int ntime, i64& total) {
  const int n = static_cast<int>(size.size());
  std::vector<i64> off(n, 0);
  std::vector<std::vector<int>> st(std::max(ntime, 1)), en(std::max(ntime, 1));
  for (int k = 0; k < n; ++k)
    if (size[k] > 0) {
      st[start[k]].push_back(k);
      en[end[k]].push_back(k);
    }
  std::map<i64, i64> by_off;             // free blocks: offset -> size
  std::multimap<i64, i64> by_size;       // size -> offset
  auto erase_free = [&](i64 o, i64 z) {
    auto r = by_size.equal_range(z);
    for (auto it = r.first; it != r.second; ++it)
      if (it->second == o) {
        by_size.erase(it);
        break;
      }
    by_off.erase(o);
  };
  total = 0;
  for (int t = 0; t < ntime; ++t) {
    std::vector<int>& a = st[t];
    std::stable_sort(a.begin(), a.end(), [&](int x, int y) { return size[x] > size[y]; });
    for (int k : a) {
      auto it = by_size.lower_bound(size[k]);
      if (it == by_size.end()) {
        off[k] = total;
        total += size[k];
        continue;
      }
      const i64 z = it->first, o = it->second;
      erase_free(o, z);
      off[k] = o;
      if (z > size[k]) {
        by_off[o + size[k]] = z - size[k];
        by_size.insert({z - size[k], o + size[k]});
      }
    }
    for (int k : en[t]) {
      i64 o = off[k], z = size[k];
      auto nx = by_off.lower_bound(o);
      if (nx != by_off.end() && nx->first == o + z) {
        const i64 no = nx->first, nz = nx->second;
        erase_free(no, nz);
        z += nz;
      }
      auto pv = by_off.lower_bound(o);
      if (pv != by_off.begin()) {
        --pv;
        if (pv->first + pv->second == o) {
          const i64 po = pv->first, pz = pv->second;
          erase_free(po, pz);
          o = po;
          z += pz;
        }
      }
      by_off[o] = z;
      by_size.insert({z, o});
    }
  }
  return off;
}

void plan_update_arenas(const Symbolic& s, const std::vector<i32>& owner, int rank,
                        std::vector<i64>& fo, std::vector<i64>& so, i64& arena_f, i64& arena_s) {
  auto mine = [&](int k) { return owner[k] == rank; };
  std::vector<i64> size(s.ns, 0);
  for (int k = 0; k < s.ns; ++k) {
    const int p = s.sn_parent[k];
    if (p >= 0 && (mine(k) || mine(p))) size[k] = static_cast<i64>(s.r(k)) * s.r(k);
  }
  std::vector<int> f0, fl, s0, sl;
  int nf = 0, nsl = 0;
  chunk_levels(s, f0, fl, nf, kSmallRows);
  chunk_levels(s, s0, sl, nsl, 0);
  std::vector<int> a(s.ns, 0), b(s.ns, 0);
  for (int k = 0; k < s.ns; ++k) {
    const int p = s.sn_parent[k];
    if (!size[k]) continue;
    if (mine(k) && mine(p)) {
      a[k] = f0[k];
      b[k] = f0[p];
    } else if (mine(k)) {  // sent to the parent's rank after its last level
      a[k] = f0[k];
      b[k] = fl[k];
    } else {  // received from the child's rank
      a[k] = fl[k];
      b[k] = f0[p];
    }
  }
  fo = plan_arena(size, a, b, nf, arena_f);
  // selected inversion, time = nsl - 1 - level
  auto T = [&](int lvl) { return nsl - 1 - lvl; };
  for (int k = 0; k < s.ns; ++k) {
    const int p = s.sn_parent[k];
    if (!size[k]) continue;
    if (!mine(k)) {  // ghost gather on the parent's rank, sent right away
      a[k] = b[k] = T(s0[p]);
      continue;
    }
    int last = s0[k];  // lowest level still reading Σ_RR(k)
    for (int q = s.ch_ptr[k]; q < s.ch_ptr[k + 1]; ++q) {
      const int c = s.ch_list[q];
      if (mine(c)) last = std::min(last, sl[c]);
    }
    a[k] = T(mine(p) ? sl[k] : s0[p]);
    b[k] = T(last);
  }
  so = plan_arena(size, a, b, nsl, arena_s);
}

std::vector<char> selinv_blocked(const Symbolic& s, long long max_level_stage, int min_single_w) {
  std::vector<int> l0, la;
  int nl = 0;
  chunk_levels(s, l0, la, nl, 0);
  std::vector<i64> tot(std::max(nl, 1), 0);
  std::vector<char> blk(s.ns, 0);
  if (max_level_stage <= 0) return blk;
  for (int k = 0; k < s.ns; ++k) {
    const int w = s.w(k), rows = s.rows(k), nch = (w + kNB - 1) / kNB;
    if (w <= kNB) {
      blk[k] = w >= min_single_w;
      continue;
    }
    const i64 need = static_cast<i64>(w) * rows;  // w² + r·w
    i64& t = tot[l0[k] + nch - 1];
    if (t + need <= max_level_stage) {
      t += need;
      blk[k] = 1;
    }
  }
  return blk;
}

std::vector<i64> selinv_staging(const Symbolic& s, const std::vector<i32>* owner, int rank,
                                const std::vector<char>& blocked) {
  std::vector<int> l0, la;
  int nl = 0;
  chunk_levels(s, l0, la, nl, 0);
  std::vector<i64> st(std::max(nl, 1), 0);
  for (int k = 0; k < s.ns; ++k) {
    if (owner && (*owner)[k] != rank) continue;
    const int w = s.w(k), rows = s.rows(k), nch = (w + kNB - 1) / kNB;
    if (blocked[k]) {
      st[l0[k] + nch - 1] += static_cast<i64>(w) * rows;
      continue;
    }
    for (int c = 0; c * kNB < w; ++c)
      st[l0[k] + c] += static_cast<i64>(rows - c * kNB) * std::min(kNB, w - c * kNB);
  }
  return st;
}

std::vector<RankMemory> partition_memory(const Symbolic& s, const std::vector<i32>& owner,
                                         int nranks, int max_rhs) {
  std::vector<RankMemory> out(nranks);
  const std::vector<char> sel_blk = selinv_blocked(s, kSelBlockLevelStage, 16);
  for (int r = 0; r < nranks; ++r) {
    RankMemory& m = out[r];
    for (int k = 0; k < s.ns; ++k)
      if (owner[k] == r) {
        m.l_panels += 8 * static_cast<i64>(s.rows(k)) * s.w(k);
        m.supernodes += 1;
        m.flops += [&] {
          double f = 0;
          for (int j = 0; j < s.w(k); ++j) f += static_cast<double>(s.rows(k) - j) * (s.rows(k) - j);
          return f;
        }();
      }
    std::vector<i64> fo, so;
    i64 af = 0, as = 0;
    plan_update_arenas(s, owner, r, fo, so, af, as);
    m.u_arena_factor = 8 * af;
    m.u_arena_selinv = 8 * as;
    // the pipelines run the selected inversion in place (Σ overwrites L): only
    // the per-level Y / W staging is extra (DeviceFactor::build_selinv_plan)
    {
      const std::vector<i64> st = selinv_staging(s, &owner, r, sel_blk);
      m.sigma_panels = 8 * *std::max_element(st.begin(), st.end());
    }
    // replicated per rank: Q values + qmap over the pattern, solve vectors
    m.replicated = 16 * static_cast<i64>(s.qri.size()) + 8 * 4 * static_cast<i64>(s.n) * max_rhs;
  }
  return out;
}

}  // namespace gmrf
