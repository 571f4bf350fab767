// Supernode ownership and exchange schedule of the partitioned factorization
// (partition.hpp). Host code, no device calls: tests query it on CPU.
#include "partition.hpp"

#include <algorithm>
#include <functional>

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
  while (!todo.empty()) {
    Item it = std::move(todo.back());
    todo.pop_back();
    if (it.roots.empty()) continue;
    if (it.r1 - it.r0 == 1) {
      for (int k : it.roots) fill(k, it.r0);
      continue;
    }
    if (it.roots.size() == 1) {
      const int k = it.roots[0];
      owner[k] = it.r0;
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

}  // namespace gmrf
