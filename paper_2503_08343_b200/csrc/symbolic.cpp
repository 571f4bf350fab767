// Host symbolic analysis. See symbolic.hpp.
#include "symbolic.hpp"

#include <algorithm>
#include <cstring>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <numeric>

extern "C" int METIS_NodeND(int64_t* nvtxs, int64_t* xadj, int64_t* adjncy, int64_t* vwgt,
                            int64_t* options, int64_t* perm, int64_t* iperm);

namespace gmrf {

namespace {

// Upper pattern of P A Pᵀ: column k holds rows i < k (permuted numbering),
// built from the entries the reference reads (cholesky.hpp:32-33, 55-56).
void permuted_upper(i32 n, const i64* qcp, const i32* qri, const std::vector<i32>& pinv,
                    std::vector<i64>& ucp, std::vector<i32>& uri) {
  ucp.assign(n + 1, 0);
  for (i32 c = 0; c < n; ++c)
    for (i64 p = qcp[c]; p < qcp[c + 1]; ++p) {
      i32 pr = pinv[qri[p]], pc = pinv[c];
      if (pr < pc) ucp[pc + 1]++;
    }
  for (i32 k = 0; k < n; ++k) ucp[k + 1] += ucp[k];
  uri.resize(ucp[n]);
  std::vector<i64> next(ucp.begin(), ucp.end() - 1);
  for (i32 c = 0; c < n; ++c)
    for (i64 p = qcp[c]; p < qcp[c + 1]; ++p) {
      i32 pr = pinv[qri[p]], pc = pinv[c];
      if (pr < pc) uri[next[pc]++] = pr;
    }
}

// Liu's elimination tree with path compression (cholesky.hpp:28-43).
std::vector<i32> etree(i32 n, const std::vector<i64>& ucp, const std::vector<i32>& uri) {
  std::vector<i32> parent(n, -1), anc(n, -1);
  for (i32 k = 0; k < n; ++k)
    for (i64 p = ucp[k]; p < ucp[k + 1]; ++p) {
      i32 i = uri[p];
      while (i != -1 && i < k) {
        i32 nx = anc[i];
        anc[i] = k;
        if (nx == -1) parent[i] = k;
        i = nx;
      }
    }
  return parent;
}

std::vector<i32> postorder(i32 n, const std::vector<i32>& parent) {
  std::vector<i32> head(n, -1), next(n, -1), stack, post;
  post.reserve(n);
  for (i32 j = n - 1; j >= 0; --j) {
    if (parent[j] == -1) continue;
    next[j] = head[parent[j]];
    head[parent[j]] = j;
  }
  for (i32 root = 0; root < n; ++root) {
    if (parent[root] != -1) continue;
    stack.push_back(root);
    while (!stack.empty()) {
      i32 p = stack.back();
      i32 c = head[p];
      if (c == -1) {
        stack.pop_back();
        post.push_back(p);
      } else {
        head[p] = next[c];
        stack.push_back(c);
      }
    }
  }
  return post;
}

// Column counts of L (diagonal included) — the numbers the reference gets by
// walking every row subtree (cholesky.hpp:80-83, O(nnz(L)): 3e10 steps for the
// full config 5) — computed here in O(nnz(A) α(n)) with the skeleton-leaf
// algorithm of Gilbert, Ng and Peyton: in postorder, an entry A(i, j), i > j,
// adds one to column j when j is a leaf of row i's subtree, and the overlap of
// two consecutive leaves is removed at their least common ancestor (found with
// path-compressed disjoint sets); the per-node deltas are then summed up the
// tree. lcp/lri: lower pattern (column j holds the rows i > j). Exact.
std::vector<i64> column_counts(i32 n, const std::vector<i64>& lcp, const std::vector<i32>& lri,
                               const std::vector<i32>& parent) {
  const std::vector<i32> post = postorder(n, parent);
  std::vector<i64> delta(n, 0);
  std::vector<i32> first(n, -1), maxfirst(n, -1), prevleaf(n, -1), anc(n);
  std::iota(anc.begin(), anc.end(), 0);
  for (i32 k = 0; k < n; ++k) {
    i32 j = post[k];
    delta[j] = first[j] == -1 ? 1 : 0;  // leaves of the elimination tree start at 1
    for (; j != -1 && first[j] == -1; j = parent[j]) first[j] = k;
  }
  for (i32 k = 0; k < n; ++k) {
    const i32 j = post[k];
    if (parent[j] != -1) delta[parent[j]]--;
    for (i64 p = lcp[j]; p < lcp[j + 1]; ++p) {
      const i32 i = lri[p];
      if (first[j] <= maxfirst[i]) continue;  // j is not a leaf of row i's subtree
      maxfirst[i] = first[j];
      const i32 jprev = prevleaf[i];
      prevleaf[i] = j;
      delta[j]++;
      if (jprev == -1) continue;  // first leaf of the row subtree
      i32 q = jprev;
      while (q != anc[q]) q = anc[q];
      for (i32 t = jprev; t != q;) {  // path compression
        const i32 nx = anc[t];
        anc[t] = q;
        t = nx;
      }
      delta[q]--;  // the two leaves' paths overlap from their common ancestor on
    }
    if (parent[j] != -1) anc[j] = parent[j];
  }
  for (i32 j = 0; j < n; ++j)  // parents have larger indices: children are summed first
    if (parent[j] != -1) delta[parent[j]] += delta[j];
  return delta;
}

}  // namespace

std::vector<i32> nd_order(i32 n, const i64* qcp, const i32* qri) {
  std::vector<i32> perm(n);
  if (n <= 2) {
    std::iota(perm.begin(), perm.end(), 0);
    return perm;
  }
  // Symmetrized adjacency without the diagonal.
  std::vector<i64> deg(n + 1, 0);
  for (i32 c = 0; c < n; ++c)
    for (i64 p = qcp[c]; p < qcp[c + 1]; ++p)
      if (qri[p] != c) {
        deg[c + 1]++;
        deg[qri[p] + 1]++;
      }
  for (i32 i = 0; i < n; ++i) deg[i + 1] += deg[i];
  std::vector<int64_t> adj(deg[n]);
  std::vector<i64> nx(deg.begin(), deg.end() - 1);
  for (i32 c = 0; c < n; ++c)
    for (i64 p = qcp[c]; p < qcp[c + 1]; ++p)
      if (qri[p] != c) {
        adj[nx[c]++] = qri[p];
        adj[nx[qri[p]]++] = c;
      }
  // Deduplicate each adjacency list (the pattern may already be symmetric).
  std::vector<int64_t> xadj(n + 1, 0), adjc;
  adjc.reserve(adj.size() / 2 + 1);
  std::vector<i32> mark(n, -1);
  for (i32 i = 0; i < n; ++i) {
    for (i64 p = deg[i]; p < deg[i + 1]; ++p) {
      i32 j = static_cast<i32>(adj[p]);
      if (mark[j] != i) {
        mark[j] = i;
        adjc.push_back(j);
      }
    }
    xadj[i + 1] = static_cast<int64_t>(adjc.size());
  }
  if (adjc.empty()) {
    std::iota(perm.begin(), perm.end(), 0);
    return perm;
  }
  int64_t nv = n;
  std::vector<int64_t> mp(n), mip(n);
  int rc = METIS_NodeND(&nv, xadj.data(), adjc.data(), nullptr, nullptr, mp.data(), mip.data());
  require(rc == 1, kNumerical, "METIS_NodeND failed with code " + std::to_string(rc));
  for (i32 i = 0; i < n; ++i) perm[i] = static_cast<i32>(mp[i]);
  return perm;
}

std::vector<i32> grid_nd_order(i32 nx, i32 nt, i32 xw, i32 tw, const std::vector<char>& first,
                               i32 leaf) {
  return grid_nd_order3(nx, 1, nt, xw, 1, tw, first, leaf);
}

// Geometric nested dissection of an nx × ny × nt grid (DoF t·nx·ny + y·nx + x):
// recursively cut the box across the axis with the largest extent / separator
// thickness (thickness = the pattern's coupling radius along that axis),
// number both halves, then the separator slab; boxes of ≤ leaf unknowns are
// numbered directly. `first` unknowns (Dirichlet slack) are numbered first.
std::vector<i32> grid_nd_order3(i32 nx, i32 ny, i32 nt, i32 xw, i32 yw, i32 tw,
                                const std::vector<char>& first, i32 leaf) {
  const i64 plane = static_cast<i64>(nx) * ny;
  std::vector<i32> perm;
  perm.reserve(static_cast<size_t>(plane * nt));
  for (i64 i = 0; i < plane * nt; ++i)
    if (first[static_cast<size_t>(i)]) perm.push_back(static_cast<i32>(i));
  struct Box {
    i32 lo[3], hi[3];
  };
  auto emit = [&](const Box& b) {
    for (i32 t = b.lo[2]; t < b.hi[2]; ++t)
      for (i32 y = b.lo[1]; y < b.hi[1]; ++y)
        for (i32 x = b.lo[0]; x < b.hi[0]; ++x) {
          const i64 id = t * plane + static_cast<i64>(y) * nx + x;
          if (!first[static_cast<size_t>(id)]) perm.push_back(static_cast<i32>(id));
        }
  };
  const i32 wid[3] = {xw, yw, tw};
  // explicit recursion: (box, stage) with stage 0 = split, 1 = emit separator
  struct Frame {
    Box b;
    int stage;
  };
  std::vector<Frame> st;
  st.push_back({{{0, 0, 0}, {nx, ny, nt}}, 0});
  while (!st.empty()) {
    Frame f = st.back();
    st.pop_back();
    if (f.stage == 1) {
      emit(f.b);
      continue;
    }
    const Box b = f.b;
    i32 ext[3];
    i64 vol = 1;
    for (int a = 0; a < 3; ++a) {
      ext[a] = b.hi[a] - b.lo[a];
      vol *= ext[a];
    }
    int axis = -1;
    double best = 0.0;
    for (int a = 0; a < 3; ++a)
      if (ext[a] > wid[a] + 1) {
        const double r = static_cast<double>(ext[a]) / wid[a];
        if (axis < 0 || r > best || (r == best && a == 2)) {
          axis = a;
          best = r;
        }
      }
    if (vol <= leaf || axis < 0) {
      emit(b);
      continue;
    }
    const i32 mid = b.lo[axis] + (ext[axis] - wid[axis]) / 2;
    Box lo = b, sep = b, hi = b;
    lo.hi[axis] = mid;
    sep.lo[axis] = mid;
    sep.hi[axis] = mid + wid[axis];
    hi.lo[axis] = mid + wid[axis];
    st.push_back({sep, 1});
    st.push_back({hi, 0});
    st.push_back({lo, 0});
  }
  return perm;
}

Symbolic analyze(i32 n, const i64* qcp, const i32* qri, const i32* perm_in,
                 const SymbolicOptions& opt) {
  require(n >= 0, kDimension, "symbolic_analyze: negative dimension");
  auto clk = [] {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  double t_stage = clk();
  const bool verbose = std::getenv("GMRF_VERBOSE") != nullptr;
  auto stage = [&](const char* what) {
    if (!verbose) return;
    const double t = clk();
    std::fprintf(stderr, "[gmrf] symbolic: %-30s %8.1f ms\n", what, t - t_stage);
    t_stage = t;
  };
  Symbolic s;
  s.n = n;
  s.qcp.assign(qcp, qcp + n + 1);
  s.qri.assign(qri, qri + qcp[n]);
  for (i32 c = 0; c < n; ++c) {
    require(qcp[c] <= qcp[c + 1], kStructural, "csc: col_ptr not monotone");
    for (i64 p = qcp[c]; p < qcp[c + 1]; ++p)
      require(qri[p] >= 0 && qri[p] < n, kStructural, "csc: row index out of range");
  }

  // ---- ordering ----
  if (perm_in) {
    s.perm.assign(perm_in, perm_in + n);
    std::vector<char> seen(n, 0);
    for (i32 v : s.perm) {
      require(v >= 0 && v < n && !seen[v], kDimension, "symbolic_analyze: invalid permutation");
      seen[v] = 1;
    }
  } else {
    s.perm = nd_order(n, qcp, qri);
  }
  s.pinv.assign(n, 0);
  for (i32 i = 0; i < n; ++i) s.pinv[s.perm[i]] = i;

  stage("copy + ordering");
  std::vector<i64> ucp;
  std::vector<i32> uri;
  permuted_upper(n, qcp, qri, s.pinv, ucp, uri);
  s.parent = etree(n, ucp, uri);
  stage("permuted pattern + etree");

  if ((!perm_in && opt.postorder) || (perm_in && opt.postorder_given)) {
    std::vector<i32> post = postorder(n, s.parent);
    std::vector<i32> p2(n);
    for (i32 i = 0; i < n; ++i) p2[i] = s.perm[post[i]];
    s.perm.swap(p2);
    for (i32 i = 0; i < n; ++i) s.pinv[s.perm[i]] = i;
    permuted_upper(n, qcp, qri, s.pinv, ucp, uri);
    s.parent = etree(n, ucp, uri);
  }

  stage("postorder");
  // lower pattern: column j holds rows k > j (transpose of the upper pattern)
  std::vector<i64> lcp(n + 1, 0);
  for (i32 k = 0; k < n; ++k)
    for (i64 p = ucp[k]; p < ucp[k + 1]; ++p) lcp[uri[p] + 1]++;
  for (i32 j = 0; j < n; ++j) lcp[j + 1] += lcp[j];
  std::vector<i32> lri(lcp[n]);
  {
    std::vector<i64> nx(lcp.begin(), lcp.end() - 1);
    for (i32 k = 0; k < n; ++k)
      for (i64 p = ucp[k]; p < ucp[k + 1]; ++p) lri[nx[uri[p]]++] = k;
  }
  std::vector<i64> cc = column_counts(n, lcp, lri, s.parent);
  s.colptr_l.assign(n + 1, 0);
  for (i32 j = 0; j < n; ++j) {
    s.colptr_l[j + 1] = s.colptr_l[j] + cc[j];
    s.flops_ref += static_cast<double>(cc[j]) * static_cast<double>(cc[j]);
  }
  s.nnz_l = s.colptr_l[n];
  {
    std::vector<i32> depth(n, 0);
    for (i32 j = n - 1; j >= 0; --j)
      depth[j] = s.parent[j] == -1 ? 1 : depth[s.parent[j]] + 1;
    for (i32 j = 0; j < n; ++j) s.etree_height = std::max(s.etree_height, depth[j]);
  }

  stage("column counts");
  // ---- fundamental supernodes ----
  std::vector<i32> nchild(n, 0);
  for (i32 j = 0; j < n; ++j)
    if (s.parent[j] != -1) nchild[s.parent[j]]++;
  std::vector<i32> fs_first;  // fundamental supernode starts
  for (i32 j = 0; j < n; ++j) {
    bool cont = j > 0 && s.parent[j - 1] == j && nchild[j] == 1 && cc[j - 1] == cc[j] + 1;
    if (!cont) fs_first.push_back(j);
  }
  i32 nf = static_cast<i32>(fs_first.size());
  fs_first.push_back(n);
  std::vector<i32> fcol2sn(n);
  for (i32 f = 0; f < nf; ++f)
    for (i32 j = fs_first[f]; j < fs_first[f + 1]; ++j) fcol2sn[j] = f;
  std::vector<i32> fparent(nf, -1);
  for (i32 f = 0; f < nf; ++f) {
    i32 last = fs_first[f + 1] - 1;
    if (s.parent[last] != -1) fparent[f] = fcol2sn[s.parent[last]];
  }

  // ---- relaxed amalgamation (merge a child into the contiguous parent group) ----
  // group top t: gw = width, grows = rows of the merged front, gnnz / gzero.
  std::vector<i32> rep(nf);
  std::iota(rep.begin(), rep.end(), 0);
  std::vector<double> gw(nf), grows(nf), gnnz(nf), gzero(nf, 0.0);
  auto trap = [](double w, double rows) { return w * rows - w * (w - 1.0) / 2.0; };
  for (i32 f = 0; f < nf; ++f) {
    gw[f] = fs_first[f + 1] - fs_first[f];
    grows[f] = static_cast<double>(cc[fs_first[f]]);
    gnnz[f] = trap(gw[f], grows[f]);
  }
  if (opt.amalgamate) {
    for (i32 j = nf - 2; j >= 0; --j) {
      if (fparent[j] != j + 1) continue;
      i32 t = rep[j + 1];
      double wj = gw[j], rowsj = grows[j];
      double ncols = wj + gw[t];
      double rows = wj + grows[t];
      double nnz_m = trap(ncols, rows);
      double z = gzero[t] + gzero[j] + (nnz_m - gnnz[t] - gnnz[j]);
      double zf = nnz_m > 0 ? z / nnz_m : 0.0;
      (void)rowsj;
      bool merge = ncols <= opt.relax_w0 || (ncols <= opt.relax_w1 && zf < opt.relax_z1) ||
                   (ncols <= opt.relax_w2 && zf < opt.relax_z2) || zf < opt.relax_z3;
      if (merge) {
        rep[j] = t;
        gw[t] = ncols;
        grows[t] = rows;
        gnnz[t] = nnz_m;
        gzero[t] = z;
      }
    }
  }
  // Final supernodes = groups, in ascending column order.
  s.sn_first.clear();
  for (i32 f = 0; f < nf; ++f)
    if (f == 0 || rep[f] != rep[f - 1]) s.sn_first.push_back(fs_first[f]);
  s.ns = static_cast<i32>(s.sn_first.size());
  s.sn_first.push_back(n);
  s.col2sn.assign(n, 0);
  for (i32 k = 0; k < s.ns; ++k)
    for (i32 j = s.sn_first[k]; j < s.sn_first[k + 1]; ++j) s.col2sn[j] = k;
  s.sn_parent.assign(s.ns, -1);
  for (i32 k = 0; k < s.ns; ++k) {
    i32 last = s.sn_first[k + 1] - 1;
    if (s.parent[last] != -1) s.sn_parent[k] = s.col2sn[s.parent[last]];
  }
  // children lists
  s.ch_ptr.assign(s.ns + 1, 0);
  for (i32 k = 0; k < s.ns; ++k)
    if (s.sn_parent[k] >= 0) s.ch_ptr[s.sn_parent[k] + 1]++;
  for (i32 k = 0; k < s.ns; ++k) s.ch_ptr[k + 1] += s.ch_ptr[k];
  s.ch_list.assign(s.ch_ptr[s.ns], 0);
  {
    std::vector<i32> nx(s.ch_ptr.begin(), s.ch_ptr.end() - 1);
    for (i32 k = 0; k < s.ns; ++k)
      if (s.sn_parent[k] >= 0) s.ch_list[nx[s.sn_parent[k]]++] = k;
  }

  stage("supernodes");
  // ---- supernodal row structures (from the lower pattern built above) ----
  s.sn_rptr.assign(s.ns + 1, 0);
  s.sn_rows.clear();
  std::vector<i32> mark(n, -1), buf;
  for (i32 k = 0; k < s.ns; ++k) {
    i32 f0 = s.sn_first[k], f1 = s.sn_first[k + 1];
    buf.clear();
    for (i32 j = f0; j < f1; ++j) {
      buf.push_back(j);
      mark[j] = k;
    }
    for (i32 j = f0; j < f1; ++j)
      for (i64 p = lcp[j]; p < lcp[j + 1]; ++p) {
        i32 i = lri[p];
        if (i >= f1 && mark[i] != k) {
          mark[i] = k;
          buf.push_back(i);
        }
      }
    for (i32 q = s.ch_ptr[k]; q < s.ch_ptr[k + 1]; ++q) {
      i32 c = s.ch_list[q];
      for (i64 p = s.sn_rptr[c] + s.w(c); p < s.sn_rptr[c + 1]; ++p) {
        i32 i = s.sn_rows[p];
        if (i >= f1 && mark[i] != k) {
          mark[i] = k;
          buf.push_back(i);
        }
      }
    }
    std::sort(buf.begin() + (f1 - f0), buf.end());
    s.sn_rows.insert(s.sn_rows.end(), buf.begin(), buf.end());
    s.sn_rptr[k + 1] = static_cast<i64>(s.sn_rows.size());
  }

  stage("row structures");
  // ---- extend-add maps ----
  s.relmap.assign(s.sn_rows.size(), -1);
  std::vector<i32> pos(n, -1);
  for (i32 p = 0; p < s.ns; ++p) {
    for (i64 q = s.sn_rptr[p]; q < s.sn_rptr[p + 1]; ++q)
      pos[s.sn_rows[q]] = static_cast<i32>(q - s.sn_rptr[p]);
    for (i32 q = s.ch_ptr[p]; q < s.ch_ptr[p + 1]; ++q) {
      i32 c = s.ch_list[q];
      for (i64 e = s.sn_rptr[c] + s.w(c); e < s.sn_rptr[c + 1]; ++e) {
        i32 ps = pos[s.sn_rows[e]];
        require(ps >= 0, kStructural, "symbolic: child row missing from parent structure");
        s.relmap[e] = ps;
      }
    }
  }

  // ---- levels, storage offsets, flops ----
  s.sn_level.assign(s.ns, 0);
  for (i32 k = 0; k < s.ns; ++k)
    if (s.sn_parent[k] >= 0)
      s.sn_level[s.sn_parent[k]] = std::max(s.sn_level[s.sn_parent[k]], s.sn_level[k] + 1);
  s.n_levels = 0;
  for (i32 k = 0; k < s.ns; ++k) s.n_levels = std::max(s.n_levels, s.sn_level[k] + 1);
  s.lptr.assign(s.ns + 1, 0);
  s.uptr.assign(s.ns + 1, 0);
  s.flops_sn = 0.0;
  for (i32 k = 0; k < s.ns; ++k) {
    i64 rows = s.rows(k), w = s.w(k), r = rows - w;
    s.lptr[k + 1] = s.lptr[k] + rows * w;
    s.uptr[k + 1] = s.uptr[k] + r * r;
    for (i64 j = 0; j < w; ++j) s.flops_sn += static_cast<double>(rows - j) * (rows - j);
  }
  s.nnz_l_padded = 0;
  for (i32 k = 0; k < s.ns; ++k) {
    double w = s.w(k), rows = s.rows(k);
    s.nnz_l_padded += static_cast<i64>(trap(w, rows));
  }

  stage("extend-add maps + levels");
  // ---- Q entry -> panel offset ----
  s.qmap.assign(qcp[n], -1);
  parallel_ranges(n, [&](int64_t c0, int64_t c1, int) {
    for (i32 c = static_cast<i32>(c0); c < static_cast<i32>(c1); ++c)
      for (i64 p = qcp[c]; p < qcp[c + 1]; ++p) {
        i32 pr = s.pinv[qri[p]], pc = s.pinv[c];
        if (pr > pc) continue;
        // entry A(pr, pc) with pr <= pc lands at L(pc, pr)
        i32 k = s.col2sn[pr];
        const i32* b = s.sn_rows.data() + s.sn_rptr[k];
        const i32* e = s.sn_rows.data() + s.sn_rptr[k + 1];
        const i32* it = std::lower_bound(b, e, pc);
        require(it != e && *it == pc, kStructural, "symbolic: Q entry outside L structure");
        i64 rowpos = it - b;
        s.qmap[p] = s.lptr[k] + static_cast<i64>(pr - s.sn_first[k]) * s.rows(k) + rowpos;
      }
  });
  stage("Q -> panel map");
  return s;
}

std::vector<i32> exact_l_rows(const Symbolic& s) {
  i32 n = s.n;
  std::vector<i64> ucp;
  std::vector<i32> uri;
  permuted_upper(n, s.qcp.data(), s.qri.data(), s.pinv, ucp, uri);
  std::vector<i32> rows(s.nnz_l);
  std::vector<i64> cursor(n);
  for (i32 j = 0; j < n; ++j) {
    rows[s.colptr_l[j]] = j;
    cursor[j] = s.colptr_l[j] + 1;
  }
  std::vector<i32> stamp(n, -1);
  for (i32 k = 0; k < n; ++k) {
    stamp[k] = k;
    for (i64 p = ucp[k]; p < ucp[k + 1]; ++p)
      for (i32 i = uri[p]; stamp[i] != k; i = s.parent[i]) {
        stamp[i] = k;
        rows[cursor[i]++] = k;
      }
  }
  return rows;
}

}  // namespace gmrf
