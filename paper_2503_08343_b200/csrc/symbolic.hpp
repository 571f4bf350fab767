// Host symbolic analysis for the supernodal factorization.
//
// Replaces the reference's symbolic_analyze (core/cholesky.hpp:68-88) and, for
// the default ordering, amd_order (core/amd.hpp:294) with METIS nested
// dissection. Given the SAME permutation, parent[] and col_ptr_L[] are
// bit-exact with the reference (tests/test_symbolic.py); the supernode
// partition, row structures, extend-add maps and level schedule are new.
#pragma once

#include <cstdint>
#include <vector>

#include "common.hpp"

namespace gmrf {

struct SymbolicOptions {
  // Relaxed amalgamation thresholds (merged width, zero fraction).
  i32 relax_w0 = 8;            // always merge while width <= relax_w0
  i32 relax_w1 = 32;           // merge while width <= relax_w1 and zeros < relax_z1
  double relax_z1 = 0.6;
  i32 relax_w2 = 64;
  double relax_z2 = 0.25;
  double relax_z3 = 0.03;      // any width with zeros below this
  bool amalgamate = true;
  bool postorder = true;       // applied to orderings computed here
  bool postorder_given = false;  // also postorder a caller-supplied ordering
};

struct Symbolic {
  i32 n = 0;
  // Input pattern (full symmetric CSC, as passed by the caller).
  std::vector<i64> qcp;
  std::vector<i32> qri;

  // Ordering and reference-exact column symbolic (internal numbering).
  std::vector<i32> perm;    // new -> old
  std::vector<i32> pinv;    // old -> new
  std::vector<i32> parent;  // column elimination tree
  std::vector<i64> colptr_l;  // reference L layout (exact column counts)
  i64 nnz_l = 0;
  double flops_ref = 0.0;   // Σ_j c_j² (BASELINE.md §3 numerator)
  i32 etree_height = 0;

  // Supernodes (after relaxed amalgamation): contiguous column ranges.
  i32 ns = 0;
  std::vector<i32> sn_first;   // ns+1
  std::vector<i32> sn_parent;  // -1 for roots
  std::vector<i64> sn_rptr;    // ns+1 offsets into sn_rows
  std::vector<i32> sn_rows;    // ascending global row indices (first w = columns)
  std::vector<i32> relmap;     // parallel to sn_rows: for rows >= w, position in parent rows
  std::vector<i32> col2sn;
  std::vector<i32> ch_ptr, ch_list;  // children of each supernode, ascending
  std::vector<i32> sn_level;         // 0 = leaf; parent = 1 + max(children)
  i32 n_levels = 0;
  std::vector<i64> lptr;   // ns+1 panel offsets (rows_s * w_s doubles, column-major)
  std::vector<i64> uptr;   // ns+1 update-matrix offsets (r_s * r_s doubles)
  i64 nnz_l_padded = 0;
  double flops_sn = 0.0;   // supernodal (padded) Σ over panel columns of c²

  // Q entry -> L panel offset (upper entries of the permuted matrix, as the
  // reference reads them, cholesky.hpp:136-139); -1 for entries not used.
  std::vector<i64> qmap;

  i32 w(i32 s) const { return sn_first[s + 1] - sn_first[s]; }
  i32 rows(i32 s) const { return static_cast<i32>(sn_rptr[s + 1] - sn_rptr[s]); }
  i32 r(i32 s) const { return rows(s) - w(s); }
};

// perm == nullptr -> METIS nested dissection (postordered).
Symbolic analyze(i32 n, const i64* qcp, const i32* qri, const i32* perm,
                 const SymbolicOptions& opt = {});

// METIS NodeND fill-reducing ordering (new -> old) of a symmetric pattern.
std::vector<i32> nd_order(i32 n, const i64* qcp, const i32* qri);

// Geometric nested dissection of a structured nx × nt space-time grid (node
// t·nx + x): recursively cut the axis with the larger
// extent/thickness; separators are `tw` slices thick in time and `xw` nodes
// thick in space (the coupling radii of the precision); halves first, then
// the separator. Nodes flagged in `first` (decoupled slack coordinates) are
// ordered first. Deterministic and O(n).
std::vector<i32> grid_nd_order(i32 nx, i32 nt, i32 xw, i32 tw, const std::vector<char>& first,
                               i32 leaf = 64);
std::vector<i32> grid_nd_order3(i32 nx, i32 ny, i32 nt, i32 xw, i32 yw, i32 tw,
                                const std::vector<char>& first, i32 leaf = 64);

// Exact reference L pattern (col_ptr from s.colptr_l): row indices per column,
// ascending, diagonal first — the layout of CholeskyFactor::L
// (cholesky.hpp:93, filled at :148-158).
std::vector<i32> exact_l_rows(const Symbolic& s);

}  // namespace gmrf
