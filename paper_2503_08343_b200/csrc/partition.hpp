// Partitioned (multi-GPU) factorization: supernode ownership along the top
// nested-dissection separators and the exchange schedule.
//
// The reference is single-threaded and has no distributed
// path; this is the north_star's "partition the factorisation along the top
// nested-dissection separators ... separator Schur-complement contributions
// reduced over NVLink". Ownership is subtree-to-subcube: each rank owns whole
// subtrees of the supernodal elimination tree, the separators above them are
// owned by the lowest rank of the rank range below them. A parent/child pair
// with different owners is a cross edge; every exchange is attached to one:
//
//   factor  : U_c (the child's r_c × r_c update matrix = its Schur-complement
//             contribution) child owner → parent owner, after the chunk level
//             that completes U_c; the parent's extend-add sums it in child order
//             exactly as on one GPU (bit-identical results).
//   fsolve  : the child's update vector u_c (r_c × nrhs), after the child's level.
//   bsolve  : x restricted to the child's below-diagonal rows R_c
//             (r_c × nrhs), parent owner → child owner, after the parent's level.
//   selinv  : Σ_RR(c) (r_c × r_c) gathered from the parent's Σ front on the
//             parent owner → child owner, after the parent's first chunk level.
//
// Both sides derive the same schedule from the same symbolic, so every rank
// lists its sends and receives of an exchange point in the same order.
#pragma once

#include <vector>

#include "symbolic.hpp"

namespace gmrf {

enum XPhase : i32 { kXFactor = 0, kXFsolve = 1, kXBsolve = 2, kXSelinv = 3 };

struct XEdge {
  i32 phase;   // XPhase
  i32 point;   // level after which the message moves (ascending levels for
               // factor/fsolve, descending for bsolve/selinv)
  i32 src, dst;
  i32 sn;      // the child supernode of the cross edge
  i64 count;   // doubles (per right-hand side for the solve phases)
};

// Chunk levels of the factorization / selected-inversion plans: chunk k of
// supernode s sits at lvl0(s)+k, one above the last chunk of its deepest child;
// fronts with rows <= small_rows are factored whole and occupy one level.
// last[s] = level of the chunk that completes U_s.
void chunk_levels(const Symbolic& s, std::vector<int>& lvl0, std::vector<int>& last, int& nlev,
                  int small_rows);

// Selected inversion: which supernodes are inverted whole (blocked: W = L_JJ⁻¹
// w² plus Gn r·w doubles of staging at their top chunk level) instead of chunk by
// chunk (staging (rows − c0)·w_c per chunk level). Multi-chunk supernodes are
// admitted in index order while the staging of ALL supernodes ending on the same
// chunk level — over every rank, so a partitioned factor takes the same decisions
// (same rounding) as the single-GPU one and no rank exceeds the bound — stays
// under max_level_stage doubles; single-chunk supernodes of at least
// min_single_w columns always (same staging either way).
constexpr long long kSelBlockLevelStage = 1ll << 28;  // doubles (2 GiB)
std::vector<char> selinv_blocked(const Symbolic& s, long long max_level_stage, int min_single_w);
// Per-chunk-level staging (doubles) of the supernodes with owner[k] == rank
// (owner == nullptr: all), as DeviceFactor::build_selinv_plan lays it out.
std::vector<i64> selinv_staging(const Symbolic& s, const std::vector<i32>* owner, int rank,
                                const std::vector<char>& blocked);

// Subtree-to-subcube ownership of the supernodes for `nranks` ranks, balanced by
// subtree flops. nranks == 1 gives all zeros.
std::vector<i32> partition_owners(const Symbolic& s, int nranks);

// Every cross-edge message of all four phases, ordered by (phase, point, sn).
std::vector<XEdge> partition_schedule(const Symbolic& s, const std::vector<i32>& owner);

// First-fit lifetime packing of buffers (size, [start, end] in time steps) into
// one arena; returns offsets and the arena size.
std::vector<i64> plan_arena(const std::vector<i64>& size, const std::vector<int>& start,
                            const std::vector<int>& end, int ntime, i64& total);

// Update-matrix arenas of one rank (factorization: fo, selected inversion: so;
// offsets in doubles per supernode, sizes in arena_f / arena_s): U_k lives from
// its first chunk level to the parent's first chunk level, Σ_RR(k) from its
// gather to its last reader (DeviceFactor's storage, factor.cu).
void plan_update_arenas(const Symbolic& s, const std::vector<i32>& owner, int rank,
                        std::vector<i64>& fo, std::vector<i64>& so, i64& arena_f, i64& arena_s);

// Per-rank device memory of a partitioned factorization with selected
// inversion, from the symbolic alone (no device): the plan a multi-GPU run of
// config 5 at full size is checked against before any GPU is involved.
struct RankMemory {
  i64 l_panels = 0;        // bytes of the owned supernodes' L panels
  i64 sigma_panels = 0;    // Σ beyond L: in-place selected inversion → its per-level staging
  i64 u_arena_factor = 0;  // lifetime-packed update matrices, factorization
  i64 u_arena_selinv = 0;  // the same buffer reused for Σ_RR in the selected inversion
  i64 replicated = 0;      // Q values + map over the pattern, solve vectors
  i64 supernodes = 0;
  double flops = 0;        // Σ c² of the owned panels (padded)
  i64 total() const {
    return l_panels + sigma_panels + std::max(u_arena_factor, u_arena_selinv) + replicated;
  }
};
std::vector<RankMemory> partition_memory(const Symbolic& s, const std::vector<i32>& owner,
                                         int nranks, int max_rhs = 16);

}  // namespace gmrf
