// Host side of the device factor: plan construction and launch sequences.
#include "factor.hpp"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <map>
#include <cstdlib>
#include <string>

#include "kernels.cu"  // single translation unit for all device code
#include "gemm_wide.cuh"
#include "panel.cuh"
#include "panel2.cuh"
#include "rng.hpp"
#include "small_front.cuh"
#include "solve.cuh"
#include "solve_small.cuh"
#include "selinv.cuh"
#include "solve_wide.cuh"
#include "splitk.cuh"

namespace gmrf {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

void set_smem_attrs() {
  static bool done = false;
  if (done) return;
  cuda_check(cudaFuncSetAttribute(k_gemm_wide, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  gemm_wide_smem_bytes()),
             "smem k_gemm_wide");
  cuda_check(cudaFuncSetAttribute(k_potrf_trsm<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  panel_smem_bytes<64>()),
             "smem k_potrf_trsm");
  cuda_check(cudaFuncSetAttribute(k_potrf_trsm<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  panel_smem_bytes<32>()),
             "smem k_potrf_trsm");
  cuda_check(cudaFuncSetAttribute(k_small_front<96>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  small_front_smem_bytes<96>()),
             "smem k_small_front");
  cuda_check(cudaFuncSetAttribute(k_small_front_rows<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  small_front_smem_bytes<96>()),
             "smem k_small_front_rows");
  cuda_check(cudaFuncSetAttribute(k_small_front_rows<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  small_front_smem_bytes<96>()),
             "smem k_small_front_rows");
  cuda_check(cudaFuncSetAttribute(k_small_front_rows<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  small_front_smem_bytes<96>()),
             "smem k_small_front_rows");
  cuda_check(cudaFuncSetAttribute(k_sel_diag_w<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  sel_diag_smem_bytes<64>()),
             "smem k_sel_diag");
  done = true;
}

inline int nchunks(int w) { return (w + kNB - 1) / kNB; }

// Tile GEMM launch: one CTA per 64×64 output tile.
// Timeline marker (diagnostic, GMRF_TRACE=<file>): one thread stores the
// global timer; bracketing launches on their streams (also inside the captured
// graph) gives per-level start / end times of each launch class. No numerical
// effect; adds one tiny node per marker.
__global__ void k_mark(unsigned long long* buf, int idx) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  buf[idx] = t;
}

void launch_gemm(const GemmTask* tasks, int64_t n, cudaStream_t st) {
  k_gemm_tiles<<<static_cast<unsigned>(n), 128, 0, st>>>(tasks);
}
// 128×128 tiles, TMA-staged (gemm_wide.cuh)
void launch_gemm_wide(const GemmTask* tasks, int64_t n, cudaStream_t st) {
  k_gemm_wide<<<static_cast<unsigned>(n), kWThreads, gemm_wide_smem_bytes(), st>>>(tasks);
}

template <int NR>
void set_solve_smem(int maxw) {
  const int smem_diag = (maxw * NR + 64 * 65 + kSolveFuseRows * NR) * static_cast<int>(sizeof(double));
  cuda_check(cudaFuncSetAttribute(k_fsolve_diag<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem_diag), "smem fsolve_diag");
  cuda_check(cudaFuncSetAttribute(k_bsolve_diag<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem_diag), "smem bsolve_diag");
}

template <int NR>
void set_wide_smem() {
  cuda_check(cudaFuncSetAttribute(k_fsolve_wide<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  wide_smem_bytes<NR>()), "smem fsolve_wide");
  cuda_check(cudaFuncSetAttribute(k_bsolve_wide<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  wide_smem_bytes<NR>()), "smem bsolve_wide");
}

// Algorithmic flops of one tile: 2·k per needed output entry; a tile on the
// diagonal of a symmetric update only needs its lower trapezoid.
inline double tile_flops(const GemmTask& g, bool diag) {
  const double k = static_cast<double>(g.k[0]) + g.k[1];
  const double m = g.m, n = g.n;
  const double needed = diag ? n * m - n * (n - 1.0) / 2.0 : m * n;
  return 2.0 * k * needed;
}
}  // namespace

DeviceFactor::DeviceFactor(std::shared_ptr<const Symbolic> sym, cudaStream_t stream,
                           const PartitionSpec* part)
    : sym_(std::move(sym)), stream_(stream) {
  set_smem_attrs();
  const Symbolic& s = *sym_;
  if (const char* e = std::getenv("GMRF_NO_GRAPH")) use_graph_ = e[0] == '0';
  if (const char* e = std::getenv("GMRF_PANEL1")) panel2_ = e[0] == '0';
  if (part && part->nranks > 1) {
    require(part->rank >= 0 && part->rank < part->nranks, kContract, "partition: bad rank");
    require(part->fn != nullptr, kContract, "partition: no exchange function");
    part_ = true;
    nranks_ = part->nranks;
    rank_ = part->rank;
    owner_ = part->owner.empty() ? partition_owners(s, nranks_) : part->owner;
    require(static_cast<i32>(owner_.size()) == s.ns, kContract, "partition: owner size");
    for (i32 o : owner_) require(o >= 0 && o < nranks_, kContract, "partition: owner out of range");
    xfn_ = part->fn;
    xctx_ = part->ctx;
    for (const XEdge& e : partition_schedule(s, owner_))
      if (e.src == rank_ || e.dst == rank_) sched_.push_back(e);
  }
  // storage offsets: panels of owned supernodes; update matrices of owned
  // supernodes and of the other ranks' children of owned supernodes (the
  // Schur complements received before their extend-add), packed by lifetime
  lptr_h_.assign(s.ns + 1, 0);
  for (int k = 0; k < s.ns; ++k)
    lptr_h_[k + 1] = lptr_h_[k] + (mine(k) ? static_cast<i64>(s.rows(k)) * s.w(k) : 0);
  if (const char* e = std::getenv("GMRF_U_STATIC")) u_static_ = e[0] != '0';
  if (const char* e = std::getenv("GMRF_DEFER")) defer_ = std::max(1, atoi(e));
  if (const char* e = std::getenv("GMRF_DEFER_MIN")) defer_min_ = atoll(e);
  if (const char* e = std::getenv("GMRF_INC_U")) inc_u_ = std::max(0, atoi(e));
  if (const char* e = std::getenv("GMRF_EA_SPLIT")) ea_split_ = e[0] != '0';
  if (const char* e = std::getenv("GMRF_WIDE_K")) wide_min_k_ = atoi(e);
  if (const char* e = std::getenv("GMRF_WIDE_R")) wide_min_r_ = atoi(e);
  if (const char* e = std::getenv("GMRF_GEMM_NEXT")) gemm_next_ = e[0] != '0';
  if (const char* e = std::getenv("GMRF_FUSE_FWD")) fuse_fwd_ = e[0] != '0';
  if (const char* e = std::getenv("GMRF_FUSE_LATE")) fuse_late_ = e[0] != '0';
  if (const char* e = std::getenv("GMRF_SEL_BLOCK")) sel_block_stage_ = atoll(e);  // per-level staging bound in doubles; 0: chunk chain only
  if (const char* e = std::getenv("GMRF_SEL_BLOCK_MIN")) sel_block_min_w_ = atoi(e);
  if (const char* e = std::getenv("GMRF_NEXT_TILES")) next_max_tiles_ = atoll(e);
  if (const char* e = std::getenv("GMRF_WIDE_R")) wide_min_r_ = atoi(e);
  if (const char* e = std::getenv("GMRF_INC_B")) inc_b_ = std::max(1, atoi(e));
  if (const char* e = std::getenv("GMRF_EA_CTA")) ea_cta_max_ = atoll(e);
  if (const char* e = std::getenv("GMRF_ROWS_CTAS")) rows_max_ctas_ = static_cast<unsigned>(atoi(e));
  if (const char* e = std::getenv("GMRF_TRACE")) trace_file_ = e;
  plan_update_storage();
  std::vector<i64> qm;
  if (part_) {  // Q entries of other ranks' supernodes are not stored here
    qm.resize(s.qmap.size());
    for (size_t p = 0; p < s.qmap.size(); ++p) {
      const i64 o = s.qmap[p];
      qm[p] = -1;
      if (o < 0) continue;
      const int k = static_cast<int>(std::upper_bound(s.lptr.begin(), s.lptr.end(), o) -
                                     s.lptr.begin()) - 1;
      if (mine(k)) qm[p] = o - s.lptr[k] + lptr_h_[k];
    }
    std::vector<char> cm(s.n);
    for (int j = 0; j < s.n; ++j) cm[j] = mine(s.col2sn[j]) ? 1 : 0;
    colmine_.upload(cm, stream_);
  }
  first_.upload(s.sn_first, stream_);
  rows_.upload(s.sn_rows, stream_);
  relmap_.upload(s.relmap, stream_);
  chptr_.upload(s.ch_ptr, stream_);
  chlist_.upload(s.ch_list, stream_);
  perm_.upload(s.perm, stream_);
  col2sn_.upload(s.col2sn, stream_);
  snparent_.upload(s.sn_parent, stream_);
  rptr_.upload(s.sn_rptr, stream_);
  lptr_.upload(lptr_h_, stream_);
  uptr_.upload(uptr_h_, stream_);
  uptrs_.upload(uptrs_h_, stream_);
  qmap_.upload(part_ ? qm : s.qmap, stream_);
  status_.alloc(1);
  diag_.alloc(std::max(s.n, 1));
  rdiag_.alloc(std::max(s.n, 1));
  L_.alloc(std::max<int64_t>(lptr_h_[s.ns], 1));
  U_.alloc(std::max<int64_t>(u_arena_, 1));
  q_.alloc(std::max<size_t>(s.qri.size(), 1));
  // solve schedule: supernodes grouped by tree level
  lvl_ptr_.assign(s.n_levels + 1, 0);
  for (int k = 0; k < s.ns; ++k)
    if (mine(k)) lvl_ptr_[s.sn_level[k] + 1]++;
  for (int l = 0; l < s.n_levels; ++l) lvl_ptr_[l + 1] += lvl_ptr_[l];
  std::vector<int32_t> lsn(lvl_ptr_[s.n_levels]);
  {
    std::vector<int64_t> nx(lvl_ptr_.begin(), lvl_ptr_.end() - 1);
    for (int k = 0; k < s.ns; ++k)
      if (mine(k)) lsn[nx[s.sn_level[k]]++] = k;
  }
  // wide supernodes go last in their level and get one CTA per 64-row block of
  // the triangle (solve_wide.cuh); a launch holds at most wide_cap CTAs so all
  // of them are co-resident
  set_wide_smem<1>();
  set_wide_smem<4>();
  set_wide_smem<16>();
  int nsm = 0, occ = 0;
  cuda_check(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0), "sm count");
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fsolve_wide<16>, 256,
                                                           wide_smem_bytes<16>()),
             "wide occupancy");
  const int64_t wide_cap = static_cast<int64_t>(nsm) * std::max(occ, 0);
  const int wide_w = std::getenv("GMRF_WIDE_W") ? std::atoi(std::getenv("GMRF_WIDE_W")) : kWideW;
  const int split_cols =
      std::getenv("GMRF_SPLIT_COLS") ? std::atoi(std::getenv("GMRF_SPLIT_COLS")) : kSolveSplitCols;
  auto is_wide = [&](int k) { return s.w(k) > wide_w && nchunks(s.w(k)) <= wide_cap; };
  lvl_nrm_.assign(s.n_levels, 0);
  lvl_nsm_.assign(s.n_levels, 0);
  wl_ptr_.assign(s.n_levels + 1, 0);
  wgroups_.clear();
  {
    std::vector<WideBlock> wf, wb;
    int64_t nflag = 0;
    for (int l = 0; l < s.n_levels; ++l) {
      auto b = lsn.begin() + lvl_ptr_[l], e = lsn.begin() + lvl_ptr_[l + 1];
      auto mid = std::stable_partition(b, e, [&](int32_t k) { return !is_wide(k); });
      lvl_nrm_[l] = mid - b;
      // small supernodes first: one warp each in the 1- and 4-RHS solves (solve_small.cuh)
      auto sm_end = std::stable_partition(b, mid, [&](int32_t k) {
        return s.w(k) <= kSmallSolveW && s.rows(k) <= kSmallSolveRows;
      });
      lvl_nsm_[l] = sm_end - b;
      for (auto it = mid; it != e; ++it) {
        const int k = *it, nb = nchunks(s.w(k));
        if (wgroups_.size() == static_cast<size_t>(wl_ptr_[l]) ||
            wgroups_.back().nt + nb > wide_cap)
          wgroups_.push_back({static_cast<int64_t>(wf.size()), 0});
        for (int q = 0; q < nb; ++q) wf.push_back({k, q, nb, static_cast<int32_t>(nflag)});
        for (int q = nb - 1; q >= 0; --q) wb.push_back({k, q, nb, static_cast<int32_t>(nflag)});
        wgroups_.back().nt += nb;
        nflag += nb;
      }
      wl_ptr_[l + 1] = static_cast<int64_t>(wgroups_.size());
    }
    wide_blocks_ = nflag;
    wfwd_.upload(wf, stream_);
    wbwd_.upload(wb, stream_);
    wx_.alloc(std::max<int64_t>(2 * nflag * 64 * kMaxRhs, 1));
    if (const char* e = std::getenv("GMRF_WIDE_INV")) wide_inv_ = e[0] != '0';
    if (wide_inv_ && nflag) {
      winv_.alloc(nflag * 64 * 64);
      std::vector<SelChunk> wt;
      for (const WideBlock& t : wf) {
        const int k = t.sn, rows = s.rows(k), c0 = t.b * 64;
        SelChunk c{};
        c.l = L_.p + lptr_h_[k];
        c.ld = rows;
        c.c0 = c0;
        c.w = std::min(64, s.w(k) - c0);
        c.wsn = s.w(k);
        c.rd = rdiag_.p + s.sn_first[k] + c0;
        c.dst = winv_.p + static_cast<int64_t>(t.flag0 + t.b) * 64 * 64;
        c.ldd = 64;
        wt.push_back(c);
      }
      winv_tasks_.upload(wt, stream_);
    }
  }
  lvl_sn_.upload(lsn, stream_);
  // solve workspaces: update vectors (r_s) and backward partials (tiles_s × w_s),
  // plus the 128-row tiles of every supernode's rectangular block, per level
  std::vector<int64_t> up(s.ns + 1, 0), pp(s.ns + 1, 0);
  maxw_ = 1;  // widest supernode solved by the one-CTA triangle kernels
  for (int k = 0; k < s.ns; ++k) {
    const int r = s.r(k), nt = (r + kSolveRows - 1) / kSolveRows;
    const int p = s.sn_parent[k];
    up[k + 1] = up[k] + ((mine(k) || (p >= 0 && mine(p))) ? r : 0);
    pp[k + 1] = pp[k] + (mine(k) ? static_cast<int64_t>(nt) * s.w(k) : 0);
    // over ALL supernodes: the right-hand-side blocking derived from it must be
    // the same on every rank of a partition (same exchange sequence)
    if (!is_wide(k)) maxw_ = std::max(maxw_, s.w(k));
  }
  uvptr_h_ = up;
  uv_total_ = up[s.ns];
  p_total_ = pp[s.ns];
  uvptr_.upload(up, stream_);
  pptr_.upload(pp, stream_);
  {
    // row tiles of L_RJ; wide supernodes split each row tile into column blocks
    // (forward partials in pf_, one self-resetting arrival counter per row tile)
    std::vector<SolveTile> tl;
    int32_t nslot = 0, nctr = 0;
    tile_ptr_.assign(s.n_levels + 1, 0);
    for (int l = 0; l < s.n_levels; ++l) {
      for (int64_t q = lvl_ptr_[l]; q < lvl_ptr_[l + 1]; ++q) {
        const int k = lsn[q], r = s.r(k), w = s.w(k);
        if (!is_wide(k) && r <= kSolveFuseRows) continue;  // done inside the *_diag kernels
        const int np = w > split_cols ? (w + split_cols - 1) / split_cols : 1;
        for (int t = 0; t * kSolveRows < r; ++t) {
          const int32_t slot = np > 1 ? nslot : 0, ctr = np > 1 ? nctr++ : 0;
          for (int p = 0; p < np; ++p) {
            const int c0 = np > 1 ? p * split_cols : 0;
            const int c1 = np > 1 ? std::min(w, c0 + split_cols) : w;
            tl.push_back({k, t * kSolveRows, t, c0, c1, p, np, slot, ctr});
          }
          if (np > 1) nslot += np;
        }
      }
      tile_ptr_[l + 1] = static_cast<int64_t>(tl.size());
    }
    tiles_.upload(tl, stream_);
    pf_.alloc(std::max<int64_t>(static_cast<int64_t>(nslot) * kMaxRhs * kSolveRows, 1));
    pfctr_.alloc(std::max(nctr, 1));
    cuda_check(cudaMemsetAsync(pfctr_.p, 0, pfctr_.n * sizeof(unsigned), stream_), "counters");
  }
  set_solve_smem<1>(maxw_);
  if ((200 * 1024 / 8 - 64 * 65) / (maxw_ + kSolveFuseRows) >= 4) set_solve_smem<4>(maxw_);
  if ((200 * 1024 / 8 - 64 * 65) / (maxw_ + kSolveFuseRows) >= 16) set_solve_smem<16>(maxw_);
  // solve traffic per level: the L panel (8 B/entry, lower trapezoid) + row indices
  lvl_bytes_.assign(s.n_levels, 0.0);
  for (int k = 0; k < s.ns; ++k) {
    if (!mine(k)) continue;
    const double w = s.w(k), rows = s.rows(k);
    lvl_bytes_[s.sn_level[k]] += 8.0 * (w * rows - w * (w - 1.0) / 2.0) + 4.0 * rows;
  }
  if (std::getenv("GMRF_SOLVE_STATS")) {  // diagnostic: solve schedule per level
    for (int l = 0; l < s.n_levels; ++l) {
      int64_t nsn = lvl_ptr_[l + 1] - lvl_ptr_[l], maxw = 0, maxr = 0;
      double tri = 0, rect = 0;
      for (int64_t q = lvl_ptr_[l]; q < lvl_ptr_[l + 1]; ++q) {
        const int k = lsn[q];
        const double w = s.w(k), r = s.r(k);
        maxw = std::max<int64_t>(maxw, s.w(k));
        maxr = std::max<int64_t>(maxr, s.r(k));
        tri += 8.0 * w * (w + 1) / 2;
        rect += 8.0 * w * r;
      }
      std::fprintf(stderr,
                   "solve level %d: sn %lld small %lld diag %lld wide %lld maxw %lld maxr %lld "
                   "tri %.1f MB rect %.1f MB tiles %lld\n",
                   l, (long long)nsn, (long long)lvl_nsm_[l], (long long)(lvl_nrm_[l] - lvl_nsm_[l]),
                   (long long)(nsn - lvl_nrm_[l]), (long long)maxw, (long long)maxr, tri / 1e6,
                   rect / 1e6, (long long)(tile_ptr_[l + 1] - tile_ptr_[l]));
    }
  }
  if (part_) {  // backward-solve exchange: x rows packed per cross edge
    std::vector<RowXfer> pk, un;
    std::vector<std::vector<RowXfer>> pkl(s.n_levels), unl(s.n_levels);
    int64_t off = 0;
    for (const XEdge& e : sched_) {
      if (e.phase != kXBsolve) continue;
      const RowXfer t{rows_.p + s.sn_rptr[e.sn] + s.w(e.sn), static_cast<int32_t>(e.count), off};
      bx_off_.push_back(off);
      (e.src == rank_ ? pkl : unl)[e.point].push_back(t);
      off += e.count;
    }
    bx_.assign(s.n_levels, {});
    std::vector<RowXfer> all;
    for (int l = 0; l < s.n_levels; ++l) {
      bx_[l].pk0 = static_cast<int64_t>(all.size());
      bx_[l].pkn = static_cast<int64_t>(pkl[l].size());
      all.insert(all.end(), pkl[l].begin(), pkl[l].end());
      bx_[l].up0 = static_cast<int64_t>(all.size());
      bx_[l].upn = static_cast<int64_t>(unl[l].size());
      all.insert(all.end(), unl[l].begin(), unl[l].end());
    }
    xt_.upload(all, stream_);
    xb_.alloc(std::max<int64_t>(off * kMaxRhs, 1));
  }
  build_factor_plan();
  if (std::getenv("GMRF_VERBOSE"))
    std::fprintf(stderr,
                 "[gmrf] factor storage GB: L %.2f, U arena %.2f (factor %.2f, selinv %.2f, "
                 "static %.2f), GEMM tasks %.2f, EA %.2f, solve ws/tiles %.2f\n",
                 L_.n * 8e-9, u_arena_ * 8e-9, u_arena_f_ * 8e-9, u_arena_s_ * 8e-9,
                 [&] {
                   double t = 0;
                   for (int k = 0; k < s.ns; ++k) t += double(s.r(k)) * s.r(k);
                   return t * 8e-9;
                 }(),
                 gemm_.n * sizeof(GemmTask) * 1e-9, (ea_.n * sizeof(EaTask) + eap_.n * 8) * 1e-9,
                 (tiles_.n * sizeof(SolveTile)) * 1e-9);
  {  // lookahead streams: the critical chain at high priority, the bulk updates low
    int lo = 0, hi = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priorities");
    cuda_check(cudaStreamCreateWithPriority(&main_, cudaStreamNonBlocking, hi), "main stream");
    // (numerically higher = lower priority) the bulk trailing updates feed the chain
    // a level later, so they rank above the incremental U batches
    const int mid = hi < lo ? lo - 1 : lo;
    cuda_check(cudaStreamCreateWithPriority(&aux_, cudaStreamNonBlocking, mid), "aux stream");
    cuda_check(cudaStreamCreateWithPriority(&uu_, cudaStreamNonBlocking, lo), "update stream");
    cuda_check(cudaStreamCreateWithPriority(&sf_, cudaStreamNonBlocking, lo), "fused-solve stream");
    cuda_check(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&ev_fs_, cudaEventDisableTiming), "event");
  }
  ev_panel_.resize(flev_.size());
  ev_rest_.resize(flev_.size());
  ev_uupd_.resize(flev_.size());
  ev_eau_.resize(flev_.size());
  if (!trace_file_.empty()) tbuf_.alloc(flev_.size() * kTraceSlots);
  for (size_t l = 0; l < flev_.size(); ++l) {
    cuda_check(cudaEventCreateWithFlags(&ev_panel_[l], cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&ev_rest_[l], cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&ev_uupd_[l], cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&ev_eau_[l], cudaEventDisableTiming), "event");
  }
  cuda_check(cudaStreamSynchronize(stream_), "factor setup");
}

DeviceFactor::~DeviceFactor() {
  if (fgraph_) cudaGraphExecDestroy(fgraph_);
  if (fgraph_fs_) cudaGraphExecDestroy(fgraph_fs_);
  if (ev_fs_) cudaEventDestroy(ev_fs_);
  if (sf_) cudaStreamDestroy(sf_);
  for (cudaEvent_t e : ev_panel_) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_rest_) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_uupd_) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_eau_) cudaEventDestroy(e);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (uu_) cudaStreamDestroy(uu_);
  if (aux_) cudaStreamDestroy(aux_);
  if (main_) cudaStreamDestroy(main_);
}

void DeviceFactor::plan_update_storage() {
  const Symbolic& s = *sym_;
  uptr_h_.assign(s.ns + 1, 0);
  uptrs_h_.assign(s.ns + 1, 0);
  if (u_static_) {
    for (int k = 0; k < s.ns; ++k) {
      const int p = s.sn_parent[k];
      const i64 z = (p >= 0 && (mine(k) || mine(p))) ? static_cast<i64>(s.r(k)) * s.r(k) : 0;
      uptr_h_[k + 1] = uptr_h_[k] + z;
    }
    uptrs_h_ = uptr_h_;
    u_arena_ = uptr_h_[s.ns];
    u_arena_f_ = u_arena_s_ = u_arena_;
    return;
  }
  std::vector<i64> fo, so;
  plan_update_arenas(s, part_ ? owner_ : std::vector<i32>(s.ns, 0), rank_, fo, so, u_arena_f_,
                     u_arena_s_);
  for (int k = 0; k < s.ns; ++k) {
    uptr_h_[k] = fo[k];
    uptrs_h_[k] = so[k];
  }
  uptr_h_[s.ns] = u_arena_f_;
  uptrs_h_[s.ns] = u_arena_s_;
  u_arena_ = std::max(u_arena_f_, u_arena_s_);
}

SymDev DeviceFactor::symdev_sel() const {
  SymDev d = symdev();
  d.uptr = uptrs_.p;
  return d;
}

SymDev DeviceFactor::symdev() const {
  SymDev d;
  d.sn_first = first_.p;
  d.sn_rptr = rptr_.p;
  d.sn_rows = rows_.p;
  d.relmap = relmap_.p;
  d.ch_ptr = chptr_.p;
  d.ch_list = chlist_.p;
  d.lptr = lptr_.p;
  d.uptr = uptr_.p;
  d.n = sym_->n;
  return d;
}

int64_t DeviceFactor::device_bytes() const {
  return static_cast<int64_t>((L_.n + U_.n + Sig_.n + ystage_.n + q_.n + P_.n + Uv_.n + v1_.n +
                               v2_.n) *
                              sizeof(double)) +
         static_cast<int64_t>(gemm_.n * sizeof(GemmTask) + sgemm_.n * sizeof(GemmTask));
}

// Trailing updates of chunk c of a w-wide supernode (chunks of kNB columns),
// with deferral depth D = defer_: chunk f is a flush point when (f+1) % D == 0;
// a flush updates the blocks b >= f+1+D with the D chunks of its group in one
// K = D·kNB GEMM (off the chain, D levels of slack before anything touches
// those blocks), and the chain's next-block GEMM updates block c+1 with every
// chunk not yet applied to it: (last flush f <= c-D, c]. D = 1 is plain
// right-looking (next block with chunk c; rest with chunk c).
//   emit(crit, j0, j1, k0, k1): columns [j0, j1) -= L[:, k0:k1] L[j0:j1, k0:k1]ᵀ
template <class F>
void DeviceFactor::trailing_jobs(int w, int rows, int c, F&& emit) const {
  const int D = defer_of(w, rows), nch = nchunks(w);
  auto last_flush_le = [D](int x) { return x < -1 ? -1 : ((x + 1) / D) * D - 1; };
  const int c1 = std::min(w, (c + 1) * kNB);
  if (c + 1 < nch) {
    const int fb = last_flush_le(c - D);
    emit(true, c1, std::min(w, c1 + kNB), (fb + 1) * kNB, c1);
  }
  if ((c + 1) % D == 0 && c + 1 + D < nch)
    emit(false, (c + 1 + D) * kNB, w, (c + 1 - D) * kNB, c1);
}

void DeviceFactor::build_factor_plan() {
  const Symbolic& s = *sym_;
  std::vector<int> lvl0, last;
  int nlev = 0;
  chunk_levels(s, lvl0, last, nlev, kSmallRows);
  // extend-add tasks per level: panel columns (b < w, the panel step waits for
  // them) and update-block columns (only the level's U SYRKs need them)
  std::vector<std::vector<EaTask>> ea(nlev), eau(nlev);
  std::vector<int2> ea_pairs;  // (child, first row of its update column), child order
  std::vector<int32_t> cnt;
  std::vector<std::vector<PanelTask>> pan(nlev), po(nlev), pdg(nlev), ptr2(nlev);
  // GEMM tasks per level: gm = the update of the chunk's NEXT column block (on
  // the critical chain), gr = the rest of the trailing update + the U SYRK
  // (overlapped with the next level's panel on the second stream)
  std::vector<std::vector<GemmTask>> gm(nlev), gr(nlev), gu(nlev), gw(nlev);
  // small-front buckets: rows ≤ 32 / ≤ 64 (k_small_front), rows ≤ 96 with
  // w ≤ 16 / 32 / 64 (k_small_front_rows), rows ≤ 96 with w > 64 (k_small_front)
  std::vector<std::vector<int32_t>> sm[kSmBuckets];
  for (auto& v : sm) v.resize(nlev);
  std::vector<double> ea_b(nlev, 0.0), po_f(nlev, 0.0), tr_f(nlev, 0.0), gm_f(nlev, 0.0),
      gr_f(nlev, 0.0), sm_f(nlev, 0.0), gu_f(nlev, 0.0);
  double* L = L_.p;
  double* U = U_.p;
  std::vector<int64_t> gpan(3 * static_cast<size_t>(nlev), 0);  // panel tasks of all ranks
  std::vector<int64_t> ggm(nlev, 0), ggr(nlev, 0);                // GEMM tiles of all ranks
  std::vector<int> dwait(nlev, std::max(defer_, 1));  // smallest deferral depth among a level's supernodes
  std::vector<int> kcrit(nlev, 0);                    // longest K among a level's next-block updates
  for (int k = 0; k < s.ns; ++k) {
    const int w = s.w(k), rows = s.rows(k), r = rows - w;
    if (rows <= kSmallRows) continue;
    const int nch = nchunks(w);
    for (int c = 0; c < nch; ++c) {
      const int c0 = c * kNB, wk = std::min(kNB, w - c0), nbelow = rows - c0 - wk;
      const int lv = lvl0[k] + c;
      dwait[lv] = std::min(dwait[lv], defer_of(w, rows));
      gpan[3 * lv + (wk <= 16 ? 0 : (wk <= 32 ? 1 : 2))] +=
          std::max(1, (nbelow + kRowsSR - 1) / kRowsSR);
      trailing_jobs(w, rows, c, [&](bool crit, int j0, int j1, int k0, int k1) {
        for (int jb = j0; jb < j1; jb += kTile) (crit ? ggm : ggr)[lv] += (rows - jb + kTile - 1) / kTile;
        if (crit) kcrit[lv] = std::max(kcrit[lv], k1 - k0);
      });
      if (c == nch - 1 && !use_wide(r, w - (inc_u_ && nch >= inc_u_ ? (c / inc_b_) * inc_b_ * kNB : 0)))
        for (int jb = 0; jb < r; jb += kTile) ggr[lv] += (r - jb + kTile - 1) / kTile;
    }
  }
  for (int k = 0; k < s.ns; ++k) {
    if (!mine(k)) continue;
    const int w = s.w(k), rows = s.rows(k), r = rows - w;
    if (rows <= kSmallRows) {  // fused small-front kernel, bucketed by front size
      const int lv = lvl0[k];
      sm[rows <= 32 ? 0 : (rows <= 64 ? 1 : (w <= 16 ? 2 : (w <= 32 ? 3 : (w <= 64 ? 4 : 5))))][lv]
          .push_back(k);
      for (int j = 0; j < w; ++j) sm_f[lv] += static_cast<double>(rows - j) * (rows - j);
      continue;
    }
    double* Lk = L + lptr_h_[k];
    double* Uk = U + uptr_h_[k];
    const int nch = nchunks(w);
    for (int c = 0; c < nch; ++c) {
      const int lv = lvl0[k] + c;
      const int c0 = c * kNB, wk = std::min(kNB, w - c0);
      if (c == 0 && s.ch_ptr[k + 1] == s.ch_ptr[k] && r > 0) {
        // no children: the extend-add tasks only zero the update block
        for (int b = w; b < rows; ++b) eau[lv].push_back({k, b, 0, 0});
        ea_b[lv] += 4.0 * r * (r + 1.0);
      }
      if (c == 0 && s.ch_ptr[k + 1] > s.ch_ptr[k]) {
        // front column b receives child c's update column ia where rel_c[ia] = b
        cnt.assign(rows + 1, 0);
        for (int q = s.ch_ptr[k]; q < s.ch_ptr[k + 1]; ++q) {
          const int ch = s.ch_list[q], wc = s.w(ch), rc = s.r(ch);
          const int32_t* rel = s.relmap.data() + s.sn_rptr[ch] + wc;
          for (int ia = 0; ia < rc; ++ia) cnt[rel[ia] + 1]++;
          ea_b[lv] += 12.0 * rc * (rc + 1.0);  // read U_c lower (8 B) + RMW target (16 B)
        }
        const int64_t base = static_cast<int64_t>(ea_pairs.size());
        // every update-block column gets a task: it zeroes the column first
        // (replaces a memset of all update matrices per factorization)
        for (int b = 0; b < rows; ++b) {
          if (cnt[b + 1] || b >= w)
            (b < w ? ea : eau)[lv].push_back({k, b, static_cast<int32_t>(base + cnt[b]), cnt[b + 1]});
          cnt[b + 1] += cnt[b];
        }
        ea_b[lv] += 4.0 * r * (r + 1.0);
        ea_pairs.resize(base + cnt[rows]);
        for (int q = s.ch_ptr[k]; q < s.ch_ptr[k + 1]; ++q) {
          const int ch = s.ch_list[q], wc = s.w(ch), rc = s.r(ch);
          const int32_t* rel = s.relmap.data() + s.sn_rptr[ch] + wc;
          for (int ia = 0; ia < rc; ++ia) ea_pairs[base + cnt[rel[ia]]++] = make_int2(ch, ia);
        }
      }
      const int nbelow = rows - c0 - wk;
      po_f[lv] += static_cast<double>(wk) * wk * wk / 3.0;
      tr_f[lv] += static_cast<double>(nbelow) * wk * wk;
      const PanelTask pt{Lk + c0 + static_cast<int64_t>(c0) * rows, rows, wk, nbelow, 0,
                         s.sn_first[k] + c0};
      po[lv].push_back(pt);  // chunk list for the final diagonal write-back
      {  // two-phase panel (panel2.cuh): one diagonal task + 64-row slabs
        PanelTask dt = pt;
        dt.slot = static_cast<int32_t>(pdg[lv].size());
        pdg[lv].push_back(dt);
        for (int t = 0; t * kTrsm2Rows < nbelow; ++t) {
          PanelTask tt = dt;
          tt.tile = t;
          ptr2[lv].push_back(tt);
        }
      }
      for (int t = 0; t == 0 || t * kRowsSR < nbelow; ++t) {
        PanelTask tt = pt;
        tt.tile = t;
        pan[lv].push_back(tt);
      }
      // right-looking update of the trailing panel columns [j0, j1) with the
      // finished columns [k0, k1) (trailing_jobs: next block on the chain,
      // deferred bulk updates of the blocks further right)
      // levels whose next-block updates are at most about one wave of 32×32 tiles (the
      // chain at the top of the tree): one-shot operand loads, k_gemm_next
      const bool next32 = gemm_next_ && kcrit[lv] <= kNKMax && ggm[lv] <= next_max_tiles_;
      trailing_jobs(w, rows, c, [&](bool crit, int j0, int j1, int k0, int k1) {
        const int T = crit && next32 ? kNTile : kTile;
        for (int jb = j0; jb < j1; jb += T)
          for (int ib = jb; ib < rows; ib += T) {
            GemmTask g{};
            g.c = Lk + ib + static_cast<int64_t>(jb) * rows;
            g.ldc = rows;
            g.m = std::min(T, rows - ib);
            g.n = std::min(T, std::min(w, j1) - jb);
            g.a[0] = Lk + ib + static_cast<int64_t>(k0) * rows;
            g.lda[0] = rows;
            g.b[0] = Lk + jb + static_cast<int64_t>(k0) * rows;
            g.ldb[0] = rows;
            g.k[0] = k1 - k0;
            g.flags = 2;  // B transposed
            g.alpha = -1.0;
            g.beta = 1.0;
            (crit ? gm : gr)[lv].push_back(g);
            (crit ? gm_f : gr_f)[lv] += tile_flops(g, ib == jb);
          }
      });
      // wide supernodes: U -= L21(c) L21(c)ᵀ right after this chunk (K = wk), off
      // the panel chain; same per-tile accumulation order as one K = w SYRK
      // (batches of inc_b_ chunks: K = inc_b_·kNB per pass over U; the last batch
      // is the supernode's closing SYRK below)
      const bool inc = inc_u_ && nch >= inc_u_;
      const int kb0 = inc ? (c / inc_b_) * inc_b_ * kNB : 0;  // first column of chunk c's batch
      if (inc && r > 0 && (c + 1) % inc_b_ == 0 && c != nch - 1)
        for (int jb = 0; jb < r; jb += kTile)
          for (int ib = jb; ib < r; ib += kTile) {
            GemmTask g{};
            g.c = Uk + ib + static_cast<int64_t>(jb) * r;
            g.ldc = r;
            g.m = std::min(kTile, r - ib);
            g.n = std::min(kTile, r - jb);
            g.a[0] = Lk + w + ib + static_cast<int64_t>(kb0) * rows;
            g.lda[0] = rows;
            g.b[0] = Lk + w + jb + static_cast<int64_t>(kb0) * rows;
            g.ldb[0] = rows;
            g.k[0] = c0 + wk - kb0;
            g.flags = 2;
            g.alpha = -1.0;
            g.beta = 1.0;
            gu[lv].push_back(g);
            gu_f[lv] += tile_flops(g, ib == jb);
          }
      // last chunk: full-width SYRK into the update matrix, U -= L21 L21ᵀ
      const int tile_u = use_wide(r, w - kb0) ? kWTile : kTile;  // large SYRKs: 128×128 TMA-staged tiles
      if (c == nch - 1 && r > 0)
        for (int jb = 0; jb < r; jb += tile_u)
          for (int ib = jb; ib < r; ib += tile_u) {
            GemmTask g{};
            g.c = Uk + ib + static_cast<int64_t>(jb) * r;
            g.ldc = r;
            g.m = std::min(tile_u, r - ib);
            g.n = std::min(tile_u, r - jb);
            g.a[0] = Lk + w + ib + static_cast<int64_t>(kb0) * rows;
            g.lda[0] = rows;
            g.b[0] = Lk + w + jb + static_cast<int64_t>(kb0) * rows;
            g.ldb[0] = rows;
            g.k[0] = w - kb0;
            g.flags = 2;
            g.alpha = -1.0;
            g.beta = 1.0;
            (tile_u == kWTile ? gw : gr)[lv].push_back(g);
            gr_f[lv] += tile_flops(g, ib == jb);
          }
    }
  }
  std::vector<EaTask> eaf;
  std::vector<PanelTask> panf, pof, pdf, ptf;
  size_t max_slots = 1;
  std::vector<GemmTask> gmf;
  std::vector<ReduceTask> rdf;
  std::vector<int32_t> smf;
  int64_t maxp = 1, maxr = 1;
  for (int l = 0; l < nlev; ++l) {
    maxp = std::max(maxp, split_k_parts(gm[l], ggm[l]));
    maxr = std::max(maxr, split_k_parts(gr[l], ggr[l]));
  }
  // one level's split-K partial tiles at a time, per stream
  parts_.alloc(maxp * kTile * kTile);
  rparts_.alloc(maxr * kTile * kTile);
  flev_.assign(nlev, {});
  for (int l = 0; l < nlev; ++l) {
    flev_[l] = {static_cast<int64_t>(eaf.size()), static_cast<int64_t>(ea[l].size()),
                static_cast<int64_t>(pof.size()), static_cast<int64_t>(po[l].size()),
                static_cast<int64_t>(panf.size()), static_cast<int64_t>(pan[l].size()),
                0, 0, ea_b[l], po_f[l], tr_f[l], gm_f[l], {0, 0, 0}, {0, 0, 0}, 0, 0,
                {0, 0, 0}, {0, 0, 0}, 0.0};
    {
      std::vector<GemmTask> gs;
      std::vector<ReduceTask> rs;
      split_k_level(gm[l], gs, rs, parts_.p, ggm[l]);
      flev_[l].gm0 = static_cast<int64_t>(gmf.size());
      flev_[l].gmn = static_cast<int64_t>(gs.size());
      gmf.insert(gmf.end(), gs.begin(), gs.end());
      flev_[l].rd0 = static_cast<int64_t>(rdf.size());
      flev_[l].rdn = static_cast<int64_t>(rs.size());
      rdf.insert(rdf.end(), rs.begin(), rs.end());
      gs.clear();
      rs.clear();
      split_k_level(gr[l], gs, rs, rparts_.p, ggr[l]);
      flev_[l].gr0 = static_cast<int64_t>(gmf.size());
      flev_[l].grn = static_cast<int64_t>(gs.size());
      gmf.insert(gmf.end(), gs.begin(), gs.end());
      flev_[l].rr0 = static_cast<int64_t>(rdf.size());
      flev_[l].rrn = static_cast<int64_t>(rs.size());
      rdf.insert(rdf.end(), rs.begin(), rs.end());
      flev_[l].gr_flops = gr_f[l];
      flev_[l].gu0 = static_cast<int64_t>(gmf.size());
      flev_[l].gun = static_cast<int64_t>(gu[l].size());
      flev_[l].gu_flops = gu_f[l];
      gmf.insert(gmf.end(), gu[l].begin(), gu[l].end());
      flev_[l].gw0 = static_cast<int64_t>(gmf.size());
      flev_[l].gwn = static_cast<int64_t>(gw[l].size());
      gmf.insert(gmf.end(), gw[l].begin(), gw[l].end());
    }
    pof.insert(pof.end(), po[l].begin(), po[l].end());
    eaf.insert(eaf.end(), ea[l].begin(), ea[l].end());
    flev_[l].dwait = dwait[l];
    flev_[l].gm32 = gemm_next_ && kcrit[l] <= kNKMax && ggm[l] <= next_max_tiles_;
    flev_[l].eau0 = static_cast<int64_t>(eaf.size());
    flev_[l].eaun = static_cast<int64_t>(eau[l].size());
    eaf.insert(eaf.end(), eau[l].begin(), eau[l].end());
    // panel tasks grouped by width bucket (16 / 32 / 64) so each sub-launch
    // reserves only the shared memory its chunks need
    for (int bk = 0; bk < 3; ++bk) {
      flev_[l].pb0[bk] = static_cast<int64_t>(panf.size());
      for (const PanelTask& pt : pan[l]) {
        const int b = pt.w <= 16 ? 0 : (pt.w <= 32 ? 1 : 2);
        if (b == bk) panf.push_back(pt);
      }
      flev_[l].pbn[bk] = static_cast<int64_t>(panf.size()) - flev_[l].pb0[bk];
    }
    max_slots = std::max(max_slots, pdg[l].size());
    for (int bk = 0; bk < 3; ++bk) {
      flev_[l].pd0[bk] = static_cast<int64_t>(pdf.size());
      for (const PanelTask& pt : pdg[l])
        if ((pt.w <= 16 ? 0 : (pt.w <= 32 ? 1 : 2)) == bk) pdf.push_back(pt);
      flev_[l].pdn[bk] = static_cast<int64_t>(pdf.size()) - flev_[l].pd0[bk];
      flev_[l].pt0[bk] = static_cast<int64_t>(ptf.size());
      for (const PanelTask& pt : ptr2[l])
        if ((pt.w <= 16 ? 0 : (pt.w <= 32 ? 1 : 2)) == bk) ptf.push_back(pt);
      flev_[l].ptn[bk] = static_cast<int64_t>(ptf.size()) - flev_[l].pt0[bk];
    }
    for (int bk = 0; bk < kSmBuckets; ++bk) {
      flev_[l].sm0[bk] = static_cast<int64_t>(smf.size());
      flev_[l].smn[bk] = static_cast<int64_t>(sm[bk][l].size());
      smf.insert(smf.end(), sm[bk][l].begin(), sm[bk][l].end());
    }
    flev_[l].sm_flops = sm_f[l];
    for (int bk = 0; bk < 3; ++bk) flev_[l].prow[bk] = gpan[3 * l + bk] <= rows_max_ctas_;
  }
  ea_.upload(eaf, stream_);
  eap_.upload(ea_pairs, stream_);
  pan_.upload(panf, stream_);
  po_.upload(pof, stream_);
  {  // fused forward sweep: tree levels below the first wide supernode
    int lf = s.n_levels;
    for (int l = 0; l < s.n_levels; ++l)
      if (lvl_ptr_[l + 1] - lvl_ptr_[l] > lvl_nrm_[l]) {
        lf = l;
        break;
      }
    fuse_levels_ = part_ ? 0 : lf;
    fs_ready_.assign(fuse_levels_, 0);
    std::vector<std::vector<PanelTask>> byl(fuse_levels_);
    for (int k = 0; k < s.ns; ++k) {
      const int tl = s.sn_level[k];
      if (tl >= fuse_levels_) continue;
      const int w = s.w(k), rows = s.rows(k);
      if (rows <= kSmallRows) {  // small fronts leave L in its final layout
        fs_ready_[tl] = std::max(fs_ready_[tl], lvl0[k]);
        continue;
      }
      fs_ready_[tl] = std::max(fs_ready_[tl], lvl0[k] + nchunks(w) - 1);
      double* Lk = L + lptr_h_[k];
      for (int c0 = 0; c0 < w; c0 += kNB) {
        const int wk = std::min(kNB, w - c0);
        byl[tl].push_back({Lk + c0 + static_cast<int64_t>(c0) * rows, rows, wk, rows - c0 - wk, 0,
                           s.sn_first[k] + c0});
      }
    }
    for (int l = 1; l < fuse_levels_; ++l) fs_ready_[l] = std::max(fs_ready_[l], fs_ready_[l - 1]);
    // A/B knob: hold the sweep back until the one-wave chain at the top of the tree.
    // Measured on config 4 (per factorization + solve): sweep as soon as ready +0.21 ms
    // of factorization for 0.50 ms less solve; held back +0.32 ms (its CTAs delay the
    // chain's launches more than they cost beside the throughput-bound bottom levels).
    if (fuse_late_) {
      int start = nlev;
      for (int li = nlev - 1; li >= 0; --li) {
        if (!(flev_[li].prow[0] && flev_[li].prow[1] && flev_[li].prow[2])) break;
        start = li;
      }
      if (start < nlev)
        for (int l = 0; l < fuse_levels_; ++l) fs_ready_[l] = std::max(fs_ready_[l], start);
    }
    std::vector<PanelTask> flat;
    pof_ptr_.assign(fuse_levels_ + 1, 0);
    for (int l = 0; l < fuse_levels_; ++l) {
      flat.insert(flat.end(), byl[l].begin(), byl[l].end());
      pof_ptr_[l + 1] = static_cast<int64_t>(flat.size());
    }
    pof_.upload(flat, stream_);
  }
  pd_.upload(pdf, stream_);
  pt_.upload(ptf, stream_);
  stage_.alloc(max_slots * kL11Slot);
  gemm_.upload(gmf, stream_);
  red_.upload(rdf, stream_);
  small_.upload(smf, stream_);
  fx_.assign(nlev, {});
  for (const XEdge& e : sched_)
    if (e.phase == kXFactor)
      fx_[e.point].push_back({e.src == rank_ ? 0 : 1, e.src == rank_ ? e.dst : e.src, e.sn,
                              kXFactor, U + uptr_h_[e.sn], e.count});
}

void DeviceFactor::build_selinv_plan() {
  const Symbolic& s = *sym_;
  // in place: Σ overwrites L chunk by chunk (each chunk's L is dead once its Σ
  // columns exist: Y and W = L_{R,J}ᵀ Y are staged in a per-level workspace
  // first), halving the factor's memory for the full config 5
  if (!sel_inplace_) Sig_.alloc(std::max<int64_t>(lptr_h_[s.ns], 1));
  std::vector<int> lvl0, last;
  int nlev = 0;
  chunk_levels(s, lvl0, last, nlev, 0);
  // per-level staging: Y (nbelow × w) and W / Z (w × w) of every chunk; W = L_JJ⁻¹
  // (w × w) and Gn (r × w) of every blocked supernode at its top chunk level
  sel_blk_ = selinv_blocked(s, sel_block_stage_, sel_block_stage_ > 0 ? sel_block_min_w_ : kNB + 1);
  std::vector<int64_t> yoff = selinv_staging(s, part_ ? &owner_ : nullptr, rank_, sel_blk_);
  yoff.resize(std::max<size_t>(yoff.size(), nlev), 0);
  int64_t ymax = 1;
  for (int64_t v : yoff) ymax = std::max(ymax, v);
  ystage_.alloc(ymax);
  std::fill(yoff.begin(), yoff.end(), 0);
  std::vector<std::vector<ColTask>> ga(nlev), gg(nlev);
  std::vector<std::vector<GemmTask>> yg(nlev), zg(nlev);
  std::vector<std::vector<SelChunk>> tr(nlev), dg(nlev), mi(nlev);
  std::vector<double> ga_b(nlev, 0.0), y_f(nlev, 0.0), t_f(nlev, 0.0), z_f(nlev, 0.0),
      d_f(nlev, 0.0);
  double* L = L_.p;
  double* U = U_.p;
  double* S = sig();
  // ---- blocked selected inversion of one supernode (selinv.cuh): stage ids
  // order the launches of a level; supernodes of one level share the stages
  constexpr int kStG = 1000, kStY = 1001, kStJ = 1002, kStM = 1003;
  auto blocked_tasks = [&](int w, int r, const double* Lk, double* Sk, const double* Uk,
                           double* Wv, double* Gn, const double* rdk, auto&& gem, auto&& chk) {
    const int rows = w + r;
    const int64_t lw = w, lr = std::max(r, 1);
    for (int c0 = 0; c0 < w; c0 += kNB) {  // inverses of the diagonal blocks
      SelChunk t{};
      t.l = Lk;
      t.sig = Sk;
      t.ld = rows;
      t.c0 = c0;
      t.w = std::min(kNB, w - c0);
      t.wsn = w;
      t.rd = rdk + c0;
      t.dst = Wv + c0 + c0 * lw;
      t.ldd = w;
      chk(0, t);
    }
    int depth = 0;
    for (int bs = kNB; bs < w; bs *= 2, ++depth) {
      // [A 0; B C]⁻¹ = [A⁻¹ 0; −C⁻¹ B A⁻¹ C⁻¹]: Tᵀ = A⁻ᵀ Bᵀ goes to the (unused)
      // mirror block above the diagonal, then X = −C⁻¹ T over B's place in W
      for (int a0 = 0; a0 + bs < w; a0 += 2 * bs) {
        const int a1 = a0 + bs, c1 = std::min(a0 + 2 * bs, w), mb = c1 - a1;
        for (int i0 = 0; i0 < bs; i0 += kTile)
          for (int j0 = 0; j0 < mb; j0 += kTile) {
            GemmTask g{};
            g.c = Wv + (a0 + i0) + (a1 + j0) * lw;
            g.ldc = w;
            g.m = std::min(kTile, bs - i0);
            g.n = std::min(kTile, mb - j0);
            g.a[0] = Wv + (a0 + i0) + (a0 + i0) * lw;
            g.lda[0] = w;
            g.b[0] = Lk + (a1 + j0) + static_cast<int64_t>(a0 + i0) * rows;
            g.ldb[0] = rows;
            g.k[0] = bs - i0;
            g.flags = 1 | 2;
            g.alpha = 1.0;
            gem(1 + 2 * depth, g);
          }
        for (int i0 = 0; i0 < mb; i0 += kTile)
          for (int j0 = 0; j0 < bs; j0 += kTile) {
            GemmTask g{};
            g.c = Wv + (a1 + i0) + (a0 + j0) * lw;
            g.ldc = w;
            g.m = std::min(kTile, mb - i0);
            g.n = std::min(kTile, bs - j0);
            g.a[0] = Wv + (a1 + i0) + a1 * lw;
            g.lda[0] = w;
            g.b[0] = Wv + (a0 + j0) + a1 * lw;
            g.ldb[0] = w;
            g.k[0] = std::min(i0 + kTile, mb);
            g.flags = 2;
            g.alpha = -1.0;
            gem(2 + 2 * depth, g);
          }
      }
    }
    for (int j0 = 0; j0 < w; j0 += kTile) {
      const int nn = std::min(kTile, w - j0);
      for (int i0 = 0; i0 < r; i0 += kTile) {
        const int mm = std::min(kTile, r - i0);
        GemmTask g{};  // Gn = −L_RJ W
        g.c = Gn + i0 + j0 * lr;
        g.ldc = static_cast<int>(lr);
        g.m = mm;
        g.n = nn;
        g.a[0] = Lk + (w + i0) + static_cast<int64_t>(j0) * rows;
        g.lda[0] = rows;
        g.b[0] = Wv + j0 + j0 * lw;
        g.ldb[0] = w;
        g.k[0] = w - j0;
        g.alpha = -1.0;
        gem(kStG, g);
        GemmTask y{};  // Σ_RJ = Σ_RR Gn
        y.c = Sk + (w + i0) + static_cast<int64_t>(j0) * rows;
        y.ldc = rows;
        y.m = mm;
        y.n = nn;
        y.a[0] = Uk + i0;
        y.lda[0] = static_cast<int>(lr);
        y.b[0] = Gn + j0 * lr;
        y.ldb[0] = static_cast<int>(lr);
        y.k[0] = r;
        y.alpha = 1.0;
        gem(kStY, y);
      }
      for (int i0 = j0; i0 < w; i0 += kTile) {
        const int mm = std::min(kTile, w - i0);
        GemmTask g{};  // Σ_JJ = Wᵀ W + Gnᵀ Σ_RJ (lower tiles, mirrored afterwards)
        g.c = Sk + i0 + static_cast<int64_t>(j0) * rows;
        g.ldc = rows;
        g.m = mm;
        g.n = nn;
        g.a[0] = Wv + i0 + i0 * lw;
        g.lda[0] = w;
        g.b[0] = Wv + i0 + j0 * lw;
        g.ldb[0] = w;
        g.k[0] = w - i0;
        g.flags = 1;
        if (r > 0) {
          g.a[1] = Gn + i0 * lr;
          g.lda[1] = static_cast<int>(lr);
          g.b[1] = Sk + w + static_cast<int64_t>(j0) * rows;
          g.ldb[1] = rows;
          g.k[1] = r;
          g.flags |= 1 << 2;
        }
        g.alpha = 1.0;
        gem(kStJ, g);
        SelChunk t{};
        t.sig = Sk;
        t.ld = rows;
        t.c0 = i0;
        t.tile = j0;
        t.w = mm;
        t.wsn = nn;
        chk(kStM, t);
      }
    }
  };
  struct StageBuild {
    std::vector<GemmTask> g;
    std::vector<SelChunk> c;
    int64_t tiles_all = 0;  // GEMM tiles of every rank (split-K decided on these)
    double flops = 0.0;
  };
  std::vector<std::map<int, StageBuild>> bsb(nlev);
  for (int k = 0; k < s.ns; ++k) {  // tile counts over all ranks' supernodes
    const int w = s.w(k);
    if (!sel_blk_[k]) continue;
    auto& lv = bsb[lvl0[k] + nchunks(w) - 1];
    blocked_tasks(w, s.rows(k) - w, L, L, L, L, L, L,
                  [&](int st, const GemmTask&) { ++lv[st].tiles_all; },
                  [&](int, const SelChunk&) {});
  }
  for (int k = 0; k < s.ns; ++k) {
    const int w = s.w(k), rows = s.rows(k), r = rows - w;
    const int par = s.sn_parent[k];
    if (!mine(k)) {
      // another rank's child of an owned supernode: its Σ_RR is gathered here
      // from the parent's Σ front once the parent is done, then sent
      if (par >= 0 && mine(par) && r > 0) {
        for (int b = 0; b < r; ++b) gg[lvl0[par]].push_back({k, b});
        ga_b[lvl0[par]] += 16.0 * r * r;
      }
      continue;
    }
    double* Lk = L + lptr_h_[k];
    double* Sk = S + lptr_h_[k];
    double* Uk = U + uptrs_h_[k];
    const int nch = nchunks(w);
    if (sel_blk_[k]) {
      const int lv = lvl0[k] + nch - 1;
      if (r > 0 && mine(par)) {  // else received from the parent's rank
        for (int b = 0; b < r; ++b) ga[lv].push_back({k, b});
        ga_b[lv] += 16.0 * r * r;
      }
      double* Wv = ystage_.p + yoff[lv];
      double* Gn = Wv + static_cast<int64_t>(w) * w;
      yoff[lv] += static_cast<int64_t>(w) * w + static_cast<int64_t>(r) * w;
      auto& lvb = bsb[lv];
      blocked_tasks(w, r, Lk, Sk, Uk, Wv, Gn, rdiag_.p + s.sn_first[k],
                    [&](int st, const GemmTask& g) {
                      lvb[st].g.push_back(g);
                      lvb[st].flops += 2.0 * g.m * g.n * (static_cast<double>(g.k[0]) + g.k[1]);
                    },
                    [&](int st, const SelChunk& c) {
                      lvb[st].c.push_back(c);
                      if (st == 0) lvb[st].flops += static_cast<double>(c.w) * c.w * c.w / 3.0;
                    });
      continue;
    }
    for (int c = nch - 1; c >= 0; --c) {
      const int lv = lvl0[k] + c;
      const int c0 = c * kNB, wk = std::min(kNB, w - c0);
      const int p = w - c0 - wk;
      if (c == nch - 1 && r > 0 && mine(par)) {  // else received from the parent's rank
        for (int b = 0; b < r; ++b) ga[lv].push_back({k, b});
        ga_b[lv] += 16.0 * r * r;  // read parent Σ entries + write Σ_RR
      }
      {
        const double nb = rows - c0 - wk;
        y_f[lv] += 2.0 * nb * nb * wk;
        t_f[lv] += nb * wk * wk;
        z_f[lv] += 2.0 * nb * wk * wk;
        d_f[lv] += 2.0 * wk * wk * wk;
      }
      const int nbelow = rows - c0 - wk;
      double* Yst = ystage_.p + yoff[lv];          // Y: nbelow × wk, ld nbelow
      double* Wst = Yst + static_cast<int64_t>(nbelow) * wk;  // W, then Z: wk × wk
      yoff[lv] += static_cast<int64_t>(nbelow + wk) * wk;
      auto ytile = [&](int i0, int i1) {
        GemmTask g{};
        g.c = Yst + (i0 - c0 - wk);
        g.ldc = std::max(nbelow, 1);
        g.m = i1 - i0;
        g.n = wk;
        g.alpha = 1.0;
        g.beta = 0.0;
        // seg0: Σ[i, P] · L[P, J]
        g.a[0] = Sk + i0 + static_cast<int64_t>(c0 + wk) * rows;
        g.lda[0] = rows;
        g.b[0] = Lk + (c0 + wk) + static_cast<int64_t>(c0) * rows;
        g.ldb[0] = rows;
        g.k[0] = p;
        if (i0 < w) {
          // seg1: Σ[R, i]ᵀ · L[R, J]
          g.a[1] = Sk + w + static_cast<int64_t>(i0) * rows;
          g.lda[1] = rows;
          g.flags |= 1 << 2;  // A transposed
        } else {
          g.a[1] = Uk + (i0 - w);
          g.lda[1] = std::max(r, 1);
        }
        g.b[1] = Lk + w + static_cast<int64_t>(c0) * rows;
        g.ldb[1] = rows;
        g.k[1] = r;
        yg[lv].push_back(g);
      };
      for (int i0 = c0 + wk; i0 < w; i0 += kTile) ytile(i0, std::min(i0 + kTile, w));
      for (int i0 = w; i0 < rows; i0 += kTile) ytile(i0, std::min(i0 + kTile, rows));
      const double* rdc = rdiag_.p + s.sn_first[k] + c0;
      // W = L_{R,J}ᵀ Y (before Σ_{R,J} may overwrite L_{R,J}); Z = −W L_JJ⁻¹ =
      // L_{R,J}ᵀ Σ_{R,J} (takahashi.hpp:43-60 in supernodal form)
      GemmTask z{};
      z.c = Wst;
      z.ldc = wk;
      z.m = wk;
      z.n = wk;
      z.a[0] = Lk + (c0 + wk) + static_cast<int64_t>(c0) * rows;
      z.lda[0] = rows;
      z.b[0] = Yst;
      z.ldb[0] = std::max(nbelow, 1);
      z.k[0] = nbelow;
      z.flags = 1;  // A transposed
      z.alpha = 1.0;
      z.beta = 0.0;
      zg[lv].push_back(z);
      SelChunk base{Lk, Sk, rows, c0, wk, w, 0, rdc, nullptr, nullptr, 0, 0, 0, Wst, wk};
      for (int t = 0; t * kTrsmRows < nbelow; ++t) {  // Σ_{R,J} = −Y L_JJ⁻¹ into the Σ panel
        SelChunk c = base;
        c.tile = t;
        c.src = Yst;
        c.lds = nbelow;
        c.dst = Sk + (c0 + wk) + static_cast<int64_t>(c0) * rows;
        c.ldd = rows;
        c.nrows = nbelow;
        tr[lv].push_back(c);
      }
      {  // Z = −W L_JJ⁻¹, in its staging slot
        SelChunk c = base;
        c.src = Wst;
        c.dst = Wst;
        c.lds = c.ldd = wk;
        c.nrows = wk;
        tr[lv].push_back(c);
      }
      dg[lv].push_back(base);
      for (int t = 0; t * 64 < p; ++t) {
        SelChunk c = base;
        c.tile = t;
        mi[lv].push_back(c);
      }
    }
  }
  std::vector<int64_t> gyt(nlev, 0), gzt(nlev, 0);  // Y / Z tiles of all ranks per level
  for (int k = 0; k < s.ns; ++k) {
    const int w = s.w(k), rows = s.rows(k);
    if (sel_blk_[k]) continue;
    for (int c = 0; c < nchunks(w); ++c) {
      const int c0 = c * kNB, wk = std::min(kNB, w - c0);
      gyt[lvl0[k] + c] += (w - c0 - wk + kTile - 1) / kTile + (rows - w + kTile - 1) / kTile;
      gzt[lvl0[k] + c] += 1;
    }
  }
  std::vector<ColTask> gaf;
  std::vector<GemmTask> gmf;
  std::vector<SelChunk> trf, dgf, mif;
  std::vector<ReduceTask> rdf;
  int64_t maxp = 1;
  for (int l = 0; l < nlev; ++l)
    maxp = std::max(maxp, std::max(split_k_parts(yg[l], gyt[l]), split_k_parts(zg[l], gzt[l])));
  for (int l = 0; l < nlev; ++l)
    for (auto& [st, b] : bsb[l]) maxp = std::max(maxp, split_k_parts(b.g, b.tiles_all));
  sparts_.alloc(maxp * kTile * kTile);
  std::vector<SelChunk> blf;
  slev_.assign(nlev, {});
  for (int l = 0; l < nlev; ++l) {
    SLevel& e = slev_[l];
    e.ga0 = gaf.size();
    e.gan = ga[l].size();
    gaf.insert(gaf.end(), ga[l].begin(), ga[l].end());
    e.gg0 = gaf.size();
    e.ggn = gg[l].size();
    gaf.insert(gaf.end(), gg[l].begin(), gg[l].end());
    std::vector<GemmTask> gs;
    std::vector<ReduceTask> rs;
    split_k_level(yg[l], gs, rs, sparts_.p, gyt[l]);
    e.y0 = gmf.size();
    e.yn = gs.size();
    gmf.insert(gmf.end(), gs.begin(), gs.end());
    e.yr0 = rdf.size();
    e.yrn = rs.size();
    rdf.insert(rdf.end(), rs.begin(), rs.end());
    gs.clear();
    rs.clear();
    split_k_level(zg[l], gs, rs, sparts_.p, gzt[l]);
    e.z0 = gmf.size();
    e.zn = gs.size();
    gmf.insert(gmf.end(), gs.begin(), gs.end());
    e.zr0 = rdf.size();
    e.zrn = rs.size();
    rdf.insert(rdf.end(), rs.begin(), rs.end());
    e.t0 = trf.size();
    e.tn = tr[l].size();
    e.d0 = dgf.size();
    e.dn = dg[l].size();
    auto bucket = [](int w) { return w <= 16 ? 0 : (w <= 32 ? 1 : 2); };
    for (int bk = 0; bk < 3; ++bk) {
      e.tb0[bk] = trf.size();
      for (const SelChunk& c : tr[l])
        if (bucket(c.w) == bk) trf.push_back(c);
      e.tbn[bk] = static_cast<int64_t>(trf.size()) - e.tb0[bk];
      e.db0[bk] = dgf.size();
      for (const SelChunk& c : dg[l])
        if (bucket(c.w) == bk) dgf.push_back(c);
      e.dbn[bk] = static_cast<int64_t>(dgf.size()) - e.db0[bk];
    }
    e.mi0 = mif.size();
    e.min_ = mi[l].size();
    mif.insert(mif.end(), mi[l].begin(), mi[l].end());
    for (auto& [st, b] : bsb[l]) {  // std::map: ascending stage id = launch order
      if (!b.g.empty()) {
        gs.clear();
        rs.clear();
        split_k_level(b.g, gs, rs, sparts_.p, b.tiles_all);
        e.bst.push_back({0, static_cast<int64_t>(gmf.size()), static_cast<int64_t>(gs.size()),
                         static_cast<int64_t>(rdf.size()), static_cast<int64_t>(rs.size()), b.flops});
        gmf.insert(gmf.end(), gs.begin(), gs.end());
        rdf.insert(rdf.end(), rs.begin(), rs.end());
      }
      if (!b.c.empty()) {
        e.bst.push_back({st == 0 ? 1 : 2, static_cast<int64_t>(blf.size()),
                         static_cast<int64_t>(b.c.size()), 0, 0, b.flops});
        blf.insert(blf.end(), b.c.begin(), b.c.end());
      }
    }
    e.ga_bytes = ga_b[l];
    e.y_flops = y_f[l];
    e.t_flops = t_f[l];
    e.z_flops = z_f[l];
    e.d_flops = d_f[l];
  }
  sga_.upload(gaf, stream_);
  sgemm_.upload(gmf, stream_);
  sred_.upload(rdf, stream_);
  strsm_.upload(trf, stream_);
  sdiag_.upload(dgf, stream_);
  smir_.upload(mif, stream_);
  sblk_.upload(blf, stream_);
  sx_.assign(nlev, {});
  for (const XEdge& e : sched_)
    if (e.phase == kXSelinv)
      sx_[e.point].push_back({e.src == rank_ ? 0 : 1, e.src == rank_ ? e.dst : e.src, e.sn,
                              kXSelinv, U + uptrs_h_[e.sn], e.count});
  selinv_plan_ = true;
}

void DeviceFactor::begin_numeric() {
  launches_numeric_ = 0;
  cuda_check(cudaMemsetAsync(L_.p, 0, L_.n * sizeof(double), stream_), "memset L");
  // update matrices: zeroed column by column by the extend-add tasks of their
  // level (k_extend_add); small fronts write theirs whole
  cuda_check(cudaMemsetAsync(status_.p, 0x7f, sizeof(int), stream_), "status");
}

int32_t DeviceFactor::numeric(const double* q, bool q_on_device) {
  const Symbolic& s = *sym_;
  const int64_t nnzq = static_cast<int64_t>(s.qri.size());
  const double* dq = q;
  if (!q_on_device) {
    if (nnzq)
      cuda_check(cudaMemcpyAsync(q_.p, q, nnzq * sizeof(double), cudaMemcpyHostToDevice, stream_),
                 "copy Q");
    dq = q_.p;
  }
  begin_numeric();
  if (nnzq) {
    int blocks = static_cast<int>(std::min<int64_t>((nnzq + 255) / 256, 148 * 16));
    k_scatter_q<<<blocks, 256, 0, stream_>>>(dq, qmap_.p, nnzq, L_.p);
    ++launches_numeric_;
  }
  return factor_panels();
}

int32_t DeviceFactor::factor_panels(const double* fwd_rhs) {
  const Symbolic& s = *sym_;
  KernelProfiler& pf = *prof_;
  const bool la = lookahead_ && !pf.on;
  const bool graph = la && !part_ && use_graph_;
  const bool fuse = fwd_rhs && graph && fuse_fwd_ && fuse_levels_ > 0;
  rhs_pending_ = false;
  if (fwd_rhs && s.n > 0) {
    ensure_solve_ws(1);
    launches_solve_ = 0;
    k_permute_gather<<<static_cast<int>(std::min<int64_t>((s.n + 255) / 256, 148 * 8)), 256, 0,
                       stream_>>>(fwd_rhs, perm_.p, s.n, 1, v1_.p);
    ++launches_solve_;
    rhs_pending_ = true;
    fwd_done_ = 0;
  }
  // The level sequence is fixed per symbolic: captured once into a CUDA graph
  // (both lookahead streams, their event edges) and replayed per factorization,
  // so the ~100-level chain at the top of the tree is not paced by host launches.
  if (graph) {
    cudaGraphExec_t& exec = fuse ? fgraph_fs_ : fgraph_;
    int64_t& glaunches = fuse ? graph_fs_launches_ : graph_launches_;
    if (!exec) {
      const int64_t l0 = launches_numeric_, s0 = launches_solve_;
      cuda_check(cudaStreamBeginCapture(main_, cudaStreamCaptureModeThreadLocal), "capture");
      enqueue_levels(main_, aux_, true, true, fuse);
      cudaGraph_t g = nullptr;
      cuda_check(cudaStreamEndCapture(main_, &g), "end capture");
      // per-node priorities (copied from the capturing streams): the chain runs
      // ahead of the bulk updates, as it does with plain stream launches
      cuda_check(cudaGraphInstantiate(&exec, g, cudaGraphInstantiateFlagUseNodePriority),
                 "graph instantiate");
      cuda_check(cudaGraphDestroy(g), "graph destroy");
      glaunches = (launches_numeric_ - l0) + (launches_solve_ - s0);
      launches_numeric_ = l0;
      launches_solve_ = s0;
    }
    cuda_check(cudaGraphLaunch(exec, stream_), "graph launch");
    dump_trace();
    launches_numeric_ += glaunches;
    if (fuse) fwd_done_ = fuse_levels_;
  } else {
    enqueue_levels(la ? main_ : stream_, la ? aux_ : stream_, la, false);
  }
  if (po_.n) {
    pf.run(stream_, "factor.diag_writeback", 0.0, 16.0 * s.n * kNB / 2.0, [&] {
      k_diag_writeback<<<static_cast<unsigned>(po_.n), 128, 0, stream_>>>(po_.p, diag_.p,
                                                                         rdiag_.p);
    });
    ++launches_numeric_;
  }
  if (winv_tasks_.n) {  // inverted diagonal blocks of the wide supernodes, for the solves
    pf.run(stream_, "factor.wide_block_inverse", winv_tasks_.n * (64.0 * 64 * 64 / 3.0), 0.0, [&] {
      k_tri_inv64<<<static_cast<unsigned>(winv_tasks_.n), 64, 0, stream_>>>(winv_tasks_.p);
    });
    ++launches_numeric_;
  }
  cuda_check(cudaGetLastError(), "factor launch");
  if (part_) exchange({{3, -1, -1, -1, status_.p, 1}});  // smallest failing pivot over ranks
  int st = INT_MAX;
  cuda_check(cudaMemcpyAsync(&st, status_.p, sizeof(int), cudaMemcpyDeviceToHost, stream_),
             "status read");
  cuda_check(cudaStreamSynchronize(stream_), "numeric factorization");
  factored_ = st == 0x7f7f7f7f;
  selinv_done_ = false;
  return factored_ ? -1 : s.perm[st];
}

// The chunk levels of one numeric factorization on the chain stream sa and the
// bulk stream sb (la: two-stream lookahead, else sa == sb == stream_). In a
// graph capture sa is the origin stream and the fork/join to stream_ is left
// to the graph launch.
void DeviceFactor::enqueue_levels(cudaStream_t sa, cudaStream_t sb, bool la, bool in_graph,
                                  bool fuse_fwd) {
  const SymDev sd = symdev();
  KernelProfiler& pf = *prof_;
  // GMRF_WHATIF_BUILD: diagnostic-only build (tools/) that drops launch classes to
  // time the rest; compiled out of the product library (results would be invalid)
#ifdef GMRF_WHATIF_BUILD
  static const int whatif = std::getenv("GMRF_WHATIF") ? atoi(std::getenv("GMRF_WHATIF")) : 0;
#else
  constexpr int whatif = 0;
#endif
  if (la && !in_graph) {
    cuda_check(cudaEventRecord(ev_fork_, stream_), "record");
    cuda_check(cudaStreamWaitEvent(sa, ev_fork_, 0), "wait");
  }
  int fs_next = 0;  // next tree level of the fused forward sweep
  for (size_t li = 0; li < flev_.size(); ++li) {
    const FLevel& lv = flev_[li];
    const int lvl = static_cast<int>(li);
    // Lookahead (two streams): sa runs assembly → panel → next-block
    // update; aux_ runs the rest of the level's trailing update and the U
    // SYRKs, concurrently with the next level's panel. Ordering:
    //   rest(l)               after panel(l)           (reads the chunk's L)
    //   assembly(l)           after rest(l-1)          (children's U SYRKs)
    //   next(l)               after rest(l-D)          (same tiles, k order; D = the level's
    //                                                   smallest deferral depth, defer_of)
    // Profiling runs keep one stream so every launch is attributed to its class.
    int64_t nsmall = 0;
    for (int bk = 0; bk < kSmBuckets; ++bk) nsmall += lv.smn[bk];
    const bool assembles = lv.ean > 0 || lv.eaun > 0 || nsmall > 0;
    if (la && li > 0 && assembles) {
      cuda_check(cudaStreamWaitEvent(sa, ev_rest_[li - 1], 0), "wait");
      cuda_check(cudaStreamWaitEvent(sa, ev_uupd_[li - 1], 0), "wait");
    }
    if (nsmall > 0) {
      pf.run(sa, pf.tag("factor.small_front", lvl), lv.sm_flops, 0.0, [&] {
        auto g = [&](int bk) { return static_cast<unsigned>(lv.smn[bk]); };
        auto sn = [&](int bk) { return small_.p + lv.sm0[bk]; };
        if (lv.smn[0])
          k_small_front<32><<<g(0), 256, small_front_smem_bytes<32>(), sa>>>(sn(0), sd, L_.p, U_.p,
                                                                           status_.p, rdiag_.p);
        if (lv.smn[1])
          k_small_front<64><<<g(1), 256, small_front_smem_bytes<64>(), sa>>>(sn(1), sd, L_.p, U_.p,
                                                                           status_.p, rdiag_.p);
        if (lv.smn[2])
          k_small_front_rows<16><<<g(2), small_rows_threads<16>(), small_front_smem_bytes<96>(),
                                   sa>>>(sn(2), sd, L_.p, U_.p, status_.p, rdiag_.p);
        if (lv.smn[3])
          k_small_front_rows<32><<<g(3), small_rows_threads<32>(), small_front_smem_bytes<96>(),
                                   sa>>>(sn(3), sd, L_.p, U_.p, status_.p, rdiag_.p);
        if (lv.smn[4])
          k_small_front_rows<64><<<g(4), small_rows_threads<64>(), small_front_smem_bytes<96>(),
                                   sa>>>(sn(4), sd, L_.p, U_.p, status_.p, rdiag_.p);
        if (lv.smn[5])
          k_small_front<96><<<g(5), 256, small_front_smem_bytes<96>(), sa>>>(sn(5), sd, L_.p, U_.p,
                                                                           status_.p, rdiag_.p);
      });
      for (int bk = 0; bk < kSmBuckets; ++bk) launches_numeric_ += lv.smn[bk] > 0;
    }
    auto mark = [&](cudaStream_t st, int slot) {
      if (tbuf_.p) k_mark<<<1, 1, 0, st>>>(tbuf_.p, lvl * kTraceSlots + slot);
    };
    mark(sa, 8);
    // extend-add: the panel columns on the chain; the update-block columns (needed
    // only by the level's U SYRKs) on the bulk stream, beside the panel step
    auto launch_ea = [&](cudaStream_t st, int64_t t0, int64_t tn, double bytes) {
      const int blocks = static_cast<int>((tn * 32 + 255) / 256);
      pf.run(st, pf.tag("factor.extend_add", lvl), 0.0, bytes, [&] {
        if (tn <= ea_cta_max_)  // few long columns (top of the tree): one CTA per column
          k_extend_add_cta<<<static_cast<unsigned>(tn), kEaCtaThreads, 0, st>>>(
              ea_.p + t0, eap_.p, sd, L_.p, U_.p);
        else
          k_extend_add<<<blocks, 256, 0, st>>>(ea_.p + t0, static_cast<int>(tn), eap_.p, sd,
                                               L_.p, U_.p);
      });
      ++launches_numeric_;
    };
    const double ea_share = lv.ean + lv.eaun > 0 ? static_cast<double>(lv.ean) / (lv.ean + lv.eaun) : 0.0;
    if (lv.ean && !(whatif & 8)) launch_ea(sa, lv.ea0, lv.ean, lv.ea_bytes * ea_share);
    mark(sa, 0);
    if (lv.eaun && !(whatif & 8)) {
      const bool split = la && li > 0 && ea_split_;
      if (split) cuda_check(cudaStreamWaitEvent(sb, ev_uupd_[li - 1], 0), "wait");
      launch_ea(split ? sb : sa, lv.eau0, lv.eaun, lv.ea_bytes * (1.0 - ea_share));
      if (split) cuda_check(cudaEventRecord(ev_eau_[li], sb), "record");
    }
    // one-wave levels (the chain at the top of the tree) keep the fused row
    // sweep: one launch, no staging round trip; multi-wave levels split
    const bool two_phase = panel2_ && !(lv.prow[0] && lv.prow[1] && lv.prow[2]);
    if (lv.pann && two_phase && !(whatif & 2)) {
      // two-phase panel: diagonal blocks once per chunk, then barrier-free
      // row-per-thread TRSM slabs (panel2.cuh)
      pf.run(sa, pf.tag("factor.potrf_trsm", lvl), lv.po_flops + lv.tr_flops, 0.0, [&] {
        if (lv.pdn[0])
          k_panel_diag<16><<<static_cast<unsigned>(lv.pdn[0]), panel_rows_diag<16>(), 0, sa>>>(
              pd_.p + lv.pd0[0], status_.p, diag_.p, rdiag_.p, stage_.p);
        if (lv.pdn[1])
          k_panel_diag<32><<<static_cast<unsigned>(lv.pdn[1]), panel_rows_diag<32>(), 0, sa>>>(
              pd_.p + lv.pd0[1], status_.p, diag_.p, rdiag_.p, stage_.p);
        if (lv.pdn[2])
          k_panel_diag<64><<<static_cast<unsigned>(lv.pdn[2]), panel_rows_diag<64>(), 0, sa>>>(
              pd_.p + lv.pd0[2], status_.p, diag_.p, rdiag_.p, stage_.p);
        if (lv.ptn[0])
          k_panel_trsm<16><<<static_cast<unsigned>(lv.ptn[0]), kTrsm2Rows, 0, sa>>>(
              pt_.p + lv.pt0[0], stage_.p);
        if (lv.ptn[1])
          k_panel_trsm<32><<<static_cast<unsigned>(lv.ptn[1]), kTrsm2Rows, 0, sa>>>(
              pt_.p + lv.pt0[1], stage_.p);
        if (lv.ptn[2])
          k_panel_trsm<64><<<static_cast<unsigned>(lv.ptn[2]), kTrsm2Rows, 0, sa>>>(
              pt_.p + lv.pt0[2], stage_.p);
      });
      for (int bk = 0; bk < 3; ++bk) launches_numeric_ += (lv.pdn[bk] > 0) + (lv.ptn[bk] > 0);
    } else if (lv.pann && !(whatif & 2)) {
      // latency-bound levels (one wave) use the row-per-thread sweep; levels
      // with several waves of chunk slabs keep the blocked smem kernel, whose
      // CTAs are small enough to co-reside 4-5 per SM
      pf.run(sa, pf.tag("factor.potrf_trsm", lvl), lv.po_flops + lv.tr_flops, 0.0, [&] {
        if (lv.pbn[0]) {
          const unsigned g = static_cast<unsigned>(lv.pbn[0]);
          if (lv.prow[0])
            k_panel_rows<16, kRowsSR><<<g, panel_rows_threads<16, kRowsSR>(), 0, sa>>>(
                pan_.p + lv.pb0[0], status_.p, diag_.p);
          else
            k_potrf_trsm<16><<<g, 128, panel_smem_bytes<16>(), sa>>>(pan_.p + lv.pb0[0],
                                                                          status_.p, diag_.p);
        }
        if (lv.pbn[1]) {
          const unsigned g = static_cast<unsigned>(lv.pbn[1]);
          if (lv.prow[1])
            k_panel_rows<32, kRowsSR><<<g, panel_rows_threads<32, kRowsSR>(), 0, sa>>>(
                pan_.p + lv.pb0[1], status_.p, diag_.p);
          else
            k_potrf_trsm<32><<<g, 128, panel_smem_bytes<32>(), sa>>>(pan_.p + lv.pb0[1],
                                                                          status_.p, diag_.p);
        }
        if (lv.pbn[2]) {
          const unsigned g = static_cast<unsigned>(lv.pbn[2]);
          if (lv.prow[2])
            k_panel_rows<64, kRowsSR><<<g, panel_rows_threads<64, kRowsSR>(), 0, sa>>>(
                pan_.p + lv.pb0[2], status_.p, diag_.p);
          else
            k_potrf_trsm<64><<<g, 128, panel_smem_bytes<64>(), sa>>>(pan_.p + lv.pb0[2],
                                                                          status_.p, diag_.p);
        }
      });
      launches_numeric_ += (lv.pbn[0] > 0) + (lv.pbn[1] > 0) + (lv.pbn[2] > 0);
    }
    mark(sa, 1);
    if (la) cuda_check(cudaEventRecord(ev_panel_[li], sa), "record");
    if (fuse_fwd) {
      // forward sweep of the tree levels whose panels are final now: diagonal
      // blocks moved into place for these chunks, then the level's solve kernels
      bool waited = false;
      for (; fs_next < fuse_levels_ && fs_ready_[fs_next] <= lvl; ++fs_next) {
        if (!waited) cuda_check(cudaStreamWaitEvent(sf_, ev_panel_[li], 0), "wait");
        waited = true;
        const int64_t nc = pof_ptr_[fs_next + 1] - pof_ptr_[fs_next];
        if (nc) {
          k_diag_writeback<<<static_cast<unsigned>(nc), 128, 0, sf_>>>(pof_.p + pof_ptr_[fs_next],
                                                                    diag_.p, rdiag_.p);
          ++launches_numeric_;
        }
        fwd_level<1>(fs_next, v1_.p, 1, sf_);
      }
    }
    // next(l) writes block c+1, last written off the chain by the flush D levels back
    if (la && li >= static_cast<size_t>(lv.dwait))
      cuda_check(cudaStreamWaitEvent(sa, ev_rest_[li - lv.dwait], 0), "wait");
    mark(sa, 2);
    if (lv.gmn && !(whatif & 4)) {
      pf.run(sa, pf.tag(lv.gm32 ? "factor.gemm_next" : "factor.gemm_dmma", lvl), lv.gm_flops, 0.0, [&] {
        if (lv.gm32)
          k_gemm_next<<<static_cast<unsigned>(lv.gmn), 128, 0, sa>>>(gemm_.p + lv.gm0);
        else
          launch_gemm(gemm_.p + lv.gm0, lv.gmn, sa);
        if (lv.rdn)
          k_reduce_parts<<<static_cast<unsigned>(lv.rdn), 256, 0, sa>>>(red_.p + lv.rd0,
                                                                             parts_.p);
      });
      launches_numeric_ += 1 + (lv.rdn > 0);
    }
    mark(sa, 3);
    if (la) cuda_check(cudaStreamWaitEvent(sb, ev_panel_[li], 0), "wait");
    // closing SYRKs of incrementally updated supernodes: after their earlier batches
    if (la && li > 0 && inc_u_) cuda_check(cudaStreamWaitEvent(sb, ev_uupd_[li - 1], 0), "wait");
    mark(sb, 4);
    if ((lv.grn || lv.gwn) && !(whatif & 1)) {
      pf.run(sb, pf.tag("factor.gemm_dmma", lvl), lv.gr_flops, 0.0, [&] {
        if (lv.gwn) launch_gemm_wide(gemm_.p + lv.gw0, lv.gwn, sb);
        if (lv.grn) launch_gemm(gemm_.p + lv.gr0, lv.grn, sb);
        if (lv.rrn)
          k_reduce_parts<<<static_cast<unsigned>(lv.rrn), 256, 0, sb>>>(red_.p + lv.rr0,
                                                                        rparts_.p);
      });
      launches_numeric_ += (lv.grn > 0) + (lv.gwn > 0) + (lv.rrn > 0);
    }
    mark(sb, 5);
    if (la) cuda_check(cudaEventRecord(ev_rest_[li], sb), "record");
    // incremental update-matrix accumulation (wide supernodes), third stream
    cudaStream_t su = la ? uu_ : sa;
    if (la) cuda_check(cudaStreamWaitEvent(su, ev_panel_[li], 0), "wait");
    if (la && li > 0 && ea_split_ && lv.eaun && lv.gun)  // U zeroed / assembled on the bulk stream
      cuda_check(cudaStreamWaitEvent(su, ev_eau_[li], 0), "wait");
    mark(su, 6);
    if (lv.gun) {
      pf.run(su, pf.tag("factor.gemm_dmma", lvl), lv.gu_flops, 0.0,
             [&] { launch_gemm(gemm_.p + lv.gu0, lv.gun, su); });
      ++launches_numeric_;
    }
    mark(su, 7);
    if (la) cuda_check(cudaEventRecord(ev_uupd_[li], su), "record");
    if (part_ && !fx_[li].empty()) {
      // Schur complements completed at this level move to the parent's rank:
      // join both chains into stream_, exchange there, fork again
      if (la) {
        cuda_check(cudaStreamWaitEvent(sa, ev_rest_[li], 0), "wait");
        cuda_check(cudaStreamWaitEvent(sa, ev_uupd_[li], 0), "wait");
        cuda_check(cudaEventRecord(ev_fork_, sa), "record");
        cuda_check(cudaStreamWaitEvent(stream_, ev_fork_, 0), "wait");
      }
      exchange(fx_[li]);
      if (la) {
        cuda_check(cudaEventRecord(ev_fork_, stream_), "record");
        cuda_check(cudaStreamWaitEvent(sa, ev_fork_, 0), "wait");
      }
    }
  }
  if (la) {  // join: the caller's stream continues after both chains
    if (!flev_.empty()) {
      cuda_check(cudaStreamWaitEvent(sa, ev_rest_[flev_.size() - 1], 0), "wait");
      cuda_check(cudaStreamWaitEvent(sa, ev_uupd_[flev_.size() - 1], 0), "wait");
    }
    if (fuse_fwd && fs_next > 0) {
      cuda_check(cudaEventRecord(ev_fs_, sf_), "record");
      cuda_check(cudaStreamWaitEvent(sa, ev_fs_, 0), "wait");
    }
    if (!in_graph) {
      cuda_check(cudaEventRecord(ev_fork_, sa), "record");
      cuda_check(cudaStreamWaitEvent(stream_, ev_fork_, 0), "wait");
    }
  }
  require(!fuse_fwd || fs_next == fuse_levels_, kContract, "fused forward sweep: levels left over");
}

void DeviceFactor::dump_trace() {
  if (!tbuf_.p) return;
  std::vector<unsigned long long> t(tbuf_.n);
  cuda_check(cudaMemcpyAsync(t.data(), tbuf_.p, t.size() * 8, cudaMemcpyDeviceToHost, stream_), "trace");
  cuda_check(cudaStreamSynchronize(stream_), "trace");
  if (FILE* f = std::fopen(trace_file_.c_str(), "a")) {
    for (size_t l = 0; l < flev_.size(); ++l) {
      std::fprintf(f, "%zu", l);
      for (int k = 0; k < kTraceSlots; ++k) std::fprintf(f, " %llu", t[l * kTraceSlots + k]);
      const FLevel& lv = flev_[l];
      long long nsm = 0;
      for (int bk = 0; bk < kSmBuckets; ++bk) nsm += lv.smn[bk];
      // task counts of the level: small fronts, extend-add columns, chunks, panel
      // slabs (row sweep / TRSM), next-block tiles, bulk tiles, one-wave flag
      std::fprintf(f, " | %lld %lld %lld %lld %lld %lld %lld %d\n", nsm, (long long)lv.ean,
                   (long long)lv.pon, (long long)lv.pann,
                   (long long)(lv.ptn[0] + lv.ptn[1] + lv.ptn[2]), (long long)lv.gmn,
                   (long long)lv.grn, int(lv.prow[0] && lv.prow[1] && lv.prow[2]));
    }
    std::fprintf(f, "end\n");
    std::fclose(f);
  }
}

void DeviceFactor::exchange(const std::vector<XferMsg>& m) {
  if (m.empty()) return;
  cuda_check(cudaGetLastError(), "launch before exchange");
  const int rc = xfn_(xctx_, m.data(), static_cast<int32_t>(m.size()), stream_);
  require(rc == 0, kCuda, "partitioned factor: exchange callback failed (" + std::to_string(rc) + ")");
}

// Solve exchange after supernode level `level`: forward — update vectors of
// cross-edge children go to the parent's rank; backward — x on the child's
// rows below its diagonal block goes from the parent's rank to the child's.
void DeviceFactor::exchange_solve(int phase, int level, int nr, double* y) {
  std::vector<XferMsg> m;
  size_t be = 0;  // index among this rank's bsolve edges (bx_off_)
  for (const XEdge& e : sched_) {
    if (e.phase == kXBsolve) ++be;
    if (e.phase != phase || e.point != level) continue;
    const bool snd = e.src == rank_;
    double* p = phase == kXFsolve ? Uv_.p + uvptr_h_[e.sn] * nr : xb_.p + bx_off_[be - 1] * nr;
    m.push_back({snd ? 0 : 1, snd ? e.dst : e.src, e.sn, phase, p, e.count * nr});
  }
  if (m.empty()) return;
  const int n = sym_->n;
  if (phase == kXBsolve && bx_[level].pkn) {
    k_rows_xfer<true><<<static_cast<unsigned>(bx_[level].pkn), 256, 0, stream_>>>(
        xt_.p + bx_[level].pk0, y, n, nr, xb_.p);
    ++launches_solve_;
  }
  exchange(m);
  if (phase == kXBsolve && bx_[level].upn) {
    k_rows_xfer<false><<<static_cast<unsigned>(bx_[level].upn), 256, 0, stream_>>>(
        xt_.p + bx_[level].up0, y, n, nr, xb_.p);
    ++launches_solve_;
  }
}

void DeviceFactor::ensure_solve_ws(int nrhs) {
  if (nrhs <= ws_nrhs_) return;
  const Symbolic& s = *sym_;
  if (fgraph_fs_) {  // the captured forward launches hold the old workspace pointers
    cuda_check(cudaStreamSynchronize(stream_), "solve workspace");
    cudaGraphExecDestroy(fgraph_fs_);
    fgraph_fs_ = nullptr;
  }
  Uv_.alloc(std::max<int64_t>(uv_total_ * nrhs, 1));
  P_.alloc(std::max<int64_t>(p_total_ * nrhs, 1));
  v1_.alloc(std::max<int64_t>(static_cast<int64_t>(s.n) * nrhs, 1));
  v2_.alloc(std::max<int64_t>(static_cast<int64_t>(s.n) * nrhs, 1));
  ws_nrhs_ = nrhs;
}

// Forward-solve launches of tree level l on stream st (solve(); also captured
// into the factorization graph by the fused forward sweep).
template <int NR>
void DeviceFactor::fwd_level(int l, double* y, int nr, cudaStream_t st) {
  const SymDev sd = symdev();
  KernelProfiler& pf = *prof_;
  const double* L = L_.p;
  const double* rdiag = rdiag_.p;
  const int32_t* lvl_sn = lvl_sn_.p;
  const int smem_diag =
      (maxw_ * NR + 64 * 65 + kSolveFuseRows * NR) * static_cast<int>(sizeof(double));
  constexpr int smem_wide = wide_smem_bytes<NR>();
  int64_t& launches = launches_solve_;
  auto coop = [&](const void* fn, int64_t grid, void** args) {
    cuda_check(cudaLaunchCooperativeKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(256), args,
                                           smem_wide, st),
               "wide solve launch");
    ++launches;
  };
  const int nrm = static_cast<int>(lvl_nrm_[l]);
  const int nw = static_cast<int>(lvl_ptr_[l + 1] - lvl_ptr_[l]) - nrm;
  const int nt = static_cast<int>(tile_ptr_[l + 1] - tile_ptr_[l]);
  const int nsm = NR <= 4 ? static_cast<int>(lvl_nsm_[l]) : 0;
  pf.run(st, pf.tag("solve.forward", l), 0.0, lvl_bytes_[l], [&] {
    if constexpr (NR <= 4) if (nsm) {
      k_fsolve_small<NR><<<(nsm + kSmallSolveWarps - 1) / kSmallSolveWarps, 32 * kSmallSolveWarps,
                           0, st>>>(lvl_sn + lvl_ptr_[l], nsm, sd, L, y, nr, Uv_.p, uvptr_.p,
                                    rdiag);
      ++launches;
    }
    if (nrm > nsm) {
      k_fsolve_diag<NR><<<nrm - nsm, 256, smem_diag, st>>>(lvl_sn + lvl_ptr_[l] + nsm, sd, L, y,
                                                           nr, Uv_.p, uvptr_.p, rdiag);
      ++launches;
    }
    if (nw) {
      k_fsolve_wide_prep<NR><<<nw, 256, 0, st>>>(lvl_sn + lvl_ptr_[l] + nrm, sd, y, nr, Uv_.p,
                                                 uvptr_.p);
      ++launches;
      for (int64_t g = wl_ptr_[l]; g < wl_ptr_[l + 1]; ++g) {
        const WideBlock* tasks = wfwd_.p + wgroups_[g].t0;
        double* xw = wx_.p;
        const double* wi = winv_.p;
        void* args[] = {&tasks, const_cast<SymDev*>(&sd), &L, &y, &nr, &rdiag, &xw, &wi};
        coop(reinterpret_cast<const void*>(k_fsolve_wide<NR>), wgroups_[g].nt, args);
      }
    }
  });
  if (nt)
    pf.run(st, pf.tag("solve.forward_off", l), 0.0, 0.0, [&] {
      k_fsolve_off<NR><<<nt, kSolveRows, 0, st>>>(tiles_.p + tile_ptr_[l], sd, L, y, nr, Uv_.p,
                                                  uvptr_.p, pf_.p, pfctr_.p);
      ++launches;
    });
}

template <int NR>
void DeviceFactor::launch_solve_levels(bool fwd, bool bwd, double* y, int nr, int fwd_from) {
  const Symbolic& s = *sym_;
  const SymDev sd = symdev();
  KernelProfiler& pf = *prof_;
  cudaStream_t st = stream_;
  const double* L = L_.p;
  const double* rdiag = rdiag_.p;
  const int32_t* lvl_sn = lvl_sn_.p;
  const int smem_diag =
      (maxw_ * NR + 64 * 65 + kSolveFuseRows * NR) * static_cast<int>(sizeof(double));
  constexpr int smem_wide = wide_smem_bytes<NR>();
  int64_t& launches = launches_solve_;
  if (wide_blocks_) {
    // every slot back to the all-ones sentinel (k_*solve_wide poll their inputs)
    cuda_check(cudaMemsetAsync(wx_.p, 0xFF, 2 * wide_blocks_ * 64 * nr * sizeof(double), st),
               "wide exchange");
    ++launches;
  }
  auto coop = [&](const void* fn, int64_t grid, void** args) {
    cuda_check(cudaLaunchCooperativeKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(256), args,
                                           smem_wide, st),
               "wide solve launch");
    ++launches;
  };
  if (fwd)
    for (int l = fwd_from; l < s.n_levels; ++l) {
      fwd_level<NR>(l, y, nr, st);
      if (part_) exchange_solve(kXFsolve, l, nr, y);
    }
  if (bwd)
    for (int l = s.n_levels - 1; l >= 0; --l) {
      const int nrm = static_cast<int>(lvl_nrm_[l]);
      const int nt = static_cast<int>(tile_ptr_[l + 1] - tile_ptr_[l]);
      if (nt)
        pf.run(st, pf.tag("solve.backward_off", l), 0.0, 0.0, [&] {
          k_bsolve_off<NR><<<nt, 256, 0, st>>>(tiles_.p + tile_ptr_[l], sd, L, y, nr, P_.p, pptr_.p);
          ++launches;
        });
      const int nsm = NR <= 4 ? static_cast<int>(lvl_nsm_[l]) : 0;
      pf.run(st, pf.tag("solve.backward", l), 0.0, lvl_bytes_[l], [&] {
        if constexpr (NR <= 4) if (nsm) {
          k_bsolve_small<NR><<<(nsm + kSmallSolveWarps - 1) / kSmallSolveWarps, 32 * kSmallSolveWarps,
                               0, st>>>(lvl_sn + lvl_ptr_[l], nsm, sd, L, y, nr, rdiag);
          ++launches;
        }
        if (nrm > nsm) {
          k_bsolve_diag<NR><<<nrm - nsm, 256, smem_diag, st>>>(lvl_sn + lvl_ptr_[l] + nsm, sd, L, y,
                                                               nr, P_.p, pptr_.p, rdiag);
          ++launches;
        }
        for (int64_t g = wl_ptr_[l]; g < wl_ptr_[l + 1]; ++g) {
          const WideBlock* tasks = wbwd_.p + wgroups_[g].t0;
          const double* P = P_.p;
          const int64_t* pptr = pptr_.p;
          double* xw = wx_.p + wide_blocks_ * 64 * nr;
          const double* wi = winv_.p;
          void* args[] = {&tasks, const_cast<SymDev*>(&sd), &L, &y, &nr, &P, &pptr, &rdiag, &xw, &wi};
          coop(reinterpret_cast<const void*>(k_bsolve_wide<NR>), wgroups_[g].nt, args);
        }
      });
      if (part_) exchange_solve(kXBsolve, l, nr, y);
    }
}

void DeviceFactor::solve(int mode, int nrhs, const double* b, double* x, bool on_device) {
  require(factored_, kContract, "solve: factor not computed (or consumed by an in-place selected inversion)");
  require(mode >= 0 && mode <= 2, kContract, "solve_triangular: unknown mode");
  const Symbolic& s = *sym_;
  const int n = s.n;
  if (n == 0 || nrhs == 0) return;
  launches_solve_ = 0;
  // right-hand sides per pass: 1, or up to 16 within the shared-memory budget
  const int cap = static_cast<int>((200 * 1024 / 8 - 64 * 65) / (maxw_ + kSolveFuseRows));
  require(cap >= 1, kContract, "solve: supernode too wide for the shared-memory triangle");
  const int nrb = nrhs == 1 ? 1 : (cap >= 16 ? 16 : (cap >= 4 ? 4 : 1));
  for (int r0 = 0; r0 < nrhs; r0 += nrb) {
    const int nr = std::min(nrb, nrhs - r0);
    ensure_solve_ws(nr);
    const double* bb = b + static_cast<int64_t>(r0) * n;
    double* xx = x + static_cast<int64_t>(r0) * n;
    const int64_t tot = static_cast<int64_t>(n) * nr;
    const int pblocks = static_cast<int>(std::min<int64_t>((tot + 255) / 256, 148 * 8));
    double* y = v1_.p;
    if (mode == 2) {
      const double* src = bb;
      if (!on_device) {
        cuda_check(cudaMemcpyAsync(v2_.p, bb, tot * sizeof(double), cudaMemcpyHostToDevice, stream_),
                   "copy b");
        src = v2_.p;
      }
      k_permute_gather<<<pblocks, 256, 0, stream_>>>(src, perm_.p, n, nr, y);
      ++launches_solve_;
    } else {
      cuda_check(cudaMemcpyAsync(y, bb, tot * sizeof(double),
                                 on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                 stream_),
                 "copy b");
    }
    const bool fwd = mode == 0 || mode == 2, bwd = mode == 1 || mode == 2;
    if (nrb == 1) launch_solve_levels<1>(fwd, bwd, y, nr);
    else if (nrb == 4) launch_solve_levels<4>(fwd, bwd, y, nr);
    else launch_solve_levels<16>(fwd, bwd, y, nr);
    if (part_) {  // each rank holds its own columns: complete y on every rank
      k_mask_cols<<<pblocks, 256, 0, stream_>>>(y, colmine_.p, n, nr);
      ++launches_solve_;
      exchange({{2, -1, -1, -1, y, tot}});
    }
    if (mode == 2) {
      double* dst = on_device ? xx : v2_.p;
      k_permute_scatter<<<pblocks, 256, 0, stream_>>>(y, perm_.p, n, nr, dst);
      ++launches_solve_;
      if (!on_device)
        cuda_check(cudaMemcpyAsync(xx, v2_.p, tot * sizeof(double), cudaMemcpyDeviceToHost, stream_),
                   "copy x");
    } else {
      cuda_check(cudaMemcpyAsync(xx, y, tot * sizeof(double),
                                 on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                 stream_),
                 "copy x");
    }
  }
  cuda_check(cudaGetLastError(), "solve launch");
  if (!on_device) cuda_check(cudaStreamSynchronize(stream_), "solve");
}

void DeviceFactor::selinv(double* diag_out, bool on_device) {
  require(factored_, kContract, "selinv: factor not computed (or consumed by an in-place selected inversion)");
  if (!selinv_plan_) build_selinv_plan();
  const Symbolic& s = *sym_;
  launches_selinv_ = 0;
  const SymDev sd = symdev_sel();
  for (int l = static_cast<int>(slev_.size()) - 1; l >= 0; --l) {
    const SLevel& e = slev_[l];
    KernelProfiler& pf = *prof_;
    if (e.gan) {
      int blocks = static_cast<int>((e.gan * 32 + 255) / 256);
      pf.run(stream_, pf.tag("selinv.gather", l), 0.0, e.ga_bytes, [&] {
        k_sel_gather<<<blocks, 256, 0, stream_>>>(sga_.p + e.ga0, static_cast<int>(e.gan), sd,
                                                 snparent_.p, sig(), U_.p);
      });
      ++launches_selinv_;
    }
    for (const SLevel::BStage& b : e.bst) {
      if (b.kind == 0) {
        pf.run(stream_, pf.tag("selinv.gemm_dmma", l), b.flops, 0.0, [&] {
          launch_gemm(sgemm_.p + b.t0, b.tn, stream_);
          if (b.rn)
            k_reduce_parts<<<static_cast<unsigned>(b.rn), 256, 0, stream_>>>(sred_.p + b.r0,
                                                                             sparts_.p);
        });
        launches_selinv_ += 1 + (b.rn > 0);
      } else if (b.kind == 1) {
        pf.run(stream_, pf.tag("selinv.diag", l), b.flops, 0.0, [&] {
          k_tri_inv64<<<static_cast<unsigned>(b.tn), 64, 0, stream_>>>(sblk_.p + b.t0);
        });
        ++launches_selinv_;
      } else {
        pf.run(stream_, pf.tag("selinv.mirror", l), 0.0, 0.0, [&] {
          k_sel_mirror_blk<<<static_cast<unsigned>(b.tn), 256, 0, stream_>>>(sblk_.p + b.t0);
        });
        ++launches_selinv_;
      }
    }
    if (e.yn) {
      pf.run(stream_, pf.tag("selinv.gemm_dmma", l), e.y_flops, 0.0, [&] {
        launch_gemm(sgemm_.p + e.y0, e.yn, stream_);
        if (e.yrn)
          k_reduce_parts<<<static_cast<unsigned>(e.yrn), 256, 0, stream_>>>(sred_.p + e.yr0,
                                                                            sparts_.p);
      });
      launches_selinv_ += 1 + (e.yrn > 0);
    }
    if (e.zn) {
      pf.run(stream_, pf.tag("selinv.gemm_dmma", l), e.z_flops, 0.0, [&] {
        launch_gemm(sgemm_.p + e.z0, e.zn, stream_);
        if (e.zrn)
          k_reduce_parts<<<static_cast<unsigned>(e.zrn), 256, 0, stream_>>>(sred_.p + e.zr0,
                                                                            sparts_.p);
      });
      launches_selinv_ += 1 + (e.zrn > 0);
    }
    if (e.tn) {
      pf.run(stream_, pf.tag("selinv.trsm", l), e.t_flops, 0.0, [&] {
        if (e.tbn[0])
          k_sel_trsm_w<16><<<static_cast<unsigned>(e.tbn[0]), kTrsmRows, 0, stream_>>>(strsm_.p +
                                                                                       e.tb0[0]);
        if (e.tbn[1])
          k_sel_trsm_w<32><<<static_cast<unsigned>(e.tbn[1]), kTrsmRows, 0, stream_>>>(strsm_.p +
                                                                                       e.tb0[1]);
        if (e.tbn[2])
          k_sel_trsm_w<64><<<static_cast<unsigned>(e.tbn[2]), kTrsmRows, 0, stream_>>>(strsm_.p +
                                                                                       e.tb0[2]);
      });
      launches_selinv_ += (e.tbn[0] > 0) + (e.tbn[1] > 0) + (e.tbn[2] > 0);
    }
    if (e.dn) {
      pf.run(stream_, pf.tag("selinv.diag", l), e.d_flops, 0.0, [&] {
        if (e.dbn[0])
          k_sel_diag_w<16><<<static_cast<unsigned>(e.dbn[0]), 32, sel_diag_smem_bytes<16>(),
                             stream_>>>(sdiag_.p + e.db0[0]);
        if (e.dbn[1])
          k_sel_diag_w<32><<<static_cast<unsigned>(e.dbn[1]), 32, sel_diag_smem_bytes<32>(),
                             stream_>>>(sdiag_.p + e.db0[1]);
        if (e.dbn[2])
          k_sel_diag_w<64><<<static_cast<unsigned>(e.dbn[2]), 64, sel_diag_smem_bytes<64>(),
                             stream_>>>(sdiag_.p + e.db0[2]);
      });
      launches_selinv_ += (e.dbn[0] > 0) + (e.dbn[1] > 0) + (e.dbn[2] > 0);
    }
    if (e.min_) {
      pf.run(stream_, pf.tag("selinv.mirror", l), 0.0, 0.0, [&] {
        k_sel_mirror<<<static_cast<unsigned>(e.min_), 256, 0, stream_>>>(smir_.p + e.mi0);
      });
      ++launches_selinv_;
    }
    if (e.ggn) {  // Σ_RR of other ranks' children, now that their parents are done
      int blocks = static_cast<int>((e.ggn * 32 + 255) / 256);
      pf.run(stream_, pf.tag("selinv.gather", l), 0.0, 0.0, [&] {
        k_sel_gather<<<blocks, 256, 0, stream_>>>(sga_.p + e.gg0, static_cast<int>(e.ggn), sd,
                                                 snparent_.p, sig(), U_.p);
      });
      ++launches_selinv_;
    }
    if (part_) exchange(sx_[l]);
  }
  double* out = diag_out;
  if (!on_device) {
    ensure_solve_ws(1);
    out = v1_.p;
  }
  if (s.n > 0) {
    k_extract_diag<<<std::max(1, std::min((s.n + 255) / 256, 148 * 8)), 256, 0, stream_>>>(
        sd, col2sn_.p, perm_.p, sig(), part_ ? colmine_.p : nullptr, out);
    ++launches_selinv_;
    if (part_) exchange({{2, -1, -1, -1, out, static_cast<int64_t>(s.n)}});
  }
  cuda_check(cudaGetLastError(), "selinv launch");
  if (!on_device) {
    cuda_check(cudaMemcpyAsync(diag_out, out, s.n * sizeof(double), cudaMemcpyDeviceToHost, stream_),
               "copy diag");
    cuda_check(cudaStreamSynchronize(stream_), "selinv");
  }
  selinv_done_ = true;
  if (sel_inplace_) factored_ = false;  // L now holds Σ: solves need a new factorization
}

// Completes the solve started by factor_panels(fwd_rhs): forward levels not
// covered by the fused sweep, backward sweep, permutation back (same launches
// as solve(kFull) on one right-hand side).
void DeviceFactor::solve_pending(double* x_dev) {
  require(factored_, kContract, "solve_pending: factor not computed");
  require(rhs_pending_, kContract, "solve_pending: no right-hand side was passed to factor_panels");
  const Symbolic& s = *sym_;
  const int n = s.n;
  rhs_pending_ = false;
  if (n == 0) return;
  double* y = v1_.p;
  const int pblocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8));
  launch_solve_levels<1>(true, true, y, 1, fwd_done_);
  if (part_) {
    k_mask_cols<<<pblocks, 256, 0, stream_>>>(y, colmine_.p, n, 1);
    ++launches_solve_;
    exchange({{2, -1, -1, -1, y, static_cast<int64_t>(n)}});
  }
  k_permute_scatter<<<pblocks, 256, 0, stream_>>>(y, perm_.p, n, 1, x_dev);
  ++launches_solve_;
  cuda_check(cudaGetLastError(), "solve launch");
}

// Batches of up to kMaxRhs samples: z drawn on the host in the reference's
// order, one multi-RHS upper solve (kUpper, cholesky.hpp:194-201), Pᵀ, + μ.
void DeviceFactor::sample_direct(const double* d_mean, int ns, uint64_t seed, double* d_out) {
  require(factored_, kContract, "sample_direct: factor not computed (or consumed by an in-place selected inversion)");
  const Symbolic& s = *sym_;
  const int n = s.n;
  if (n == 0 || ns <= 0) return;
  HostRng rng(seed);
  std::vector<double> z(static_cast<size_t>(n) * kMaxRhs);
  zb_.alloc(z.size());
  wb_.alloc(z.size());
  for (int s0 = 0; s0 < ns; s0 += kMaxRhs) {
    const int nb = std::min(kMaxRhs, ns - s0);
    for (size_t q = 0; q < static_cast<size_t>(n) * nb; ++q) z[q] = rng.normal();
    cuda_check(cudaMemcpyAsync(zb_.p, z.data(), sizeof(double) * n * nb, cudaMemcpyHostToDevice,
                               stream_), "upload z");
    solve(1, nb, zb_.p, wb_.p, true);
    double* u = d_out + static_cast<int64_t>(s0) * n;
    const int64_t tot = static_cast<int64_t>(n) * nb;
    const int blocks = static_cast<int>(std::min<int64_t>((tot + 255) / 256, 148 * 8));
    k_permute_scatter<<<blocks, 256, 0, stream_>>>(wb_.p, perm_.p, n, nb, u);
    k_add_mean<<<blocks, 256, 0, stream_>>>(d_mean, n, nb, u);
    // z is reused by the next batch: the copy above must have been consumed
    cuda_check(cudaStreamSynchronize(stream_), "sample batch");
  }
  cuda_check(cudaGetLastError(), "sample launch");
}

void DeviceFactor::rbmc_variance(const double* d_qv, const double* d_mean, int ns, uint64_t seed,
                                 double* d_var) {
  require(ns >= 2, kContract, "rbmc_variance: need at least 2 samples");
  require(factored_, kContract, "rbmc_variance: factor not computed (or consumed by an in-place selected inversion)");
  const Symbolic& s = *sym_;
  const int n = s.n;
  if (n == 0) return;
  if (!qcp_d_.p) {
    qcp_d_.upload(s.qcp, stream_);
    qri_d_.upload(s.qri, stream_);
  }
  const int gb = std::max(1, std::min((n + 255) / 256, 148 * 8));
  qdg_.alloc(n);
  k_csc_diag<<<gb, 256, 0, stream_>>>(qcp_d_.p, qri_d_.p, d_qv, n, qdg_.p);
  {
    std::vector<double> qd(n);
    cuda_check(cudaMemcpyAsync(qd.data(), qdg_.p, sizeof(double) * n, cudaMemcpyDeviceToHost,
                               stream_), "qdiag");
    cuda_check(cudaStreamSynchronize(stream_), "qdiag");
    for (double v : qd)
      if (!(v > 0.0)) fail(kNumerical, "rbmc_variance: non-positive precision diagonal");
  }
  rbm_.alloc(n);
  rbm2_.alloc(n);
  cuda_check(cudaMemsetAsync(rbm_.p, 0, sizeof(double) * n, stream_), "mm");
  cuda_check(cudaMemsetAsync(rbm2_.p, 0, sizeof(double) * n, stream_), "m2");
  ub_.alloc(static_cast<size_t>(n) * kMaxRhs);
  qc_.alloc(static_cast<size_t>(n) * kMaxRhs);
  HostRng rng(seed);
  std::vector<double> z(static_cast<size_t>(n) * kMaxRhs);
  zb_.alloc(z.size());
  wb_.alloc(z.size());
  for (int s0 = 0; s0 < ns; s0 += kMaxRhs) {
    const int nb = std::min(kMaxRhs, ns - s0);
    for (size_t q = 0; q < static_cast<size_t>(n) * nb; ++q) z[q] = rng.normal();
    cuda_check(cudaMemcpyAsync(zb_.p, z.data(), sizeof(double) * n * nb, cudaMemcpyHostToDevice,
                               stream_), "upload z");
    solve(1, nb, zb_.p, wb_.p, true);
    const int64_t tot = static_cast<int64_t>(n) * nb;
    const int blocks = static_cast<int>(std::min<int64_t>((tot + 255) / 256, 148 * 8));
    k_permute_scatter<<<blocks, 256, 0, stream_>>>(wb_.p, perm_.p, n, nb, ub_.p);
    k_add_mean<<<blocks, 256, 0, stream_>>>(d_mean, n, nb, ub_.p);
    k_rbmc_spmv<<<blocks, 256, 0, stream_>>>(qcp_d_.p, qri_d_.p, d_qv, d_mean, ub_.p, n, nb, qc_.p);
    k_rbmc_welford<<<gb, 256, 0, stream_>>>(d_mean, ub_.p, qc_.p, qdg_.p, n, nb, s0, rbm_.p,
                                            rbm2_.p);
    cuda_check(cudaStreamSynchronize(stream_), "rbmc batch");
  }
  k_rbmc_final<<<gb, 256, 0, stream_>>>(qdg_.p, rbm2_.p, n, ns, d_var);
  cuda_check(cudaGetLastError(), "rbmc launch");
}

void DeviceFactor::copy_l_panels(std::vector<double>& out) const {
  out.resize(L_.n);
  cuda_check(cudaMemcpyAsync(out.data(), L_.p, L_.n * sizeof(double), cudaMemcpyDeviceToHost, stream_),
             "copy L");
  cuda_check(cudaStreamSynchronize(stream_), "copy L");
}

void DeviceFactor::copy_sig_panels(std::vector<double>& out) const {
  out.resize(sel_inplace_ ? L_.n : Sig_.n);
  cuda_check(cudaMemcpyAsync(out.data(), sig(), out.size() * sizeof(double), cudaMemcpyDeviceToHost,
                             stream_),
             "copy Sigma");
  cuda_check(cudaStreamSynchronize(stream_), "copy Sigma");
}

void bench_fp64(double* dmma_tflops, double* dfma_tflops) {
  int dev = 0, sms = 0;
  cuda_check(cudaGetDevice(&dev), "dev");
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sms");
  DevBuf<double> o;
  o.alloc(1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, threads = 256, blocks = sms * 4;
  k_bench_dmma<<<blocks, threads>>>(o.p, 16);
  cudaEventRecord(e0);
  k_bench_dmma<<<blocks, threads>>>(o.p, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  // each warp-level m8n8k4 = 8*8*4*2 flops; 8 per iteration per warp
  double flops = double(blocks) * (threads / 32) * iters * 8 * 512.0;
  *dmma_tflops = flops / (ms * 1e-3) / 1e12;
  k_bench_dfma<<<blocks, threads>>>(o.p, 16);
  cudaEventRecord(e0);
  k_bench_dfma<<<blocks, threads>>>(o.p, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  flops = double(blocks) * threads * iters * 16 * 2.0;
  *dfma_tflops = flops / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cuda_check(cudaGetLastError(), "bench");
}

}  // namespace gmrf
