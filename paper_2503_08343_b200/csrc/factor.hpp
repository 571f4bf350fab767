// Device-resident supernodal factor: storage, launch plans and the numeric
// factorization / solve / selected-inversion sequences.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "partition.hpp"
#include "profiler.hpp"
#include "solve_tile.hpp"
#include "symbolic.hpp"

namespace gmrf {

void cuda_check(cudaError_t e, const char* what);

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count == n && p) return;
    reset();
    if (count == 0) return;
    // + slack: 16-byte operand copies (load_operand) and the wide GEMM's bulk copies
    // read whole 64- / 128-row tile columns, past the last row of a partial tile at
    // the end of a buffer
    cuda_check(cudaMalloc(&p, count * sizeof(T) + 2048), "cudaMalloc");
    n = count;
  }
  void upload(const std::vector<T>& v, cudaStream_t s) {
    alloc(v.size());
    if (!v.empty())
      cuda_check(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s),
                 "upload");
  }
};

// One message of an exchange point of a partitioned factor (same layout as
// gmrf_msg_t, include/gmrf_b200.h). kind: 0 send, 1 receive, 2 all-reduce sum
// of doubles, 3 all-reduce min of int32.
struct XferMsg {
  int32_t kind;
  int32_t peer;
  int32_t tag;    // child supernode of the cross edge (-1 for all-reduces)
  int32_t phase;  // XPhase, or -1 for all-reduces
  void* dptr;     // device buffer
  int64_t count;  // elements
};
// Completes (or enqueues on `stream`) every message before returning 0.
using ExchangeFn = int (*)(void* ctx, const XferMsg* msgs, int32_t count, void* stream);

struct PartitionSpec {
  int nranks = 1, rank = 0;
  std::vector<i32> owner;  // per supernode; empty: partition_owners(sym, nranks)
  ExchangeFn fn = nullptr;
  void* ctx = nullptr;
};

struct FactorTimes {
  float numeric_ms = 0, solve_ms = 0, selinv_ms = 0;
};

class DeviceFactor {
 public:
  // part: nullptr (or nranks == 1) = the whole factor on this GPU; otherwise
  // this rank's share of a partitioned factor (partition.hpp): storage and
  // kernels for the supernodes it owns, the cross-edge exchanges through
  // part->fn. numeric/solve/selinv keep their semantics: every rank returns
  // the complete status, solution and variances.
  explicit DeviceFactor(std::shared_ptr<const Symbolic> sym, cudaStream_t stream = nullptr,
                        const PartitionSpec* part = nullptr);
  ~DeviceFactor();

  const Symbolic& sym() const { return *sym_; }
  void set_stream(cudaStream_t s) { stream_ = s; }
  cudaStream_t stream() const { return stream_; }

  // Numeric factorization from Q values in the symbolic's CSC order.
  // Returns -1 on success or the ORIGINAL index of the failing pivot.
  int32_t numeric(const double* q, bool q_on_device);
  // Split form for callers that write the panels themselves (fixed-pattern
  // updates, spacetime.cu): begin_numeric zeroes the storage, the caller fills
  // L through d_qmap(), factor_panels runs the levels and returns like numeric.
  void begin_numeric();
  // fwd_rhs (device, original coordinates, one right-hand side): the forward
  // sweep of H x = rhs rides along with the factorization — tree levels without
  // wide supernodes are solved on a side stream of the replayed graph as soon as
  // their panels are final (the top of the tree leaves most SMs idle), the same
  // kernels on the same data as solve(): bit-identical. solve_pending(x) then
  // runs the remaining forward levels, the backward sweep and the permutation.
  int32_t factor_panels(const double* fwd_rhs = nullptr);
  void solve_pending(double* x_dev);
  const int64_t* d_qmap() const { return qmap_.p; }
  // Solves; b/x are n×nrhs column-major (original coordinates for kFull,
  // permuted coordinates for kLower/kUpper, as cholesky.hpp:179-222).
  void solve(int mode, int nrhs, const double* b, double* x, bool on_device);
  // Selected inversion; fills the Σ panels and returns diag(Q⁻¹) in original order.
  void selinv(double* diag_out, bool on_device);
  // Builds the selected-inversion plan and Σ storage ahead of time.
  void prepare_selinv() {
    if (!selinv_plan_) build_selinv_plan();
  }

  // sample_direct (gmrf.hpp:173,182) repeated: out[:, s] = mean + Pᵀ L⁻ᵀ z_s with
  // z_s the s-th normal_vector(n) of Rng(seed) (core/rng.hpp); device pointers,
  // out is n × ns column-major.
  void sample_direct(const double* d_mean, int ns, uint64_t seed, double* d_out);
  // rbmc_variance (gmrf.hpp:213-240): Rao-Blackwellized Monte Carlo marginal
  // variances from ns exact samples; q_values (device) in the symbolic's CSC order.
  void rbmc_variance(const double* d_qvals, const double* d_mean, int ns, uint64_t seed,
                     double* d_var);

  // Host copies (tests / small n).
  void copy_l_panels(std::vector<double>& out) const;
  void copy_sig_panels(std::vector<double>& out) const;

  bool partitioned() const { return part_; }
  int rank() const { return rank_; }
  int nranks() const { return nranks_; }
  const std::vector<i32>& owners() const { return owner_; }

  double* d_l() { return L_.p; }
  double* d_sig() { return sig(); }
  // Σ overwrites L (halves the factor's memory); after selinv the factor is
  // consumed (solves fail until the next numeric factorization). Set before
  // prepare_selinv / the first selinv.
  void set_selinv_inplace(bool on) {
    require(!selinv_plan_ || on == sel_inplace_, kContract, "selinv: in-place mode fixed by its plan");
    sel_inplace_ = on;
  }
  bool selinv_inplace() const { return sel_inplace_; }
  bool factored() const { return factored_; }
  bool has_selinv() const { return selinv_done_; }
  int64_t device_bytes() const;
  int64_t launches_numeric() const { return launches_numeric_; }
  int64_t launches_solve() const { return launches_solve_; }
  int64_t launches_selinv() const { return launches_selinv_; }
  // Per-kernel-class timing (off unless enabled); callers may share one profiler.
  void set_profiler(KernelProfiler* p) { prof_ = p ? p : &own_prof_; }
  KernelProfiler& profiler() { return *prof_; }

 private:
  void build_factor_plan();
  void build_selinv_plan();
  void ensure_solve_ws(int nrhs);
  template <int NR>
  void launch_solve_levels(bool fwd, bool bwd, double* y, int nr, int fwd_from = 0);
  SymDev symdev() const;
  SymDev symdev_sel() const;  // same, with the selected inversion's U offsets
  void plan_update_storage();
  bool mine(int k) const { return !part_ || owner_[k] == rank_; }
  void exchange(const std::vector<XferMsg>& m);
  void enqueue_levels(cudaStream_t sa, cudaStream_t sb, bool la, bool in_graph, bool fuse_fwd = false);
  template <int NR>
  void fwd_level(int l, double* y, int nr, cudaStream_t st);
  void exchange_solve(int phase, int level, int nr, double* y);

  std::shared_ptr<const Symbolic> sym_;
  cudaStream_t stream_;
  // partition (single GPU: part_ false, every supernode mine)
  bool part_ = false;
  int nranks_ = 1, rank_ = 0;
  std::vector<i32> owner_;
  ExchangeFn xfn_ = nullptr;
  void* xctx_ = nullptr;
  std::vector<XEdge> sched_;              // this rank's cross-edge messages
  std::vector<i64> lptr_h_, uptr_h_, uvptr_h_;  // this rank's storage offsets
  std::vector<i64> uptrs_h_;                    // U offsets during the selected inversion
  i64 u_arena_ = 0, u_arena_f_ = 0, u_arena_s_ = 0;
  bool u_static_ = false;                       // GMRF_U_STATIC=1: Σ r² layout (A/B)
  std::vector<std::vector<XferMsg>> fx_;  // factor messages after each chunk level
  std::vector<std::vector<XferMsg>> sx_;  // selinv messages after each chunk level
  struct BxPoint {
    int64_t pk0, pkn, up0, upn;  // pack / unpack tasks in xt_
  };
  std::vector<BxPoint> bx_;       // backward-solve exchange per supernode level
  std::vector<int64_t> bx_off_;   // pack-buffer offset of each bsolve edge in sched_ order
  DevBuf<RowXfer> xt_;
  DevBuf<double> xb_;             // backward-solve pack buffer (Σ r_c × kMaxRhs)
  DevBuf<char> colmine_;          // per internal column: owned by this rank
  // sampling / RBMC workspaces (pattern of Q for the SpMV, sample batches)
  DevBuf<int64_t> qcp_d_;
  DevBuf<int32_t> qri_d_;
  DevBuf<double> zb_, wb_, ub_, qc_, rbm_, rbm2_, qdg_;
  bool factored_ = false, selinv_done_ = false;

  DevBuf<int32_t> first_, rows_, relmap_, chptr_, chlist_, perm_, col2sn_, snparent_, status_;
  DevBuf<int64_t> rptr_, lptr_, uptr_, uptrs_, qmap_, pptr_, uvptr_;
  DevBuf<double> L_, U_, Sig_, q_, P_, Uv_, v1_, v2_, diag_, rdiag_;
  DevBuf<double> ystage_;      // selected inversion: per-level Y / W staging
  bool sel_inplace_ = false;
  double* sig() const { return sel_inplace_ ? L_.p : Sig_.p; }
  DevBuf<SolveTile> tiles_;
  DevBuf<double> pf_;       // forward column-block partials (solve.cuh)
  DevBuf<unsigned> pfctr_;  // their arrival counters
  std::vector<int64_t> tile_ptr_;
  int maxw_ = 1;
  int64_t uv_total_ = 0, p_total_ = 0;
  int ws_nrhs_ = 0;

  static constexpr int kSmBuckets = 6;
  struct FLevel {
    int64_t ea0, ean, po0, pon, pan0, pann, gm0, gmn;
    double ea_bytes, po_flops, tr_flops, gm_flops;  // algorithmic work per launch
    int64_t pb0[3], pbn[3];  // panel tasks split by width bucket 16 / 32 / 64
    int64_t rd0, rdn;        // split-K reductions of the level's GEMM tiles
    int64_t sm0[kSmBuckets], smn[kSmBuckets];  // small fronts (build_factor_plan), one CTA each
    double sm_flops;
    int64_t gr0, grn, rr0, rrn;  // rest of the trailing update + U SYRK (second stream)
    double gr_flops;
    int64_t pd0[3], pdn[3], pt0[3], ptn[3];  // two-phase panel: diagonal / TRSM tasks
    int64_t gu0, gun;  // incremental U updates of wide supernodes (third stream)
    double gu_flops;
    bool prow[3];  // panel kernel per bucket: row sweep (one wave) or blocked; decided on
                   // the level's task count over ALL supernodes, so a partitioned factor
                   // runs the same kernels (same rounding) as the single-GPU one
    int64_t eau0, eaun;  // extend-add tasks of update-block columns (bulk stream)
    int dwait;           // the chain's next-block update waits for the bulk stream's level l - dwait
    bool gm32;           // the next-block update runs on 32×32 tiles (k_gemm_next)
    int64_t gw0, gwn;    // 128×128 tiles (k_gemm_wide) of the level's large U SYRKs / flushes (bulk stream)
  };
  DevBuf<int32_t> small_;
  std::vector<FLevel> flev_;
  DevBuf<EaTask> ea_;
  DevBuf<int2> eap_;
  DevBuf<PanelTask> pan_, po_;
  DevBuf<GemmTask> gemm_;

  struct SLevel {
    int64_t ga0, gan, y0, yn, t0, tn, z0, zn, d0, dn;
    int64_t gg0, ggn;  // ghost gathers: Σ_RR of other ranks' children of this level's supernodes
    double ga_bytes, y_flops, t_flops, z_flops, d_flops;
    int64_t yr0, yrn, zr0, zrn;  // split-K reductions of the Y and Z tiles
    int64_t tb0[3], tbn[3], db0[3], dbn[3];  // TRSM / diag chunks by width bucket 16/32/64
    int64_t mi0, min_;                       // Σ_{P,J} → Σ_{J,P} mirror tiles
    // blocked selected inversion of the level's multi-chunk supernodes
    // (selinv.cuh): launches in order; kind 0 = GEMM tiles of sgemm_ (+ split-K
    // reductions of sred_), 1 = diagonal-block inverses, 2 = Σ_JJ mirror tiles (sblk_)
    struct BStage {
      int kind;
      int64_t t0, tn, r0, rn;
      double flops;
    };
    std::vector<BStage> bst;
  };
  DevBuf<ReduceTask> red_, sred_;
  DevBuf<double> parts_, rparts_, sparts_;  // split-K partial tiles
  // lookahead: the rest-of-update GEMMs run on aux_ (events order the levels)
  cudaStream_t main_ = nullptr, aux_ = nullptr, uu_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr;
  std::vector<cudaEvent_t> ev_panel_, ev_rest_, ev_uupd_, ev_eau_;
  // supernodes of at least inc_u_ chunks accumulate their update matrix chunk by
  // chunk (U -= L21(c) L21(c)ᵀ right after chunk c's panel, on uu_) instead of
  // one K = w SYRK after the last chunk on the critical path; 0 disables
  int inc_u_ = 0;
  // k_gemm_wide for bulk GEMMs with at least wide_min_r_ rows and K >= wide_min_k_ (0 disables)
  int wide_min_r_ = 2048, wide_min_k_ = 512;
  bool use_wide(int r, int K) const { return wide_min_k_ > 0 && r >= wide_min_r_ && K >= wide_min_k_; }
  int64_t next_max_tiles_ = 222;   // ... on levels with at most this many 64×64 next-block tiles (over all ranks)
  bool gemm_next_ = true;          // k_gemm_next for the chain GEMMs of one-wave levels (GMRF_GEMM_NEXT=0: A/B)
  bool ea_split_ = true;           // update-block extend-add on the bulk stream (GMRF_EA_SPLIT=0: A/B)
  int inc_b_ = 2;                  // chunks per incremental batch (K = inc_b_·kNB per pass over U)
  int64_t ea_cta_max_ = 4096;      // extend-add: one CTA per column on levels with at most this many columns
  unsigned rows_max_ctas_ = 148;   // row-sweep panel on levels with at most this many slabs (one wave)
  // GMRF_TRACE=<file>: per-level timeline markers (k_mark), appended per factorization
  static constexpr int kTraceSlots = 10;
  std::string trace_file_;
  DevBuf<unsigned long long> tbuf_;
  void dump_trace();
  bool lookahead_ = true;
  int defer_ = 4;
  bool gemm_cap_ = true;  // cap bulk GEMM residency on one-wave levels (launch_gemm)  // trailing-update deferral depth (chunks per flush), trailing_jobs
  template <class F>
  void trailing_jobs(int w, int rows, int c, F&& emit) const;
  // deferral depth of a supernode: fronts whose panel exceeds defer_min_ entries
  // (their K = kNB trailing passes are HBM-bound) flush every defer_ chunks
  int64_t defer_min_ = 8ll << 20;
  int defer_of(int w, int rows) const {
    return static_cast<int64_t>(w) * rows >= defer_min_ ? defer_ : 1;
  }
  bool use_graph_ = true;             // GMRF_NO_GRAPH=1 disables (A/B)
  bool panel2_ = true;                // GMRF_PANEL1=1: fused one-phase panel kernels (A/B)
  DevBuf<PanelTask> pd_, pt_;         // two-phase panel tasks
  DevBuf<double> stage_;              // per-level L11 staging slots (panel2.cuh)
  cudaGraphExec_t fgraph_ = nullptr;  // captured chunk-level sequence
  // fused forward sweep (factor_panels(fwd_rhs)): a second captured sequence with
  // the forward-solve launches of tree levels [0, fuse_levels_) on sf_
  cudaGraphExec_t fgraph_fs_ = nullptr;
  int64_t graph_fs_launches_ = 0;
  cudaStream_t sf_ = nullptr;
  cudaEvent_t ev_fs_ = nullptr;
  bool fuse_fwd_ = true;            // GMRF_FUSE_FWD=0 disables (A/B)
  bool fuse_late_ = false;          // GMRF_FUSE_LATE=1: hold the fused sweep back until the one-wave chain (A/B: slower)
  int fuse_levels_ = 0;             // tree levels below the first one with a wide supernode
  std::vector<int> fs_ready_;       // chunk level whose panel step completes tree levels <= l
  DevBuf<PanelTask> pof_;           // chunks by tree level (per-level diagonal write-back)
  std::vector<int64_t> pof_ptr_;
  int fwd_done_ = 0;                // forward levels already solved for the pending rhs
  bool rhs_pending_ = false;
  int64_t graph_launches_ = 0;
  std::vector<double> lvl_bytes_;  // solve: L panel + row-index bytes per tree level
  KernelProfiler own_prof_;
  KernelProfiler* prof_ = &own_prof_;
  std::vector<SLevel> slev_;
  DevBuf<ColTask> sga_;
  DevBuf<GemmTask> sgemm_;
  DevBuf<SelChunk> strsm_, sdiag_, smir_, sblk_;
  // blocked selected inversion (W = L_JJ⁻¹ by recursive doubling + four GEMM
  // stages instead of the chunk chain): multi-chunk supernodes while their
  // level's staging stays under sel_block_stage_ doubles, single-chunk ones of at
  // least sel_block_min_w_ columns (their register-resident TRSM / diagonal
  // kernels run at 1-3 TFLOP/s; config 4: 21.4 -> 19.0 ms per selected inversion
  // at 16; 48: 19.8, 32: 19.1, 1: 19.2). selinv_blocked (partition.hpp) decides,
  // partition_memory models the same rule; GMRF_SEL_BLOCK=0 disables (A/B).
  long long sel_block_stage_ = kSelBlockLevelStage;
  int sel_block_min_w_ = 16;
  std::vector<char> sel_blk_;
  bool selinv_plan_ = false;

  std::vector<int64_t> lvl_ptr_;
  DevBuf<int32_t> lvl_sn_;
  // wide supernodes (solve_wide.cuh): per level, the first lvl_nrm_[l] entries
  // of the level's lvl_sn_ range are narrow, the rest wide; their 64-row blocks
  // form cooperative launch groups wgroups_[wl_ptr_[l] .. wl_ptr_[l+1])
 public:
  struct WideGroup {
    int64_t t0, nt;  // tasks [t0, t0+nt) of wfwd_ / wbwd_
  };

 private:
  std::vector<int64_t> lvl_nrm_, lvl_nsm_, wl_ptr_;
  std::vector<WideGroup> wgroups_;
  DevBuf<WideBlock> wfwd_, wbwd_;
  DevBuf<double> wx_;  // wide-solve block exchange: solved 64-row blocks, sentinel until written
  // inverted 64×64 diagonal blocks of the wide supernodes (k_tri_inv64 after every
  // factorization): a wide-block step ends with a 64×64 GEMV on all 256 threads
  // instead of a 64-step dependent warp substitution. GMRF_WIDE_INV=0: substitution (A/B)
  bool wide_inv_ = true;
  DevBuf<double> winv_;
  DevBuf<SelChunk> winv_tasks_;
  int64_t wide_blocks_ = 0;

  int64_t launches_numeric_ = 0, launches_solve_ = 0, launches_selinv_ = 0;
};

// FP64 issue-rate microbenchmarks (TFLOP/s), for the roofline denominator.
void bench_fp64(double* dmma_tflops, double* dfma_tflops);

}  // namespace gmrf
