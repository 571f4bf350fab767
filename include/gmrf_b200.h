/*
 * gmrf_b200 — C-ABI of the B200-native sparse-precision GMRF engine.
 *
 * The drop-in boundary for the reference's hot path. The reference has no FFI
 * (SURVEY §8(b)): its API is the header-only C++ in
 * /root/reference/proj/include/gmrfpde/**. Each entry point below states the
 * reference function it replaces (file:line under that directory); the C++
 * shim in paper_2503_08343_b200/include/gmrfpde_b200/ re-exposes them with the
 * reference signatures, and INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - CSC with int64 column pointers (the reference's int32 nnz counter
 *    overflows at config 5), int32 row indices sorted ascending,
 *    double values. Matrices passed to the factorization are full symmetric
 *    (both triangles), as the reference's SparseMatrixCSC Q.
 *  - Permutations are new -> old (reference cholesky.hpp:17).
 *  - Every function returns GMRF_OK (0) or a status; gmrf_last_error() gives
 *    the message (thread-local). There is no CPU fallback: without a CUDA
 *    device the numeric entry points fail with GMRF_ERR_CUDA.
 *  - *_device variants take device pointers and enqueue on the factor's
 *    stream (gmrf_factor_set_stream); host variants synchronize.
 */
#ifndef GMRF_B200_H
#define GMRF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GMRF_OK = 0,
  GMRF_ERR_NOT_SPD = 1,    /* NotPositiveDefiniteError, core/types.hpp:40-48 */
  GMRF_ERR_DIMENSION = 2,  /* DimensionError, core/types.hpp:21-24 */
  GMRF_ERR_STRUCTURAL = 3, /* StructuralError, core/types.hpp:16-19 */
  GMRF_ERR_CONTRACT = 4,   /* ContractError, core/types.hpp:27-30 */
  GMRF_ERR_CUDA = 5,       /* device failure */
  GMRF_ERR_NUMERICAL = 6   /* NumericalError, core/types.hpp:33-36 */
};

enum { GMRF_SOLVE_LOWER = 0, GMRF_SOLVE_UPPER = 1, GMRF_SOLVE_FULL = 2 }; /* cholesky.hpp:174 */

typedef struct gmrf_symbolic gmrf_symbolic_t;
typedef struct gmrf_factor gmrf_factor_t;

typedef struct {
  int32_t n;
  int64_t nnz_q;
  int64_t nnz_l;          /* exact, = reference SymbolicFactor::nnz_L */
  int64_t nnz_l_padded;   /* supernodal storage after relaxed amalgamation */
  int64_t update_entries; /* Σ r_s² (multifrontal update matrices) */
  int32_t n_supernodes;
  int32_t n_levels;       /* supernodal tree height */
  int32_t etree_height;   /* column elimination tree height */
  int32_t max_front;      /* max rows of a supernode */
  double flops_ref;       /* Σ_j c_j², BASELINE.md §3 factorization numerator */
  double flops_sn;        /* padded supernodal Σ c² actually executed */
} gmrf_symbolic_info_t;

typedef struct {
  int64_t device_bytes;
  int64_t launches_numeric; /* kernels launched by the last numeric factorization */
  int64_t launches_solve;   /* ... by the last solve */
  int64_t launches_selinv;  /* ... by the last selected inversion */
} gmrf_factor_stats_t;

const char* gmrf_last_error(void);
int gmrf_version(void);

/* Fill-reducing nested-dissection ordering (METIS NodeND), new -> old.
 * Replaces amd_order (core/amd.hpp:294) as the default ordering. */
int gmrf_nd_order(int32_t n, const int64_t* col_ptr, const int32_t* row_idx, int32_t* perm);

/* symbolic_analyze (core/cholesky.hpp:68). perm == NULL selects the ND
 * ordering (postordered), as cholesky_factor(q) selects AMD (cholesky.hpp:170). */
int gmrf_symbolic_analyze(int32_t n, const int64_t* col_ptr, const int32_t* row_idx,
                          const int32_t* perm, gmrf_symbolic_t** out);
int gmrf_symbolic_info(const gmrf_symbolic_t* s, gmrf_symbolic_info_t* info);
/* SymbolicFactor fields (cholesky.hpp:16-23): perm[n], parent[n], col_ptr_l[n+1];
 * any pointer may be NULL. */
int gmrf_symbolic_export(const gmrf_symbolic_t* s, int32_t* perm, int32_t* parent,
                         int64_t* col_ptr_l);
void gmrf_symbolic_free(gmrf_symbolic_t* s);
/* Supernode partition (after relaxed amalgamation): first column [ns+1],
 * front rows [ns], tree level [ns], parent supernode [ns] (-1 root). */
int gmrf_symbolic_supernodes(const gmrf_symbolic_t* s, int32_t* first, int32_t* rows,
                             int32_t* level, int32_t* parent);

/* Device storage for a factor of the symbolic's pattern. */
int gmrf_factor_create(const gmrf_symbolic_t* s, gmrf_factor_t** out);
int gmrf_factor_set_stream(gmrf_factor_t* f, void* cuda_stream);
/* cholesky_refactor (core/cholesky.hpp:113): values in the symbolic's CSC
 * order. On GMRF_ERR_NOT_SPD, *bad_index = ORIGINAL index of the failing
 * pivot (cholesky.hpp:153-156); else -1. */
int gmrf_factor_numeric(gmrf_factor_t* f, const double* q_values, int32_t* bad_index);
int gmrf_factor_numeric_device(gmrf_factor_t* f, const double* d_q_values, int32_t* bad_index);

/* solve_triangular / solve (core/cholesky.hpp:179,225) for nrhs right-hand
 * sides (n × nrhs column-major). LOWER/UPPER work in permuted coordinates,
 * FULL in original coordinates. sample_direct (gmrf.hpp:173) = UPPER + Pᵀ. */
int gmrf_solve(gmrf_factor_t* f, int mode, int32_t nrhs, const double* b, double* x);
int gmrf_solve_device(gmrf_factor_t* f, int mode, int32_t nrhs, const double* d_b, double* d_x);

/* Selected inversion in place (on = 1): Σ overwrites L chunk by chunk, halving
 * the factor's device memory; the factor is consumed (solves, samples and a
 * second selected inversion fail with GMRF_ERR_CONTRACT until the next
 * numeric factorization). Default 0 for generic factors; the pipelines
 * (gmrf_spacetime_*, gmrf_regression_*) use it — variances are their last step.
 * Set before the first selected inversion of the factor. */
int gmrf_factor_set_selinv_inplace(gmrf_factor_t* f, int32_t on);
/* takahashi_diagonal (core/takahashi.hpp:67): diag(Q⁻¹) in original order. */
int gmrf_selinv_diag(gmrf_factor_t* f, double* diag);
int gmrf_selinv_diag_device(gmrf_factor_t* f, double* d_diag);
/* sample_direct (gmrf.hpp:173,182) repeated n_samples times with one
 * Rng(seed) stream (core/rng.hpp, same draws as the reference):
 * out[:, s] = mean + Pᵀ L⁻ᵀ z_s (n × n_samples column-major, host). Batched
 * multi-right-hand-side upper solves on the device. */
int gmrf_sample_direct(gmrf_factor_t* f, const double* mean, int32_t n_samples, uint64_t seed,
                       double* out);
/* rbmc_variance (gmrf.hpp:213-240): Rao-Blackwellized Monte Carlo marginal
 * variances of N(mean, Q⁻¹) from n_samples exact samples of Rng(seed).
 * q_values: Q (the factored matrix) in the symbolic's CSC order. Errors:
 * GMRF_ERR_CONTRACT if n_samples < 2, GMRF_ERR_NUMERICAL for a non-positive
 * Q_ii (as the reference). */
int gmrf_rbmc_variance(gmrf_factor_t* f, const double* q_values, const double* mean,
                       int32_t n_samples, uint64_t seed, double* var);

/* takahashi_selected_inverse (core/takahashi.hpp:19): Σ on the pattern of
 * L+Lᵀ mapped back to original indices (sorted CSC). Call after selinv_diag.
 * nnz query first (host memory, small n). */
int gmrf_selinv_pattern_nnz(gmrf_factor_t* f, int64_t* nnz);
int gmrf_selinv_pattern(gmrf_factor_t* f, int64_t* col_ptr, int32_t* row_idx, double* values);

/* CholeskyFactor::L in the reference layout (cholesky.hpp:92-109): exact
 * pattern col_ptr[n+1] (== symbolic col_ptr_l), rows ascending with the
 * diagonal first, and perm[n]. Host copy, for tests / small n. */
int gmrf_factor_l(gmrf_factor_t* f, int64_t* col_ptr, int32_t* row_idx, double* values,
                  int32_t* perm);
int gmrf_factor_stats(const gmrf_factor_t* f, gmrf_factor_stats_t* st);
void gmrf_factor_free(gmrf_factor_t* f);

/* ---- Conjugate gradients (core/cg.hpp:39-105) and CG sampling --------------
 * Matrix-free alternative to the factorization (gmrf.hpp:188-202). Same
 * recurrence, stopping rule ‖r‖ ≤ max(rtol‖b‖, atol) and breakdown error as
 * the reference; reductions are deterministic device trees. */
typedef struct {
  double rtol;             /* CGConfig::rtol (> 0) */
  double atol;
  int64_t max_iter;        /* 0: 10·n */
  int32_t preconditioner;  /* 0 kNone, 1 kJacobi (diag of Q) */
} gmrf_cg_config_t;
typedef struct {
  int64_t iterations;
  double final_residual;
  int32_t converged;
} gmrf_cg_result_t; /* CGResult (cg.hpp:29-34) */
/* cg_solve(q, b, x0, cfg) (cg.hpp:98): Q full CSC n × n; x0 may be NULL. */
int gmrf_cg_solve(int32_t n, const int64_t* col_ptr, const int32_t* row_idx, const double* values,
                  const double* b, const double* x0, const gmrf_cg_config_t* cfg, double* x,
                  gmrf_cg_result_t* res);
/* sample_cg (gmrf.hpp:188): out = mean + Q⁻¹ S z, S the n × m square root (CSC);
 * GMRF_ERR_NUMERICAL if CG does not converge. */
int gmrf_sample_cg(int32_t n, const int64_t* q_col_ptr, const int32_t* q_row_idx,
                   const double* q_values, int32_t m, const int64_t* s_col_ptr,
                   const int32_t* s_row_idx, const double* s_values, const double* mean,
                   const double* z, const gmrf_cg_config_t* cfg, double* out);

/* ---- Partitioned factorization across ranks (multi-GPU) -----
 * No reference analogue (the reference is single-threaded):
 * the supernodal tree is split along its top nested-dissection separators
 * (subtree-to-subcube: whole subtrees per rank, each separator on the lowest
 * rank of the range below it). A partitioned handle behaves like a
 * gmrf_factor_t — gmrf_factor_numeric*, gmrf_solve*, gmrf_selinv_diag* keep
 * their semantics and return complete results on every rank — but stores
 * and factors only its own supernodes. Cross-rank data (Schur complements
 * child → parent in the factorization, update vectors in the forward solve,
 * x rows parent → child in the backward solve, Σ blocks parent → child in
 * the selected inversion) moves through a caller-supplied exchange function,
 * e.g. torch.distributed over NCCL (paper_2503_08343_b200/partition.py). */
enum { GMRF_MSG_SEND = 0, GMRF_MSG_RECV = 1, GMRF_MSG_ALLREDUCE_SUM_F64 = 2,
       GMRF_MSG_ALLREDUCE_MIN_I32 = 3 };
enum { GMRF_PHASE_FACTOR = 0, GMRF_PHASE_FSOLVE = 1, GMRF_PHASE_BSOLVE = 2,
       GMRF_PHASE_SELINV = 3 };

typedef struct {
  int32_t kind;   /* GMRF_MSG_* */
  int32_t peer;   /* other rank (send / recv), -1 for all-reduces */
  int32_t tag;    /* child supernode of the cross edge, -1 for all-reduces */
  int32_t phase;  /* GMRF_PHASE_*, -1 for all-reduces */
  void* dptr;     /* device buffer */
  int64_t count;  /* elements (double, or int32 for ALLREDUCE_MIN_I32) */
} gmrf_msg_t;

/* Called at every exchange point with this rank's messages of that point, in
 * the same order on both sides of each pair. It must complete the messages, or
 * enqueue them on `cuda_stream` so that later work on that stream sees them,
 * and return 0. All-reduces are called on every rank. */
typedef int (*gmrf_exchange_fn)(void* ctx, const gmrf_msg_t* msgs, int32_t count,
                                void* cuda_stream);

/* Native NCCL transport (csrc/nccl_exchange.cpp): gmrf_nccl_exchange() is a
 * gmrf_exchange_fn that posts the messages on the factor's stream with
 * ncclSend / ncclRecv (one group per exchange point) and ncclAllReduce; pass it
 * with ctx = the communicator from gmrf_nccl_comm_create. Rank 0 obtains the
 * 128-byte unique id (gmrf_nccl_unique_id) and hands it to the other ranks by
 * any means (torch.distributed broadcast, MPI, a file); every rank then calls
 * gmrf_nccl_comm_create with the GPU it will use already current. NCCL is
 * loaded at run time (the process's libnccl.so.2, or $GMRF_NCCL_LIB). */
int gmrf_nccl_unique_id(uint8_t* id128);
int gmrf_nccl_comm_create(int32_t nranks, int32_t rank, const uint8_t* id128, void** comm);
void gmrf_nccl_comm_destroy(void* comm);
gmrf_exchange_fn gmrf_nccl_exchange(void);
const char* gmrf_nccl_last_error(void);

/* Owner rank of each supernode (ns entries) for nranks ranks. Host only. */
int gmrf_partition_owners(const gmrf_symbolic_t* s, int32_t nranks, int32_t* owner);
/* The full cross-edge message schedule for an owner map (host only, tests):
 * rows of 6 int64 (phase, point, src, dst, child supernode, count [per RHS
 * for the solve phases]). Call with rows == NULL for the count. */
int gmrf_partition_schedule(const gmrf_symbolic_t* s, const int32_t* owner, int64_t* rows,
                            int64_t* n_rows);
/* Per-rank device memory plan (bytes) of a partitioned factorization with
 * selected inversion, from the symbolic alone (host only): rows of 7 values
 * per rank — L panels, Σ panels, update-matrix arena (factorization), the same
 * arena in the selected inversion, replicated pattern-sized data, total, owned
 * supernodes. owner == NULL: gmrf_partition_owners. */
int gmrf_partition_memory(const gmrf_symbolic_t* s, int32_t nranks, const int32_t* owner,
                          int64_t* rows);
/* This rank's share of the factor. owner == NULL: gmrf_partition_owners. */
int gmrf_factor_create_partitioned(const gmrf_symbolic_t* s, int32_t nranks, int32_t rank,
                                   const int32_t* owner, gmrf_exchange_fn fn, void* ctx,
                                   gmrf_factor_t** out);

/* Rng (core/rng.hpp:14-47): n draws of Rng(seed).uniform() (kind 0) or
 * .normal() (kind 1, Box-Muller with the cached spare), host only — the
 * reference's seeded synthetic inputs without the reference. */
int gmrf_rng_fill(uint64_t seed, int32_t kind, int64_t n, double* out);
/* One Rng(seed) stream: n_uniform uniform() draws, then n_normal normal() draws,
 * into out[n_uniform + n_normal] — SURVEY §8(d)'s pinned draw order (e.g. C1:
 * 100 observation coordinates, then 100 noises). */
int gmrf_rng_draw(uint64_t seed, int64_t n_uniform, int64_t n_normal, double* out);

/* FP64 issue-rate microbenchmark (TFLOP/s) of DMMA m8n8k4 and DFMA. */
int gmrf_bench_fp64(double* dmma_tflops, double* dfma_tflops);

/* ---- Fixed-pattern conditioning update (north_star rows 1-2) ---------------
 * H = symmetrize(base + c · Aᵀ diag(w) A) on the symbolic's pattern: the
 * reference's condition_affine update (gmrf.hpp:150-155, A = observation
 * operator, w = Λ), its Gauss-Newton matrix (gauss_newton.hpp:137-138, A = J_k,
 * w = Λ_pde, base = q_eff) and Laplace precision (:231-232), and the Matérn
 * precision (priors/matern.hpp:70-80, A = K, w = 1/m̃, c = 1/τ², no base).
 * The plan (a product map: for each pattern entry, the pairs of A entries
 * sharing a row) is built once per A pattern; updates stream values only and
 * write the factor's panels directly — no permute, sort or triplet pass per
 * refactorization (cholesky.hpp:117). Same per-entry summation order as the
 * reference's SpGEMM + symmetrize. A: m × n CSR, columns ascending per row;
 * every product A_kR A_kC must fall in the pattern (GMRF_ERR_STRUCTURAL). */
typedef struct gmrf_gram gmrf_gram_t;
int gmrf_gram_create(const gmrf_symbolic_t* s, int32_t m, const int64_t* a_row_ptr,
                     const int32_t* a_col_idx, gmrf_gram_t** out);
void gmrf_gram_free(gmrf_gram_t* g);
/* Assembled values on the symbolic's CSC pattern (host in/out): out[nnz_q];
 * base (nnz_q, may be NULL = 0), a_values (A's nnz, CSR order), w (m, NULL = 1). */
int gmrf_gram_apply(gmrf_gram_t* g, const double* base, const double* a_values, const double* w,
                    double c, double* out);
/* gmrf_update_fixed_pattern: writes H straight into f's panels and factors it
 * (cholesky_refactor of H). bad_index as gmrf_factor_numeric. Host arrays /
 * device arrays (enqueued on the factor's stream). */
int gmrf_factor_update_fixed_pattern(gmrf_factor_t* f, gmrf_gram_t* g, const double* base,
                                     const double* a_values, const double* w, double c,
                                     int32_t* bad_index);
int gmrf_factor_update_fixed_pattern_device(gmrf_factor_t* f, gmrf_gram_t* g, const double* d_base,
                                            const double* d_a_values, const double* d_w, double c,
                                            int32_t* bad_index);

/* Update system: H = symmetrize(B + Aᵀ diag(w) A) on the fixed union pattern
 * and its device factor, B = Q (base_kind 0: b_* is Q, n × n CSC with values)
 * or B = symmetrize(S Sᵀ) (base_kind 1: b_* is S, n × b_cols CSC). A: m × n CSC
 * pattern; its values (same CSC order) and w arrive per refactor. perm: the
 * factor's ordering (new -> old), NULL for nested dissection. One object per
 * update site of the reference: condition_affine (gmrf.hpp:150-161),
 * gauss_newton (gauss_newton.hpp:110-141), laplace_posterior (:228-232) —
 * the drop-in headers under paper_2503_08343_b200/include use it. */
typedef struct gmrf_update_system gmrf_update_system_t;
int gmrf_update_system_create(int32_t n, int32_t base_kind, int32_t b_cols, const int64_t* b_col_ptr,
                              const int32_t* b_row_idx, const double* b_values, int32_t m,
                              const int64_t* a_col_ptr, const int32_t* a_row_idx,
                              const int32_t* perm, gmrf_update_system_t** out);
/* 1 if (m, A's CSC pattern) is the one the system was built for, else 0. */
int gmrf_update_system_same_operator(const gmrf_update_system_t* h, int32_t m,
                                     const int64_t* a_col_ptr, const int32_t* a_row_idx);
/* H from A's values and w, factorized; GMRF_ERR_NOT_SPD with *bad_index as
 * gmrf_factor_numeric. */
int gmrf_update_system_refactor(gmrf_update_system_t* h, const double* a_values, const double* w,
                                int32_t* bad_index);
/* refactor followed by the solve H x = b (host vectors of n values): the step
 * gauss_newton takes every iteration (gauss_newton.hpp:137-141). The forward
 * sweep rides along with the factorization on the device; same results as
 * gmrf_update_system_refactor + gmrf_solve(GMRF_SOLVE_FULL). */
int gmrf_update_system_refactor_solve(gmrf_update_system_t* h, const double* a_values,
                                      const double* w, const double* b, double* x,
                                      int32_t* bad_index);
/* H's values only (no factorization), into values[nnz] in the union pattern's
 * order: symmetrize(B + c · Aᵀ diag(w) A) — e.g. the Matérn precision with
 * B = 0, A = K̂, w = 1/m̃, c = 1/τ² (priors/matern.hpp:70-80). */
int gmrf_update_system_assemble(gmrf_update_system_t* h, const double* a_values, const double* w,
                                double c, double* values);
/* The union pattern (col_ptr[n+1]; row_idx == NULL queries) and H's values of
 * the last refactor / assemble (values may be NULL). */
int gmrf_update_system_matrix(const gmrf_update_system_t* h, int64_t* col_ptr, int32_t* row_idx,
                              double* values);
/* Borrowed views, valid while the system lives: its symbolic and its factor
 * (for gmrf_solve*, gmrf_selinv_*, gmrf_sample_direct, gmrf_factor_l); NULL
 * before the first refactor (the symbolic analysis and factor storage are
 * created on first use; assemble needs neither). */
const gmrf_symbolic_t* gmrf_update_system_symbolic(const gmrf_update_system_t* h);
gmrf_factor_t* gmrf_update_system_factor(gmrf_update_system_t* h);
void gmrf_update_system_free(gmrf_update_system_t* h);

/* ---- Matérn SPDE regression posterior (configs 1-2) -------------------------
 * P1 FEM on an interval (dim 1: n_el elements over [xa, xb],
 * build_interval_mesh, fem/mesh.hpp:63) or the unit square (dim 2: n_el × n_el
 * cells split along the diagonal, build_unit_square_mesh, mesh.hpp:142). */
typedef struct {
  int32_t dim;
  int32_t n_el;
  double xa, xb;
  double kappa; /* MaternSpec {κ, α, τ} (priors/matern.hpp) */
  int32_t alpha;
  double tau;
} gmrf_matern_config_t;

/* point_observation_operator / eval_basis (solver/info_operator.hpp:108-123,
 * fem/space.hpp:67-109,376-394): A (m × n) with the P1 shape values of the
 * element containing each point; CSR, 2 (1-D) or 3 (2-D) entries per row.
 * Host only. Call with col_idx == NULL for the nnz (row_ptr[m] filled). */
int gmrf_point_operator(const gmrf_matern_config_t* mesh, int32_t m, const double* points,
                        int64_t* row_ptr, int32_t* col_idx, double* values);
/* P1 element assembly on the device (fem_device.cu), one thread per matrix
 * column, element contributions summed in the reference's triplet order:
 *   which 0: assemble_mass (fem/assembly.hpp:81-101), M_ij = ∫ φ_i φ_j;
 *   which 1: assemble_stiffness (assembly.hpp:104-161): dim 1 — diffusion ·
 *            ∫φ'_i φ'_j + advection · ∫φ_i φ'_j + reaction · ∫φ_i φ_j; dim 2 —
 *            diffusion · ∫∇φ_i·∇φ_j (laplace_operator, assembly.hpp:48).
 * The mesh is cfg's (kappa/alpha/tau unused). Full CSC out: call with
 * row_idx == NULL to get col_ptr[n+1], then again for row_idx / values.
 * lumped (may be NULL, n values, which 0 only): lumped_mass_vector row sums
 * (assembly.hpp:241-262). dirichlet != 0 (dim 1): the matrix with both end
 * nodes constrained, fold_and_mask with T = I (fem/constraints.hpp:111-128):
 * their rows/columns removed and `constrained_diag` on their diagonal
 * (apply_constraints_precision_pair :158-173 uses 1 for K and ε² for M).
 * gmrf_fem_assemble_host evaluates the same formulas in host loops (no device):
 * the two agree bit for bit. */
int gmrf_fem_assemble(const gmrf_matern_config_t* cfg, int32_t which, double diffusion,
                      double advection, double reaction, int32_t dirichlet,
                      double constrained_diag, int32_t* n, int64_t* col_ptr, int32_t* row_idx,
                      double* values, double* lumped);
int gmrf_fem_assemble_host(const gmrf_matern_config_t* cfg, int32_t which, double diffusion,
                           double advection, double reaction, int32_t dirichlet,
                           double constrained_diag, int32_t* n, int64_t* col_ptr,
                           int32_t* row_idx, double* values, double* lumped);

/* matern_prior (priors/matern.hpp:53-80): the prior precision Q assembled on
 * the device (fixed-pattern Gram product of K = K_Δ + κ²M with the lumped mass),
 * full symmetric CSC. col_ptr[n+1] first (row_idx == NULL), then the rest. */
int gmrf_matern_prior(const gmrf_matern_config_t* cfg, int32_t* n, int64_t* col_ptr,
                      int32_t* row_idx, double* values);

/* Posterior of the Matérn prior conditioned on m point observations
 * (condition_on(matern_prior, point_observation_operator), gmrf.hpp:145-170):
 * Q assembly, Q + AᵀΛA straight into the factor, factorization, mean solve,
 * Takahashi variances and sample_direct draws — all on the device. perm: the
 * factor's ordering (new -> old) or NULL for nested dissection; samples depend
 * on it, as the reference's (pass its AMD order to reproduce its draws). */
typedef struct gmrf_regression gmrf_regression_t;
int gmrf_regression_create(const gmrf_matern_config_t* cfg, int32_t m, const double* points,
                           const int32_t* perm, gmrf_regression_t** out);
/* y, noise_prec: m values. mean, var: n (may be NULL); samples: n × n_samples
 * column-major (may be NULL), sample s = the s-th sample_direct(post, rng) of
 * Rng(seed) (gmrf.hpp:182-184). */
int gmrf_regression_run(gmrf_regression_t* h, const double* y, const double* noise_prec,
                        int32_t want_var, int32_t n_samples, uint64_t seed, double* mean,
                        double* var, double* samples);
typedef struct {
  int32_t n, m;
  int64_t nnz_pattern, nnz_l;
  double setup_host_ms, run_ms, flops_ref;
  int64_t kernel_launches;
} gmrf_regression_info_t;
int gmrf_regression_info(const gmrf_regression_t* h, gmrf_regression_info_t* info);
/* Q_prior and Q_post on the pattern (tests): col_ptr[n+1], row_idx, values. */
int gmrf_regression_precisions(const gmrf_regression_t* h, int64_t* col_ptr, int32_t* row_idx,
                               double* q_prior, double* q_post);
gmrf_factor_t* gmrf_regression_factor(gmrf_regression_t* h); /* borrowed */
void gmrf_regression_free(gmrf_regression_t* h);

/* ---- Space-time posterior pipeline (1D space × implicit-Euler time) --------
 * The chain the reference runs in bench/runner.hpp:457-632 (run_burgers):
 *   spatiotemporal_prior (priors/spatiotemporal.hpp:79)      → device assembly
 *   condition_on / condition_affine on the IC (gmrf.hpp:145)  → device update + factor
 *   gauss_newton (solver/gauss_newton.hpp:93) with
 *     burgers_fem_residual, implicit Euler (solver/residual.hpp:244)
 *   laplace_posterior (gauss_newton.hpp:228) + variance_takahashi (gmrf.hpp:205)
 * residual = 0 gives the linear (heat, config 3) posterior: conditioned prior. */
typedef struct gmrf_spacetime gmrf_spacetime_t;

typedef struct {
  int32_t n_el;            /* spatial P1 elements, n_s = n_el + 1 */
  double xa, xb;           /* spatial interval */
  int32_t n_t;             /* time slices over [0, t_end], uniform */
  double t_end;
  double diffusion;        /* proxy ν (laplace_operator / linear_proxy_operator) */
  double advection;        /* proxy c (0 for the heat proxy) */
  double noise_kappa;      /* spatial noise Matérn {κ, α, τ} */
  int32_t noise_alpha;
  double noise_tau;
  double init_kappa;       /* initial-slice Matérn {κ, α, τ} */
  int32_t init_alpha;
  double init_tau;
  double tau;              /* SpatiotemporalSpec::tau */
  double eps;              /* Dirichlet slack variance, embed_dirichlet(eps) */
  int32_t dirichlet;       /* 1: homogeneous Dirichlet at both ends */
  double ic_noise_prec;    /* Λ of the t=0 observation */
  int32_t residual;        /* 0: linear posterior, 1: Burgers weak form (implicit Euler, 1-D),
                              2: Allen-Cahn weak form (implicit Euler, lumped cubic, 1-D/2-D) */
  double pde_noise_prec;   /* Λ_pde of the residual rows */
  int32_t gn_max_iters;    /* GaussNewtonConfig (gauss_newton.hpp:19-24) */
  double gn_decrement_tol;
  double gn_armijo_c;
  double gn_shrink;
  int32_t gn_max_backtracks;
  int32_t dim;             /* 1: interval [xa, xb] with n_el elements; 2: unit square with
                              n_el × n_el cells split into triangles (mesh.hpp:108-149) */
} gmrf_spacetime_config_t;

typedef struct {
  int32_t iter;
  double objective, decrement, step_size;
  int32_t backtracks;
} gmrf_gn_iter_t; /* GaussNewtonIteration, gauss_newton.hpp:35-42 */

typedef struct {
  double setup_host_ms, init_ms, assemble_ms, condition_ms, gn_ms, laplace_ms, selinv_ms, numeric_ms;
  int32_t n_factorizations;
  int64_t kernel_launches;
  int32_t n, n_space, n_res;
  int64_t nnz_pattern, nnz_l, nnz_l_padded;
  double flops_ref, flops_sn;
  int64_t factor_device_bytes; /* L panels + lifetime-packed update matrices + Σ panels + work */
  /* numeric_ms covers every factorization, including the forward sweep that rides along
   * with those followed by a solve; numeric_pure_ms / n_pure_factorizations count only the
   * factorizations with nothing fused (the Laplace precision): the Cholesky rate. */
  double numeric_pure_ms;
  int32_t n_pure_factorizations;
} gmrf_spacetime_info_t;

int gmrf_spacetime_create(const gmrf_spacetime_config_t* cfg, gmrf_spacetime_t** out);
/* u0: IC values at the n_s nodes (host). mean/var: n outputs (host, may be NULL);
 * trace: up to max_trace GN iterations. Returns GMRF_ERR_NUMERICAL with the
 * trace filled on line-search stagnation (GaussNewtonStagnation). */
int gmrf_spacetime_run(gmrf_spacetime_t* h, const double* u0, int32_t want_var, double* mean,
                       double* var, gmrf_gn_iter_t* trace, int32_t max_trace, int32_t* n_trace,
                       int32_t* converged);
int gmrf_spacetime_info(const gmrf_spacetime_t* h, gmrf_spacetime_info_t* info);
/* Host only: the symbolic analysis of the pipeline's factor (master pattern,
 * geometric nested dissection, supernodes) without a device — for front
 * statistics and the per-rank memory plan of a partitioned run. */
int gmrf_spacetime_symbolic(const gmrf_spacetime_config_t* cfg, gmrf_symbolic_t** out);
/* Device pointers of the last run's mean / variances (n doubles each). */
int gmrf_spacetime_device_results(const gmrf_spacetime_t* h, const double** d_mean,
                                  const double** d_var);
/* Assembled joint precisions on the master pattern (tests): col_ptr[n+1],
 * row_idx[nnz], Q_cond values, q_eff values. */
int gmrf_spacetime_pattern(const gmrf_spacetime_t* h, int64_t* col_ptr, int32_t* row_idx,
                           double* q_cond, double* q_eff);
/* Residual rows f(u) and its Jacobian (CSR) at a host state u (tests). */
int gmrf_spacetime_residual(gmrf_spacetime_t* h, const double* u, double* f);
int gmrf_spacetime_jacobian_nnz(const gmrf_spacetime_t* h, int64_t* nnz);
int gmrf_spacetime_jacobian(gmrf_spacetime_t* h, const double* u, int64_t* row_ptr,
                            int32_t* col_idx, double* values);
void gmrf_spacetime_free(gmrf_spacetime_t* h);
/* The same pipeline with this rank's share of a partitioned factorization
 * (see gmrf_factor_create_partitioned); assembly, residuals and the line
 * search are replicated, every rank returns the complete mean and variances. */
int gmrf_spacetime_create_partitioned(const gmrf_spacetime_config_t* cfg, int32_t nranks,
                                      int32_t rank, gmrf_exchange_fn fn, void* ctx,
                                      gmrf_spacetime_t** out);

/* Per-kernel-class profile of the following runs (CUDA events on the launch
 * stream around every launch; ALGORITHMIC flops and bytes per class). */
typedef struct {
  char name[40];
  int64_t launches;
  double ms, flops, bytes;
} gmrf_kernel_stat_t;
int gmrf_spacetime_set_profile(gmrf_spacetime_t* h, int32_t on);
int gmrf_spacetime_kernel_stats(gmrf_spacetime_t* h, gmrf_kernel_stat_t* out, int32_t max,
                                int32_t* n);

#ifdef __cplusplus
}
#endif
#endif
