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

/* takahashi_diagonal (core/takahashi.hpp:67): diag(Q⁻¹) in original order. */
int gmrf_selinv_diag(gmrf_factor_t* f, double* diag);
int gmrf_selinv_diag_device(gmrf_factor_t* f, double* d_diag);
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

/* FP64 issue-rate microbenchmark (TFLOP/s) of DMMA m8n8k4 and DFMA. */
int gmrf_bench_fp64(double* dmma_tflops, double* dfma_tflops);

#ifdef __cplusplus
}
#endif
#endif
