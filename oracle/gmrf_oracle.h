/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference's CPU hot path (gmrfpde core/*), used
 * only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as
 * the checker. Pinned against the reference itself (oracle/_ref, built from
 * /root/reference by oracle/Makefile) and the committed golden fixtures in
 * tests/golden/ — see tests/test_oracle_pins.py.
 *
 * Layout: CSC with int64 col_ptr (the reference's int32 overflows at C5,
 * SURVEY §0.5), int32 row indices sorted ascending per column, f64 values.
 * Permutations are new -> old (reference core/cholesky.hpp:17).
 */
#ifndef GMRF_ORACLE_H
#define GMRF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* B = P A Pᵀ, full symmetric pattern, rows sorted (sparse.hpp:290-303). */
int64_t orc_permute_symmetric(int32_t n, const int64_t* cp, const int32_t* ri,
                              const double* v, const int32_t* perm, int64_t* ocp,
                              int32_t* ori, double* ov);

/* symbolic_analyze (cholesky.hpp:68-88): parent[n], col_ptr_L[n+1]. */
int orc_symbolic(int32_t n, const int64_t* cp, const int32_t* ri, const int32_t* perm,
                 int32_t* parent, int64_t* colptr_l);

/* cholesky_refactor (cholesky.hpp:113-161), simplicial up-looking. Returns -1
 * on success or the ORIGINAL index of the first non-positive pivot. */
int32_t orc_cholesky(int32_t n, const int64_t* cp, const int32_t* ri, const double* v,
                     const int32_t* perm, const int64_t* lcp, int32_t* lri, double* lv);

/* solve_triangular (cholesky.hpp:179-222): mode 0 L y=b, 1 Lᵀ x=b (permuted
 * coordinates), 2 full Q⁻¹b in original coordinates. */
void orc_solve(int32_t n, const int64_t* lcp, const int32_t* lri, const double* lv,
               const int32_t* perm, int mode, int32_t nrhs, const double* b, double* x);

/* takahashi_selected_inverse (takahashi.hpp:19-64) on the pattern of L
 * (lower part, permuted coordinates; the upper half is its mirror). */
void orc_takahashi(int32_t n, const int64_t* lcp, const int32_t* lri, const double* lv,
                   double* sv);

/* takahashi_diagonal (takahashi.hpp:67-70) in original coordinates. */
void orc_takahashi_diag(int32_t n, const int64_t* lcp, const int32_t* lri,
                        const double* lv, const int32_t* perm, double* out);

#ifdef __cplusplus
}
#endif
#endif
