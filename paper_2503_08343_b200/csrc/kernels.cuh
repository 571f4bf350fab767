// Device-side task descriptors shared by the plan builder and the kernels.
#pragma once

#include <cstdint>

namespace gmrf {

constexpr int kNB = 64;        // supernode chunk width (columns per dense panel step)
constexpr int kTile = 64;      // GEMM output tile (kTile x kTile)
constexpr int kTrsmRows = 128; // rows per TRSM task
constexpr int kRowsSR = 64;    // slab rows per k_panel_rows CTA (one-wave levels)
constexpr int kSmallRows = 96; // fronts with at most this many rows use k_small_front

// C = beta*C + alpha * Σ_seg opA(A_seg) · opB(B_seg), all column-major.
// opA(A) is m×k: N → A(i,l) = a[i + l*lda]; T → a[l + i*lda].
// opB(B) is k×n: N → B(l,j) = b[l + j*ldb]; T → b[j + l*ldb].
struct GemmTask {
  double* c;
  const double* a[2];
  const double* b[2];
  int32_t ldc;
  int32_t lda[2], ldb[2];
  int32_t m, n;
  int32_t k[2];
  int32_t flags;  // bit (2*seg): transA, bit (2*seg+1): transB
  double alpha, beta;
};

// Split-K reduction of one output tile (splitk.cuh).
struct ReduceTask {
  double* c;
  int32_t ldc, m, n;
  int32_t nparts;
  int64_t part0;  // first partial tile (index into the scratch, kTile*kTile each)
  double alpha, beta;
};

// Diagonal-block Cholesky + TRSM of the rows below it, for one chunk.
struct PanelTask {
  double* d;          // top-left of the chunk's diagonal block
  int32_t ld;         // panel leading dimension (rows of the supernode)
  int32_t w;          // chunk width (<= kNB)
  int32_t nbelow;     // rows below the diagonal block
  int32_t tile;       // which kTrsmRows-row slab of the rows below
  int32_t gcol;       // internal index of the chunk's first column
  int32_t slot;       // chunk's L11 staging slot in its level (panel2.cuh)
};

// Extend-add work item: one front column b of supernode sn, receiving the
// children listed in pairs[p0 .. p0+np) = (child, first row index in the
// child's update column) in child order.
struct EaTask {
  int32_t sn;
  int32_t col;
  int32_t p0;
  int32_t np;
};

// Σ-gather work item: one (supernode, front column) pair.
struct ColTask {
  int32_t sn;
  int32_t col;
};

// Selected-inversion per-chunk dense work.
struct SelChunk {
  const double* l;   // L panel of the supernode
  double* sig;       // Σ panel of the supernode (may alias l: in-place selected inversion)
  int32_t ld;        // rows of the supernode
  int32_t c0;        // chunk offset inside the panel
  int32_t w;         // chunk width
  int32_t wsn;       // supernode width
  int32_t tile;      // TRSM row slab (for the TRSM kernel)
  const double* rd;  // 1/L_jj of the chunk's first column (factorization pivots)
  // TRSM: rows [0, nrows) of src (ld lds) → dst (ld ldd), dst = −src · L_JJ⁻¹;
  // diag: z = Z (w × w, ld ldz), Σ_JJ = L_JJ⁻ᵀ (L_JJ⁻¹ − Z)
  const double* src;
  double* dst;
  int32_t lds, ldd, nrows;
  const double* z;
  int32_t ldz;
};

// One 64-row block of a wide supernode's triangle in the solves (solve_wide.cuh).
constexpr int kWideW = 128;  // supernodes wider than this use the wide solve kernels
struct WideBlock {
  int32_t sn;
  int32_t b;      // block index inside the triangle
  int32_t nb;     // blocks in this supernode
  int32_t flag0;  // flag index of block 0 of this supernode
};

// Row gather/scatter of x for the partitioned backward-solve exchange
// (x[rows[i] + rr*n], partition.hpp).
struct RowXfer {
  const int32_t* rows;
  int32_t cnt;
  int64_t off;  // offset in the pack buffer, per right-hand side
};

// Device view of the symbolic structure (all arrays device-resident).
struct SymDev {
  const int32_t* sn_first;
  const int64_t* sn_rptr;
  const int32_t* sn_rows;
  const int32_t* relmap;
  const int32_t* ch_ptr;
  const int32_t* ch_list;
  const int64_t* lptr;
  const int64_t* uptr;
  int32_t n;
};


#ifdef __CUDACC__
// Children assembly of the solves: for every entry (ia, rr) of a child's update
// vector uc (rc × nrhs), *tgt(rel[ia], rr) += uc[ia + rr·rc]. rel is injective
// within one child, so the U entries a thread handles per pass are independent:
// all their loads (rel, uc, then the targets) are issued before any store —
// the compiler cannot reorder them itself, as the targets may alias uc.
template <int U, typename Tgt>
__device__ __forceinline__ void child_scatter(const int32_t* __restrict__ rel, const double* uc,
                                              int rc, int nrhs, Tgt tgt) {
  const int tot = rc * nrhs;
  for (int base = threadIdx.x; base < tot; base += U * blockDim.x) {
    double* p[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = base + u * blockDim.x;
      p[u] = nullptr;
      if (idx < tot) {
        const int ia = idx % rc, rr = idx / rc;
        p[u] = tgt(__ldg(rel + ia), rr);
        v[u] = uc[ia + rr * rc];
      }
    }
    double old[U];
#pragma unroll
    for (int u = 0; u < U; ++u) old[u] = p[u] ? *p[u] : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (p[u]) *p[u] = old[u] + v[u];
  }
}
#endif

}  // namespace gmrf
