// Device conjugate gradients (cg.cu): cg_solve (core/cg.hpp:39-105) and
// sample_cg (gmrf.hpp:188-202).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.hpp"

namespace gmrf {

struct CgOptions {
  double rtol = 1e-8;
  double atol = 0.0;
  int64_t max_iter = 0;  // 0: 10 n
  bool jacobi = false;   // Preconditioner::kJacobi with csc_diag(Q)
};

struct CgOutcome {
  int64_t iterations = 0;
  double final_residual = 0.0;
  bool converged = false;
};

// Q: full CSC (n × n). x0 may be null (zeros). Host b, x0, x.
CgOutcome cg_solve_device(int n, const int64_t* cp, const int32_t* ri, const double* v,
                          const double* b, const double* x0, const CgOptions& opt, double* x,
                          cudaStream_t stream = nullptr);

// out = mean + Q⁻¹ S z (S: n × m CSC, z: m); raises kNumerical if CG fails.
void sample_cg_device(int n, const int64_t* qcp, const int32_t* qri, const double* qv, int m,
                      const int64_t* scp, const int32_t* sri, const double* sv,
                      const double* mean, const double* z, const CgOptions& opt, double* out,
                      cudaStream_t stream = nullptr);

}  // namespace gmrf
