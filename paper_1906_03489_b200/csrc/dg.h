// Host launchers of the DG primitive kernels (dg.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/spechp_b200.h"

namespace sphp {

cudaError_t batched_matvec(int64_t E, int m, int n, const double* A, const double* x,
                           const double* s, double alpha, int accumulate, double* y, cudaStream_t st);
cudaError_t trace_extract(int64_t T, int nq, int np, const double* ex, const int64_t* idx,
                          const double* phys, double* out, cudaStream_t st);
cudaError_t trace_lift(int nrhs, int64_t E, int nm, int nq, int64_t T, const int64_t* rowp,
                       const int64_t* codes, const double* Lm, const double* Lp, const double* w,
                       const double* s, double* b, cudaStream_t st);
cudaError_t ape_trace_flux(int64_t npts, int riemann, int bc, const double* qm, const double* qp,
                           const double* gv, const double* nrm, const double* base,
                           const double* w, double* out, int64_t ostride, cudaStream_t st);
cudaError_t ape_volume(int64_t E, int np, const double* q, const double* base, double* G,
                       double* HX, double* HY, cudaStream_t st);
cudaError_t advect_volume(int64_t E, int np, const double* ax, const double* ay, const double* u,
                          double* F, cudaStream_t st);
cudaError_t advect_trace_flux(int64_t npts, int bc, const double* an, const double* um,
                              const double* up, const double* gv, double* out, cudaStream_t st);
cudaError_t scale_points(int64_t n, const double* c, const double* v, const double* src, double* out,
                         cudaStream_t st);

}  // namespace sphp
