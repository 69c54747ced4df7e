// Host interface of solver.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sphp {

struct DiagJob {
  int dim, m, Q, kind;
  int64_t E, stride, cs;
  double lam;
  const double* B;   // device (m, Q)
  const double* Bd;  // device (m, Q)
  const double* w;   // device (Q)
  const double* geom;
  double* out;       // (E, nm)
};

cudaError_t helmholtz_diagonal(const DiagJob& j, cudaStream_t s);
int reduction_partials();
cudaError_t vec_dot2(int64_t n, const double* a, const double* b, const double* c, const double* d,
                     double* partial, double* out, cudaStream_t s);
cudaError_t cg_init(int64_t n, const double* rhs, const double* dinv, double* x, double* r, double* z,
                    double* p, double* partial, double* out, cudaStream_t s);
cudaError_t cg_update(int64_t n, double alpha, const double* p, const double* ap, double* x, double* r,
                      const double* dinv, double* z, double* partial, double* out, cudaStream_t s);
cudaError_t cg_direction(int64_t n, double beta, const double* z, double* p, cudaStream_t s);
// device-scalar CG (solver.cu: state layout)
int cg_state_size(int max_iter);
cudaError_t cg_init_dev(int64_t n, const double* rhs, const double* dinv, double* x, double* r, double* z,
                        double* p, double* st, int max_iter, double tol, cudaStream_t s);
cudaError_t cg_step_dev(int64_t n, const double* p, const double* ap, double* x, double* r, const double* dinv,
                        double* z, double* pp, double* st, int max_iter, cudaStream_t s);

}  // namespace sphp
