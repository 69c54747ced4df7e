// Host interface of misc.cu (geometry, assembly, StdMat helpers).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sphp {

struct GeomJob {
  int dim, Q, n, kind, mapping;
  int64_t E, e0, npts, cs, stride;
  const int64_t* ids;  // device, may be null
  const double* z;     // device (Q)
  const double* w;     // device (Q)
  double L[3];
  double amp;
  double* out;
};

struct AmapDev {
  int periodic;  // 1: analytic periodic hex numbering
  int n, P;      // periodic grid
  int nm;
  int64_t E;
  int64_t num_global;
  const int* codes;  // explicit: (E, nm)
};

struct PointJob {
  int dim, kind;
  int64_t E, np, cs, stride;
  const double* geom;
  const double* wstd;  // device (np) standard weights
};

cudaError_t geom_analytic(const GeomJob& j, int* bad, cudaStream_t s);
cudaError_t geom_convert(const GeomJob& j, const double* wj, const double* inv, int* bad,
                         cudaStream_t s);
cudaError_t jacobian_factors(int64_t E, int64_t np, const double* dx, const double* dy,
                             const double* w, double* wj, double* inv, unsigned long long* bad,
                             cudaStream_t s);
// class-range kernels (periodic_ops.cu) over the x-rows [row0, row1) of
// rows ey + n ez (row1 < 0: all); cudaErrorNotSupported if the grid or
// order is outside their range
// block Z of the PERIODIC_CLASS operator mode (tiles of ne elements):
// doubles needed, and its owner-computes sum into y (rows [row0, row1) of
// (ey, ez); with or without the interior region)
int64_t class_block_doubles(int n, int P);
cudaError_t class_owner_sum(int n, int P, int ne, const double* Z, double* y, int accumulate,
                            int with_interior, cudaStream_t s, int row0 = 0, int row1 = -1);
// (ctr: one device int of the caller's per-stream workspace for the
// dynamic segment schedule, or null for the static one)
cudaError_t owner_periodic_v3(int n, int P, const double* loc, double* y, int accumulate,
                              cudaStream_t s, int row0 = 0, int row1 = -1, int* ctr = nullptr);
cudaError_t periodic_scatter_v2(int n, int P, const double* x, double* loc, cudaStream_t s,
                                int row0 = 0, int row1 = -1, int* ctr = nullptr);
cudaError_t periodic_entity_table(int n, int P, int* ent, cudaStream_t s);
cudaError_t index_gather(int64_t n, const int64_t* idx, const double* src, double* dst, cudaStream_t s);
cudaError_t index_sum2(int64_t n, const int64_t* idx, const double* lo, const double* hi, double* y,
                       cudaStream_t s);
cudaError_t amap_scatter(const AmapDev& m, const double* g, double* loc, cudaStream_t s, int* ctr = nullptr);
cudaError_t owner_assemble_csr32(int64_t ng, const int* rowp, const int* ent, const double* loc, double* y,
                                 cudaStream_t s);
cudaError_t amap_assemble(const AmapDev& m, const double* loc, double* g, int ncolours,
                          const int* elist_dev, const int64_t* colour_off, int accumulate,
                          cudaStream_t s);
cudaError_t dgemm(int64_t R, int N, int K, const double* A, const double* B, double* C,
                  cudaStream_t s);
// which: 0 = weights (IProduct), 1 = metric transform in place (PhysDeriv),
//        2 = flux (IProductWRTDerivBase)
cudaError_t pointwise(int which, const PointJob& j, const double* in, double* out, cudaStream_t s);
cudaError_t elem_matvec(int64_t E, int nm, const double* H, const double* x, double* y,
                        cudaStream_t s);
cudaError_t unit_block(int64_t E, int nm, int n, double* x, cudaStream_t s);
cudaError_t store_column(int64_t E, int nm, int n, const double* y, double* H, cudaStream_t s);
cudaError_t symmetrise(int64_t E, int nm, double* H, cudaStream_t s);
// loc is element-major (E, nm), or mode-major (nm, E) when mode_major != 0
cudaError_t owner_assemble_periodic(int n, int P, const double* loc, double* y, int accumulate,
                                    int mode_major, cudaStream_t s, int* ctr = nullptr);
cudaError_t owner_assemble_csr(int64_t ng, const int64_t* rowp, const int* ent, const double* loc,
                               double* y, int accumulate, int nm, int64_t E, int mode_major,
                               cudaStream_t s);

}  // namespace sphp
