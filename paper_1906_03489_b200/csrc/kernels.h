// Host-side launch interface of the templated kernels (one entry per
// operator family; each dispatches on (M, Q) to a fully unrolled
// instantiation and returns cudaErrorNotSupported for keys outside the
// fast set).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sphp {

// LOCAL: block in/out.  PERIODIC / EXPLICIT: one colour class, gather in,
// scatter-add out.  PERIODIC_GATHER / EXPLICIT_GATHER: all elements, gather
// in, local block out (the owner-computes assembly then sums it).
// PERIODIC_CLASS: periodic hex, all elements in order: the tile's modes are
// gathered by entity-class ranges of the global vector (16-byte cp.async
// chunks) and the results leave, class-major within each tile, into the
// tile-major block Z (the interiors straight into y), which
// class_owner_sum then reduces.
enum class AsmMode : int {
  LOCAL = 0,
  PERIODIC = 1,
  EXPLICIT = 2,
  PERIODIC_GATHER = 3,
  EXPLICIT_GATHER = 4,
  PERIODIC_CLASS = 5
};

struct OpArgs {
  int M, Q;          // modes / points per direction
  int64_t E;         // elements in the collection
  const double* in;  // device input block
  double* out;       // device output block
  const double* geom;
  int geom_kind;     // SPHP_GEOM_*
  int64_t gstride;   // geometry doubles per element
  double lam;
  int num_sms;
  // assembled Helmholtz
  AsmMode mode;
  const double* xg;   // global input
  double* yg;         // global output (accumulated, colour by colour)
  const int* elist;   // EXPLICIT: element ids of this colour (device)
  int64_t nlist;      // number of elements in this colour
  const int* codes;   // EXPLICIT: (E, nm) int32 codes
  const int* ent_g;   // PERIODIC_GATHER: precomputed (E, 27) entity bases (optional)
  int n;              // PERIODIC: grid size
  int colour;         // PERIODIC: colour id 0..7
  int reverse = 0;    // LOCAL: walk the tiles last to first
  // PERIODIC_CLASS: absolute index of the launch's first element (z-slab
  // pipelines), the output block Z (per tile of NE elements: classes 0..25,
  // class-major, NE * (nm - (P-1)^3) doubles; then n^3 (P-1)^3 interior
  // values when they do not go straight into yg)
  int64_t e0 = 0;
  double* zbuf = nullptr;
  int direct_interior = 0;
  int* ne_out = nullptr;  // PERIODIC_CLASS: receives the tile size NE (Z layout)
};

// hex (3D) sum-factorisation kernels
cudaError_t hex_helmholtz(const OpArgs& a, cudaStream_t s);
cudaError_t hex_bwd(const OpArgs& a, cudaStream_t s);
cudaError_t hex_iprod(const OpArgs& a, cudaStream_t s);
cudaError_t hex_physderiv(const OpArgs& a, cudaStream_t s);
cudaError_t hex_ipderiv(const OpArgs& a, cudaStream_t s);
// quad (2D)
cudaError_t quad_helmholtz(const OpArgs& a, cudaStream_t s);
cudaError_t quad_bwd(const OpArgs& a, cudaStream_t s);
cudaError_t quad_iprod(const OpArgs& a, cudaStream_t s);
cudaError_t quad_physderiv(const OpArgs& a, cudaStream_t s);
cudaError_t quad_ipderiv(const OpArgs& a, cudaStream_t s);

cudaError_t upload_all_tables();

}  // namespace sphp
