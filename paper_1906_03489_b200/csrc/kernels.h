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
enum class AsmMode : int { LOCAL = 0, PERIODIC = 1, EXPLICIT = 2, PERIODIC_GATHER = 3, EXPLICIT_GATHER = 4 };

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
