// Fused hex Helmholtz (K4) instantiations: local, periodic-assembled and
// explicit-map-assembled modes for the METRIC and AFFINE geometry encodings.
#include "common.cuh"
SPHP_DECLARE_TABLE_BANK(hex_helm)
#include "launch.cuh"

namespace sphp {

template <int M, int Q, int GK>
static cudaError_t helm_go(const OpArgs& oa, cudaStream_t s) {
  using Probe = HexHelm<M, Q, GK, 1, 32>;
  constexpr int NE = choose_ne(8 * per_elem_doubles<Probe>(), Q * Q);
  constexpr int NT = choose_nt(NE, Q * Q);
  using Op = HexHelm<M, Q, GK, NE, NT>;
  return launch_mode<Op>(oa, geom_record<3, Q * Q * Q>(GK), 0, s);
}

template <int M, int Q>
static cudaError_t helm_key(const OpArgs& oa, cudaStream_t s) {
  if (oa.geom_kind == SPHP_GEOM_METRIC) return helm_go<M, Q, SPHP_GEOM_METRIC>(oa, s);
  if (oa.geom_kind == SPHP_GEOM_AFFINE) return helm_go<M, Q, SPHP_GEOM_AFFINE>(oa, s);
  return cudaErrorNotSupported;
}

cudaError_t hex_helmholtz(const OpArgs& oa, cudaStream_t s) {
#define X(m, q) \
  if (oa.M == m && oa.Q == q) return helm_key<m, q>(oa, s);
#ifdef SPHP_ONE_KEY
  X(5, 6)
#else
  SPHP_HEX_KEYS(X)
#endif
#undef X
  return cudaErrorNotSupported;
}

}  // namespace sphp
