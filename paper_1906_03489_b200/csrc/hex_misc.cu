// Hex BwdTrans / IProductWRTBase / PhysDeriv / IProductWRTDerivBase
// instantiations (K1-K3 + the IProductWRTDerivBase collection).
#include "common.cuh"
SPHP_DECLARE_TABLE_BANK(hex_misc)
#include "launch.cuh"
#ifndef SPHP_HEXOPS_BUDGET
#define SPHP_HEXOPS_BUDGET (40 * 1024)  // per-CTA smem target: measured (tools/time_hexops.py)
#endif

namespace sphp {

template <template <int, int, int, int, int> class OpT, int M, int Q, int GK>
static cudaError_t go_gk(const OpArgs& oa, int64_t goff, cudaStream_t s) {
  using Probe = OpT<M, Q, GK, 1, 32>;
  constexpr int NE = choose_ne(8 * per_elem_doubles<Probe>(), Q * Q, SPHP_HEXOPS_BUDGET);
  constexpr int NT = choose_nt(NE, Q * Q);
  using Op = OpT<M, Q, GK, NE, NT>;
  return launch_pipe<Op, 0>(oa, geom_record<3, Q * Q * Q>(GK), goff, s);
}

template <int M, int Q>
static cudaError_t bwd_key(const OpArgs& oa, cudaStream_t s) {
  using Probe = HexBwd<M, Q, 1, 32>;
  constexpr int NE = choose_ne(8 * per_elem_doubles<Probe>(), Q * Q, SPHP_HEXOPS_BUDGET);
  constexpr int NT = choose_nt(NE, Q * Q);
  return launch_pipe<HexBwd<M, Q, NE, NT>, 0>(oa, 0, 0, s);
}

template <int M, int Q>
static cudaError_t iprod_key(const OpArgs& oa, cudaStream_t s) {
  switch (oa.geom_kind) {
    case SPHP_GEOM_NONE: return go_gk<HexIprod, M, Q, SPHP_GEOM_NONE>(oa, 0, s);
    case SPHP_GEOM_AFFINE: return go_gk<HexIprod, M, Q, SPHP_GEOM_AFFINE>(oa, 0, s);
    case SPHP_GEOM_POINT: return go_gk<HexIprod, M, Q, SPHP_GEOM_POINT>(oa, 0, s);
  }
  return cudaErrorNotSupported;
}

template <int M, int Q>
static cudaError_t deriv_key(const OpArgs& oa, cudaStream_t s) {
  switch (oa.geom_kind) {
    case SPHP_GEOM_NONE: return go_gk<HexPhysDeriv, M, Q, SPHP_GEOM_NONE>(oa, 0, s);
    case SPHP_GEOM_AFFINE: return go_gk<HexPhysDeriv, M, Q, SPHP_GEOM_AFFINE>(oa, 0, s);
    case SPHP_GEOM_POINT:
      return go_gk<HexPhysDeriv, M, Q, SPHP_GEOM_POINT>(oa, even_up(Q * Q * Q), s);
  }
  return cudaErrorNotSupported;
}

template <int M, int Q>
static cudaError_t ipderiv_key(const OpArgs& oa, cudaStream_t s) {
  switch (oa.geom_kind) {
    case SPHP_GEOM_NONE: return go_gk<HexIPDeriv, M, Q, SPHP_GEOM_NONE>(oa, 0, s);
    case SPHP_GEOM_AFFINE: return go_gk<HexIPDeriv, M, Q, SPHP_GEOM_AFFINE>(oa, 0, s);
    case SPHP_GEOM_POINT: return go_gk<HexIPDeriv, M, Q, SPHP_GEOM_POINT>(oa, 0, s);
  }
  return cudaErrorNotSupported;
}

#define SPHP_DISPATCH(NAME, KEYFN)                                   \
  cudaError_t NAME(const OpArgs& oa, cudaStream_t s) {               \
    SPHP_HEX_KEYS(X_##KEYFN)                                         \
    return cudaErrorNotSupported;                                    \
  }
#define X_bwd_key(m, q) \
  if (oa.M == m && oa.Q == q) return bwd_key<m, q>(oa, s);
#define X_iprod_key(m, q) \
  if (oa.M == m && oa.Q == q) return iprod_key<m, q>(oa, s);
#define X_deriv_key(m, q) \
  if (oa.M == m && oa.Q == q) return deriv_key<m, q>(oa, s);
#define X_ipderiv_key(m, q) \
  if (oa.M == m && oa.Q == q) return ipderiv_key<m, q>(oa, s);

SPHP_DISPATCH(hex_bwd, bwd_key)
SPHP_DISPATCH(hex_iprod, iprod_key)
SPHP_DISPATCH(hex_physderiv, deriv_key)
SPHP_DISPATCH(hex_ipderiv, ipderiv_key)

}  // namespace sphp
