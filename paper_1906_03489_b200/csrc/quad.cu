// Quad (2D) instantiations of every operator: BwdTrans, IProductWRTBase,
// PhysDeriv, IProductWRTDerivBase and the fused Helmholtz (local and
// explicit-map assembled).
#include "common.cuh"
SPHP_DECLARE_TABLE_BANK(quad)
#include "launch.cuh"
#ifndef SPHP_QUAD_BUDGET
#define SPHP_QUAD_BUDGET (40 * 1024)  // per-CTA smem target: measured best for cfg2 (tools/time_quad.py)
#endif

namespace sphp {

template <template <int, int, int, int, int> class OpT, int M, int Q, int GK, bool ASM = false>
static cudaError_t qgo(const OpArgs& oa, int64_t goff, cudaStream_t s) {
  using Probe = OpT<M, Q, GK, 1, 32>;
  constexpr int NE = choose_ne(8 * per_elem_doubles<Probe>(), Q, SPHP_QUAD_BUDGET);
  constexpr int NT = choose_nt(NE, Q);
  using Op = OpT<M, Q, GK, NE, NT>;
  const int64_t rec = geom_record<2, Q * Q>(GK);
  if (oa.mode == AsmMode::LOCAL) return launch_pipe<Op, 0>(oa, rec, goff, s);
  if constexpr (ASM) {
    if (oa.mode == AsmMode::EXPLICIT) return launch_pipe<Op, 2>(oa, rec, goff, s);
    if (oa.mode == AsmMode::EXPLICIT_GATHER) return launch_pipe<Op, 4>(oa, rec, goff, s);
  }
  return cudaErrorNotSupported;
}

// the Helmholtz tile is 8 elements (its bank-spread layout assumes it)
template <int M, int Q, int GK>
static cudaError_t qhelm_go(const OpArgs& oa, cudaStream_t s) {
  constexpr int NE = 8;
  constexpr int NT = choose_nt(NE, Q);
  using Op = QuadHelm<M, Q, GK, NE, NT>;
  const int64_t rec = geom_record<2, Q * Q>(GK);
  if (oa.mode == AsmMode::LOCAL) return launch_pipe<Op, 0>(oa, rec, 0, s);
  if (oa.mode == AsmMode::EXPLICIT) return launch_pipe<Op, 2>(oa, rec, 0, s);
  if (oa.mode == AsmMode::EXPLICIT_GATHER) return launch_pipe<Op, 4>(oa, rec, 0, s);
  return cudaErrorNotSupported;
}

template <int M, int Q>
static cudaError_t qhelm_key(const OpArgs& oa, cudaStream_t s) {
  if (oa.geom_kind == SPHP_GEOM_METRIC) return qhelm_go<M, Q, SPHP_GEOM_METRIC>(oa, s);
  if (oa.geom_kind == SPHP_GEOM_AFFINE) return qhelm_go<M, Q, SPHP_GEOM_AFFINE>(oa, s);
  return cudaErrorNotSupported;
}

template <int M, int Q>
static cudaError_t qbwd_key(const OpArgs& oa, cudaStream_t s) {
  using Probe = QuadBwd<M, Q, 1, 32>;
  constexpr int NE = choose_ne(8 * per_elem_doubles<Probe>(), Q, SPHP_QUAD_BUDGET);
  constexpr int NT = choose_nt(NE, Q);
  return launch_pipe<QuadBwd<M, Q, NE, NT>, 0>(oa, 0, 0, s);
}

template <int M, int Q>
static cudaError_t qiprod_key(const OpArgs& oa, cudaStream_t s) {
  switch (oa.geom_kind) {
    case SPHP_GEOM_NONE: return qgo<QuadIprod, M, Q, SPHP_GEOM_NONE>(oa, 0, s);
    case SPHP_GEOM_AFFINE: return qgo<QuadIprod, M, Q, SPHP_GEOM_AFFINE>(oa, 0, s);
    case SPHP_GEOM_POINT: return qgo<QuadIprod, M, Q, SPHP_GEOM_POINT>(oa, 0, s);
  }
  return cudaErrorNotSupported;
}

template <int M, int Q>
static cudaError_t qderiv_key(const OpArgs& oa, cudaStream_t s) {
  switch (oa.geom_kind) {
    case SPHP_GEOM_NONE: return qgo<QuadPhysDeriv, M, Q, SPHP_GEOM_NONE>(oa, 0, s);
    case SPHP_GEOM_AFFINE: return qgo<QuadPhysDeriv, M, Q, SPHP_GEOM_AFFINE>(oa, 0, s);
    case SPHP_GEOM_POINT:
      return qgo<QuadPhysDeriv, M, Q, SPHP_GEOM_POINT>(oa, even_up(Q * Q), s);
  }
  return cudaErrorNotSupported;
}

template <int M, int Q>
static cudaError_t qipderiv_key(const OpArgs& oa, cudaStream_t s) {
  switch (oa.geom_kind) {
    case SPHP_GEOM_NONE: return qgo<QuadIPDeriv, M, Q, SPHP_GEOM_NONE>(oa, 0, s);
    case SPHP_GEOM_AFFINE: return qgo<QuadIPDeriv, M, Q, SPHP_GEOM_AFFINE>(oa, 0, s);
    case SPHP_GEOM_POINT: return qgo<QuadIPDeriv, M, Q, SPHP_GEOM_POINT>(oa, 0, s);
  }
  return cudaErrorNotSupported;
}

#define SPHP_QDISPATCH(NAME, KEYFN)                    \
  cudaError_t NAME(const OpArgs& oa, cudaStream_t s) { \
    SPHP_QUAD_KEYS(X_##KEYFN)                          \
    return cudaErrorNotSupported;                      \
  }
#define X_qhelm_key(m, q) \
  if (oa.M == m && oa.Q == q) return qhelm_key<m, q>(oa, s);
#define X_qbwd_key(m, q) \
  if (oa.M == m && oa.Q == q) return qbwd_key<m, q>(oa, s);
#define X_qiprod_key(m, q) \
  if (oa.M == m && oa.Q == q) return qiprod_key<m, q>(oa, s);
#define X_qderiv_key(m, q) \
  if (oa.M == m && oa.Q == q) return qderiv_key<m, q>(oa, s);
#define X_qipderiv_key(m, q) \
  if (oa.M == m && oa.Q == q) return qipderiv_key<m, q>(oa, s);

SPHP_QDISPATCH(quad_helmholtz, qhelm_key)
SPHP_QDISPATCH(quad_bwd, qbwd_key)
SPHP_QDISPATCH(quad_iprod, qiprod_key)
SPHP_QDISPATCH(quad_physderiv, qderiv_key)
SPHP_QDISPATCH(quad_ipderiv, qipderiv_key)

}  // namespace sphp
