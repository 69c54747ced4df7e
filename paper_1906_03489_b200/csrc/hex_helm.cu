// Fused hex Helmholtz (K4) instantiations: local, periodic-assembled and
// explicit-map-assembled modes for the METRIC and AFFINE geometry encodings.
#include "common.cuh"
#ifndef HELM_PART
#define HELM_PART 0
#endif
#if HELM_PART == 0
SPHP_DECLARE_TABLE_BANK(hex_helm0)
#elif HELM_PART == 1
SPHP_DECLARE_TABLE_BANK(hex_helm1)
#else
SPHP_DECLARE_TABLE_BANK(hex_helm2)
#endif
#include <cstdlib>

#include "launch.cuh"

namespace sphp {

// Op::GDIR_LOCAL when the plan declares it: its local operator reads the
// geometry from global memory (pipeline MODE 7)
template <class Op>
constexpr auto gdir_local_impl(int) -> decltype(Op::GDIR_LOCAL, bool()) { return Op::GDIR_LOCAL; }
template <class Op>
constexpr bool gdir_local_impl(...) { return false; }

// tile-shape variants: (input stages, shared-memory budget per CTA)
constexpr int pow2_floor(int x) { return x >= 8 ? 8 : (x >= 4 ? 4 : (x >= 2 ? 2 : 1)); }
// the i-column plan runs element-fastest lanes over NE = 1, 2, 4 or 8
// elements; SPHP_COL_NE_<M> pins the local tile of one order (tuning)
template <int M, int Q, int GK, int NSTP, int BUDGET, bool COL>
constexpr int helm_ne() {
  using Probe = HexHelmSel<M, Q, GK, 1, 32, NSTP, COL>;
  constexpr int ne = choose_ne(8 * per_elem_doubles<Probe>(NSTP), Q * Q, BUDGET);
  return COL ? pow2_floor(ne) : ne;
}
template <int M, int Q, int GK, int NSTP, int NE>
static cudaError_t helm_variant_ne(const OpArgs& oa, cudaStream_t s) {
  constexpr int NT = choose_nt(NE, Q * Q);
  using Op = HexHelm<M, Q, GK, NE, NT, NSTP>;
  if constexpr (Scaffold<Op, 0>::SMEM_BYTES > 227 * 1024 || Scaffold<Op, 3>::SMEM_BYTES > 227 * 1024) {
    return cudaErrorNotSupported;
  } else {
    return launch_mode<Op>(oa, geom_record<3, Q * Q * Q>(GK), 0, s);
  }
}
template <int M, int Q, int GK, int NSTP, int BUDGET>
static cudaError_t helm_variant(const OpArgs& oa, cudaStream_t s) {
  constexpr int NE = helm_ne<M, Q, GK, NSTP, BUDGET, col_plan(Q)>();
  constexpr int NT = choose_nt(NE, Q * Q);
  using Op = HexHelm<M, Q, GK, NE, NT, NSTP>;
  if constexpr (gdir_local_impl<Op>(0)) {
    // full tiles only (the compute reads every element of a tile)
    if (oa.mode == AsmMode::LOCAL && oa.E % NE == 0)
      return launch_pipe<Op, 7>(oa, geom_record<3, Q * Q * Q>(GK), 0, s);
  }
  return launch_mode<Op>(oa, geom_record<3, Q * Q * Q>(GK), 0, s);
}

#ifdef SPHP_TUNING
static int helm_variant_env() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("SPHP_HELM_VARIANT");
    v = e ? atoi(e) : -1;
  }
  return v;
}
#endif

// default tile shapes (tools/time_helm.py sweep on B200, profiles/r01_tune.log):
// one input stage and ~74 KB (local) / ~55 KB (gathering modes) per CTA
// beat double buffering at every order: more resident CTAs hide more latency
// than a second stage does.  SPHP_HELM_VARIANT=0..4 overrides for tuning.
#ifndef SPHP_LOCAL_BUDGET_KB
#define SPHP_LOCAL_BUDGET_KB 74
#endif

// PERIODIC_CLASS (pipeline MODE 5): tiles of NE consecutive elements of an
// x-row (NE must divide n)
// MODE 6 (geometry from global memory, L2-prefetched): the k-major orders (SPHP_CLASS_GDIR)
#ifndef SPHP_CLASS_GDIR
// 1: the class launch of k-major METRIC orders (Q = 9: P = 7) reads the
// geometry from global memory too (MODE 6) — 2.577 -> 2.534 ms once the
// per-tile divisions were gone (it lost 8 % before: profiles/r02_kmajor.log)
#define SPHP_CLASS_GDIR 1
#endif
template <int M, int Q, int GK>
constexpr int class_mode() {
  return (GK == SPHP_GEOM_METRIC && !col_plan(Q) && SPHP_CLASS_GDIR && metric_kmajor(Q)) ? 6 : 5;
}
template <int M, int Q, int GK, int NE>
constexpr size_t class_smem() {
  using Op = HexHelm<M, Q, GK, NE, choose_nt(NE, Q * Q), 1>;
  return Scaffold<Op, class_mode<M, Q, GK>()>::SMEM_BYTES;
}
// tile size of the class mode: the NE in {1, 2, 4, 8} that keeps the most
// elements resident per SM (shared memory: 228 KB per SM, 1 KB per CTA;
// at most 256 work items per stage, i.e. threads, so registers do not cap
// the pointwise stage), the smaller NE (more CTAs) on ties; SPHP_CLASS_NE
// overrides (tuning builds)
template <int M, int Q, int GK, int NE>
constexpr int class_resident() {
  constexpr size_t b = class_smem<M, Q, GK, NE>();
  return (b > 227 * 1024 || (NE > 1 && NE * Q * Q > 256)) ? 0 : (int)(233472 / (b + 1024)) * NE;
}
template <int M, int Q, int GK>
constexpr int class_ne() {
#ifdef SPHP_CLASS_NE
  return SPHP_CLASS_NE;
#else
  // measured (tools/time_phases.py, cfg4 64^3, METRIC, Q = P + 2): P = 2..8
  // -> 4, 8, 4, 2, 1, 1, 1 (residency alone picks 2 at P = 3 and 1 at P = 5,
  // 9-10 % slower there; 8 vs 4 at P = 3: -1.4 %)
  // i-column plan: P = 2 8 (0.181 vs 0.184 ms at 4), P = 3 4 (0.388 vs 0.397 at 8), P = 5 2
  // P = 4 2 (0.665 vs 0.700 ms at 4: five CTAs per SM)
  if (GK == SPHP_GEOM_METRIC && Q == M + 1 && col_plan(Q)) return M == 3 ? 8 : (M == 4 ? 4 : (M <= 6 ? 2 : 1));
  if (GK == SPHP_GEOM_METRIC && Q == M + 1) return M == 4 ? 8 : (M <= 5 ? 4 : (M == 6 ? 2 : 1));
  int best = 1, score = class_resident<M, Q, GK, 1>();
  if (class_resident<M, Q, GK, 2>() > score) best = 2, score = class_resident<M, Q, GK, 2>();
  if (class_resident<M, Q, GK, 4>() > score) best = 4, score = class_resident<M, Q, GK, 4>();
  if (class_resident<M, Q, GK, 8>() > score) best = 8, score = class_resident<M, Q, GK, 8>();
  return best;
#endif
}

template <int M, int Q, int GK, int NE>
static cudaError_t helm_class_ne(const OpArgs& oa, cudaStream_t s);
template <int M, int Q, int GK>
static cudaError_t helm_class(const OpArgs& oa, cudaStream_t s) {
#ifdef SPHP_TUNING
  static const int ne_env = [] {
    const char* e = getenv("SPHP_CLASS_NE_ENV");
    return e ? atoi(e) : 0;
  }();
  switch (ne_env) {
    case 1: return helm_class_ne<M, Q, GK, 1>(oa, s);
    case 2: return helm_class_ne<M, Q, GK, 2>(oa, s);
    case 4: return helm_class_ne<M, Q, GK, 4>(oa, s);
    case 8: return helm_class_ne<M, Q, GK, 8>(oa, s);
    default: break;
  }
#endif
  return helm_class_ne<M, Q, GK, class_ne<M, Q, GK>()>(oa, s);
}
template <int M, int Q, int GK, int NE>
static cudaError_t helm_class_ne(const OpArgs& oa, cudaStream_t s) {
  if constexpr (M < 3 || class_smem<M, Q, GK, NE>() > 227 * 1024) {
    return cudaErrorNotSupported;  // not even a two-element tile fits: split
  } else {
    constexpr int NT = choose_nt(NE, Q * Q);
    using Op = HexHelm<M, Q, GK, NE, NT, 1>;
    if (M < 3 || oa.n % NE != 0 || oa.n % 2 != 0 || oa.E % NE != 0) return cudaErrorNotSupported;
    if (oa.ne_out) *oa.ne_out = NE;
    return launch_pipe<Op, class_mode<M, Q, GK>()>(oa, geom_record<3, Q * Q * Q>(GK), 0, s);
  }
}

template <int M, int Q, int GK>
static cudaError_t helm_go(const OpArgs& oa, cudaStream_t s) {
  if (oa.mode == AsmMode::PERIODIC_CLASS) return helm_class<M, Q, GK>(oa, s);
  if (oa.mode == AsmMode::LOCAL || oa.mode == AsmMode::PERIODIC_GATHER) {
#ifdef SPHP_TUNING  // tile-shape sweep build (make EXTRA_NVFLAGS=-DSPHP_TUNING)
    switch (helm_variant_env()) {
      case 0: return helm_variant<M, Q, GK, 2, 110 * 1024>(oa, s);
      case 1: return helm_variant<M, Q, GK, 1, 74 * 1024>(oa, s);
      case 2: return helm_variant<M, Q, GK, 1, 55 * 1024>(oa, s);
      case 3: return helm_variant<M, Q, GK, 2, 74 * 1024>(oa, s);
      case 4: return helm_variant<M, Q, GK, 1, 110 * 1024>(oa, s);
      case 11: return helm_variant_ne<M, Q, GK, 1, 1>(oa, s);
      case 12: return helm_variant_ne<M, Q, GK, 1, 2>(oa, s);
      case 14: return helm_variant_ne<M, Q, GK, 1, 4>(oa, s);
      case 18: return helm_variant_ne<M, Q, GK, 1, 8>(oa, s);
      default: break;
    }
#endif
    if (oa.mode == AsmMode::LOCAL) return helm_variant<M, Q, GK, 1, SPHP_LOCAL_BUDGET_KB * 1024>(oa, s);
  }
  return helm_variant<M, Q, GK, 1, 55 * 1024>(oa, s);
}

template <int M, int Q>
static cudaError_t helm_key(const OpArgs& oa, cudaStream_t s) {
  if (oa.geom_kind == SPHP_GEOM_METRIC) return helm_go<M, Q, SPHP_GEOM_METRIC>(oa, s);
  if (oa.geom_kind == SPHP_GEOM_AFFINE) return helm_go<M, Q, SPHP_GEOM_AFFINE>(oa, s);
  return cudaErrorNotSupported;
}

#if HELM_PART == 0
#define HELM_KEYS(X) X(2, 3) X(2, 4) X(3, 4) X(3, 5) X(4, 5) X(4, 6)
cudaError_t hex_helmholtz_part0(const OpArgs& oa, cudaStream_t s) {
#elif HELM_PART == 1
#define HELM_KEYS(X) X(5, 6) X(5, 7) X(6, 7) X(6, 8)
cudaError_t hex_helmholtz_part1(const OpArgs& oa, cudaStream_t s) {
#else
#define HELM_KEYS(X) X(7, 8) X(7, 9) X(8, 9) X(8, 10) X(9, 10) X(9, 11)
cudaError_t hex_helmholtz_part2(const OpArgs& oa, cudaStream_t s) {
#endif
#define X(m, q) \
  if (oa.M == m && oa.Q == q) return helm_key<m, q>(oa, s);
  HELM_KEYS(X)
#undef X
  return cudaErrorNotSupported;
}

#if HELM_PART == 0
cudaError_t hex_helmholtz_part1(const OpArgs& oa, cudaStream_t s);
cudaError_t hex_helmholtz_part2(const OpArgs& oa, cudaStream_t s);
cudaError_t hex_helmholtz(const OpArgs& oa, cudaStream_t s) {
  if (oa.M <= 4) return hex_helmholtz_part0(oa, s);
  if (oa.M <= 6) return hex_helmholtz_part1(oa, s);
  return hex_helmholtz_part2(oa, s);
}
#endif

}  // namespace sphp
