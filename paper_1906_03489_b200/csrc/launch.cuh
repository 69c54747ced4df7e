// Launch helpers: tile-size selection per (operator, M, Q) and the (M, Q)
// dispatch switch over the fast key set.
#pragma once
#include <cstdlib>

#include "quad_ops.cuh"

#ifndef SPHP_SMEM_BUDGET
#define SPHP_SMEM_BUDGET (74 * 1024)  // per CTA: three resident CTAs per SM
#endif
#ifndef SPHP_MAX_ITEMS
#define SPHP_MAX_ITEMS 256  // work items per stage per CTA
#endif

namespace sphp {

// per-element shared-memory footprint of an Op (doubles)
template <class Op1>
constexpr int per_elem_doubles(int nst = 1) {
  return nst * (Op1::IN + Op1::GEO) + Op1::OUT + Op1::WORK;
}
constexpr int choose_ne(int per_el_bytes, int items_per_el, int budget = SPHP_SMEM_BUDGET) {
  int ne = budget / per_el_bytes;
  int cap = SPHP_MAX_ITEMS / items_per_el;
  if (cap < 1) cap = 1;
  if (ne > cap) ne = cap;
  if (ne < 1) ne = 1;
  return ne;
}
constexpr int choose_nt(int ne, int items_per_el) {
  int t = ((ne * items_per_el + 31) / 32) * 32;
  return t < 64 ? 64 : (t > 512 ? 512 : t);
}

struct LaunchCache {
  int dev = -1;
  size_t smem = 0;
  int occ = 0;
};

template <class Op, int MODE>
cudaError_t launch_pipe(const OpArgs& oa, int64_t gstride, int64_t goff, cudaStream_t s) {
  using Sc = Scaffold<Op, MODE>;
  auto kern = pipe_kernel<Op, MODE>;
  static LaunchCache cache[16];
  int dev = 0;
  cudaGetDevice(&dev);
  LaunchCache& c = cache[dev & 15];
  if (c.dev != dev) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)Sc::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int occ = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Op::NT, Sc::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    c.occ = occ;
    c.smem = Sc::SMEM_BYTES;
    c.dev = dev;
  }
  DevArgs a;
  a.E = oa.E;
  a.in = oa.in;
  a.out = oa.out;
  a.geom = oa.geom;
  a.gstride = gstride;
  a.goff = goff;
  a.lam = oa.lam;
  a.use_tma = ((reinterpret_cast<uintptr_t>(oa.in) & 15) == 0) &&
              (oa.geom == nullptr || (reinterpret_cast<uintptr_t>(oa.geom) & 15) == 0);
  a.xg = oa.xg;
  a.yg = oa.yg;
  a.elist = oa.elist;
  a.nlist = oa.nlist;
  a.codes = oa.codes;
  a.ent_g = oa.ent_g;
  a.n = oa.n;
  a.n_magic = oa.n >= 2 ? (unsigned)((1ull << 32) / (unsigned)oa.n) : 0u;
  a.colour = oa.colour;
  a.reverse = oa.reverse;
  a.e0 = oa.e0;
  a.zbuf = oa.zbuf;
  a.direct_interior = oa.direct_interior;
  if (Sc::GDIR && (gstride != Op::GEO || goff != 0)) return cudaErrorNotSupported;
  const int64_t count = (MODE == 0 || MODE >= 3) ? oa.E : oa.nlist;
  if (count <= 0) return cudaSuccess;
  const int64_t ntiles = (count + Op::NE - 1) / Op::NE;
  int64_t grid = (int64_t)oa.num_sms * c.occ;
  if (grid > ntiles) grid = ntiles;
  // SPHP_MAX_GRID caps the persistent grid (tests use it to make every CTA
  // walk many tiles on small meshes)
  static const int64_t max_grid = [] {
    const char* e = getenv("SPHP_MAX_GRID");
    return e ? (int64_t)atoll(e) : (int64_t)0;
  }();
  if (max_grid > 0 && grid > max_grid) grid = max_grid;
  kern<<<(unsigned)grid, Op::NT, Sc::SMEM_BYTES, s>>>(a);
  return cudaGetLastError();
}

// global geometry record (doubles per element) of each encoding
template <int DIM, int NPTS>
constexpr int64_t geom_record(int kind) {
  return kind == SPHP_GEOM_AFFINE ? (DIM == 3 ? 10 : 6)
         : kind == SPHP_GEOM_POINT ? (int64_t)(1 + DIM * DIM) * even_up(NPTS)
         : kind == SPHP_GEOM_METRIC ? (int64_t)(DIM * (DIM + 1) / 2 + 1) * even_up(NPTS)
                                     : 0;
}

template <class Op>
cudaError_t launch_mode(const OpArgs& oa, int64_t gstride, int64_t goff, cudaStream_t s) {
  switch (oa.mode) {
    case AsmMode::LOCAL:
      return launch_pipe<Op, 0>(oa, gstride, goff, s);
    case AsmMode::PERIODIC:
      return launch_pipe<Op, 1>(oa, gstride, goff, s);
    case AsmMode::EXPLICIT:
      return launch_pipe<Op, 2>(oa, gstride, goff, s);
    case AsmMode::PERIODIC_GATHER:
      return launch_pipe<Op, 3>(oa, gstride, goff, s);
    case AsmMode::EXPLICIT_GATHER:
      return launch_pipe<Op, 4>(oa, gstride, goff, s);
    case AsmMode::PERIODIC_CLASS:
      return cudaErrorNotSupported;  // Helmholtz only (hex_helm.cu: helm_class, MODE 5 / 6)
  }
  return cudaErrorInvalidValue;
}

// fast keys: (M, Q) with Q = M+1 (reference default) or M+2 (configs)
#define SPHP_HEX_KEYS(X) \
  X(2, 3) X(2, 4) X(3, 4) X(3, 5) X(4, 5) X(4, 6) X(5, 6) X(5, 7) X(6, 7) X(6, 8) X(7, 8) X(7, 9) \
      X(8, 9) X(8, 10) X(9, 10) X(9, 11)
#define SPHP_QUAD_KEYS(X) SPHP_HEX_KEYS(X) X(10, 11) X(10, 12)

}  // namespace sphp
