// Tile pipeline shared by every sum-factorisation kernel.
//
// A CTA owns NE elements per tile and walks tiles blockIdx.x, +gridDim.x, ...
// (persistent grid sized to the SM count).  Inputs for a tile — the packed
// element block (collections.py:316-323 layout) and the tile's geometric
// factors — are staged into shared memory by TMA bulk copies
// (cp.async.bulk, SASS UBLKCP) completing on an mbarrier, double-buffered so
// the copy of tile t+2G overlaps the compute of tile t.  Each Op releases its
// input stage as soon as it has read it for the last time (hooks.release()),
// so the next load starts mid-tile.  The Op writes its per-element results
// densely into a staging buffer that is streamed back with one bulk store
// (cp.async.bulk global<-shared) per tile.
//
// The assembled modes (PERIODIC / EXPLICIT) replace the input copy by a
// signed gather from the global vector and the store by a signed scatter-add
// (assembly.py:141-160) over one colour class: elements of one colour share
// no global dof, and colours run in a fixed order, so the sum is
// deterministic and needs no atomics.
#pragma once
#include "common.cuh"
#include "kernels.h"
#include "periodic.cuh"
#include "../../include/spechp_b200.h"

#ifndef SPHP_CLASS_MINB
#define SPHP_CLASS_MINB 0
#endif
namespace sphp {

__host__ __device__ constexpr int even_up(int x) { return (x + 1) & ~1; }

// ===========================================================================
// Element-block I/O of the fused Helmholtz ops (stages S1 / S9: rows
// (e, p, q) of M modes).  BlockIO: the packed element-major block
// (collections.py:316-323).  ClassIO: the tile staged by entity class
// (pipeline MODE 5, PERIODIC_CLASS): mode (p, q, r) of element e sits at
// (t & 0xffff) + e * (t >> 16) with t = tab[(p * M + q) * M + r]; along r
// the modes r >= 2 of a row are consecutive offsets of one entity, so a row
// costs three table loads.
// ===========================================================================
struct BlockIO {
  static constexpr bool DENSE = true;
};
// hook the ops call right after S1's barrier (the element block is dead)
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
template <bool PRE, int PV = 1>
struct ClassIO {
  static constexpr bool DENSE = false;
  const int* tab;  // PV tables of IN position words
  // PRE: every thread owns at most one (e, p, q) row of S1 / S9, the same
  // for every tile: its three positions are resolved once per kernel, for
  // each of the PV tile parities (odd NE: the 16-byte parity of the tile's
  // x ranges alternates with the tile)
  int p[PV][3] = {};
  int v = 0;  // this tile's parity variant
  int in_size = 0;
  __device__ __forceinline__ static int at(int t, int e) { return (t & 0xffff) + e * (t >> 16); }
  template <int M>
  __device__ __forceinline__ void resolve(int e, int pq, int& a0, int& a1, int& a2) const {
    const int vv = PV > 1 ? v : 0;
    if constexpr (PRE) {
      // selects, not a dynamic index (which would put p in local memory)
      a0 = (PV > 1 && vv) ? p[PV - 1][0] : p[0][0];
      a1 = (PV > 1 && vv) ? p[PV - 1][1] : p[0][1];
      a2 = (PV > 1 && vv) ? p[PV - 1][2] : p[0][2];
    } else {
      const int* tr = tab + vv * in_size + pq * M;
      a0 = at(tr[0], e), a1 = at(tr[1], e), a2 = at(tr[2], e);
    }
  }
  // The M - 2 bubble modes of a row are consecutive doubles of one entity,
  // and the rows of consecutive lanes (q, q + 1, ...) follow each other at
  // stride M - 2: for even M - 2 the lanes of a half-warp share bank pairs
  // (4-way at M = 6: ncu P=5, 11.0 M of this store's 13.6 M wavefronts were
  // excess).  ROT: each lane walks its tail in the order (it + s) mod (M - 2)
  // with s from the address bits above the bank index — lanes on the same
  // bank pair start at different modes — and a log2 chain of conditional
  // register rotations restores the order (TailRot below).
#ifndef SPHP_CLASS_ROT
#define SPHP_CLASS_ROT 1
#endif
  template <int N>
  struct TailRot {
    static constexpr int NV = (N % 16 == 0) ? 16 : (N % 8 == 0) ? 8 : (N % 4 == 0) ? 4 : (N % 2 == 0) ? 2 : 1;
    static constexpr bool ON = SPHP_CLASS_ROT && NV > 1 && N > 1;
    __device__ static __forceinline__ int shift(int a2) { return (a2 >> 4) & (NV - 1); }
    // x[r] <- x[(r + SH) % N] (LEFT) or x[(r - SH) mod N] where c
    template <int SH, bool LEFT>
    __device__ static __forceinline__ void rot_if(double* x, bool c) {
      double t[N];
#pragma unroll
      for (int r = 0; r < N; ++r) t[r] = LEFT ? x[(r + SH) % N] : x[(r - SH % N + N) % N];
#pragma unroll
      for (int r = 0; r < N; ++r) x[r] = c ? t[r] : x[r];
    }
    template <bool LEFT>
    __device__ static __forceinline__ void rot(double* x, int s) {
      if constexpr (NV > 1) rot_if<1 % N, LEFT>(x, s & 1);
      if constexpr (NV > 2) rot_if<2 % N, LEFT>(x, s & 2);
      if constexpr (NV > 4) rot_if<4 % N, LEFT>(x, s & 4);
      if constexpr (NV > 8) rot_if<8 % N, LEFT>(x, s & 8);
    }
  };
  template <int M>
  __device__ __forceinline__ void load_row(const double* __restrict__ base, int e, int pq, double* x) const {
    static_assert(M > 2, "class staging needs bubbles (P >= 2)");
    int a0, a1, a2;
    resolve<M>(e, pq, a0, a1, a2);
    x[0] = base[a0];
    x[1] = base[a1];
    using TR = TailRot<M - 2>;
    if constexpr (TR::ON) {
      const int s = TR::shift(a2);
      double t[M - 2];
#pragma unroll
      for (int it = 0; it < M - 2; ++it) {
        int r = it + s;
        r -= r >= M - 2 ? M - 2 : 0;
        t[it] = base[a2 + r];  // t[it] = tail[(it + s) % N]
      }
      TR::template rot<false>(t, s);  // tail[r] = t[(r - s) mod N]
#pragma unroll
      for (int r = 2; r < M; ++r) x[r] = t[r - 2];
    } else {
#pragma unroll
      for (int r = 2; r < M; ++r) x[r] = base[a2 + r - 2];
    }
  }
  template <int M>
  __device__ __forceinline__ void store_row(double* __restrict__ base, int e, int pq, const double* c) const {
    int a0, a1, a2;
    resolve<M>(e, pq, a0, a1, a2);
    base[a0] = c[0];
    base[a1] = c[1];
    using TR = TailRot<M - 2>;
    if constexpr (TR::ON) {
      const int s = TR::shift(a2);
      double t[M - 2];
#pragma unroll
      for (int r = 2; r < M; ++r) t[r - 2] = c[r];
      TR::template rot<true>(t, s);  // t[it] = tail[(it + s) % N]
#pragma unroll
      for (int it = 0; it < M - 2; ++it) {
        int r = it + s;
        r -= r >= M - 2 ? M - 2 : 0;
        base[a2 + r] = t[it];
      }
    } else {
#pragma unroll
      for (int r = 2; r < M; ++r) base[a2 + r - 2] = c[r];
    }
  }
};

// device view of the launch arguments (plain POD, passed by value)
struct DevArgs {
  int64_t E;
  const double* in;
  double* out;
  const double* geom;
  int64_t gstride;  // doubles per element in global geometry
  int64_t goff;     // first staged double inside an element's record
  double lam;
  int use_tma;
  // assembled
  const double* xg;
  double* yg;
  const int* elist;
  int64_t nlist;
  const int* codes;
  const int* ent_g;  // PERIODIC_GATHER: precomputed (E, 27) entity bases, or null
  int n;
  unsigned n_magic;  // floor(2^32 / n): division by n as a multiply (fast_divn)
  int colour;
  int reverse;  // MODE 0: walk the tiles last to first (L2 reuse, see launch)
  // MODE 5
  int64_t e0;        // absolute index of element 0 of this launch
  double* zbuf;      // class-major output block
  int direct_interior;
};


// x / n and x % n for 0 <= x < 2^31 with magic = floor(2^32 / n), n >= 2:
// umulhi(x, magic) is the quotient or one less (x (2^32 / n - magic) < 2^32),
// one correction step.  The class launch does this per tile in every thread.
__device__ __forceinline__ void fast_divn(int x, int n, unsigned magic, int& q, int& r) {
  q = (int)__umulhi((unsigned)x, magic);
  r = x - q * n;
  if (r >= n) {
    ++q;
    r -= n;
  }
}

// ---------------------------------------------------------------------------
// The scaffold.  Op supplies: M, NE, NT, IN, OUT, GEO (staged doubles per
// element), WORK (work doubles per element) and
//   template <class R, class W> static void compute(in, geo, work, out, lam,
//        R release, W pre_out, const double* tab)
// MODE 0: local (block in, block out).
// MODE 1: periodic hex, colour class: gather in, scatter-add out.
// MODE 2: explicit map, colour class: gather in, scatter-add out.
// MODE 3: periodic hex, all elements in order: gather in, local block out.
// MODE 4: explicit map, all elements in order: gather in, local block out.
// MODE 6: MODE 5 with the geometry read from global memory (L2 prefetch).
// MODE 7: MODE 0 with the geometry read from global memory (L2 prefetch).
// MODE 5: periodic hex, all elements in order, by entity class: the tile's
//         27 class ranges of x arrive by TMA bulk copies into a class-
//         staged input, results leave by 27 bulk stores into the class-major
//         block Z (interiors optionally straight into y).  Needs even NE,
//         n % NE == 0 and even n (then every copy's 16-byte parity is static).
// Gathering modes need IN == OUT == nmodes.
template <int MODE>
struct ModeTraits {
  static constexpr bool LOCAL = MODE == 0 || MODE == 7;
  static constexpr bool GATHER = !LOCAL;
  static constexpr bool PERIODIC = MODE == 1 || MODE == 3;
  static constexpr bool EXPLICIT = MODE == 2 || MODE == 4;
  static constexpr bool SCATTER = MODE == 1 || MODE == 2;
  static constexpr bool CONTIG = LOCAL || MODE >= 3;
  static constexpr bool CLASS = MODE == 5 || MODE == 6;
  // geometry read from global memory in the compute (L2-prefetched one tile
  // ahead) instead of staged in shared memory: MODE 6 (class), MODE 7 (local;
  // full tiles only, the launcher takes MODE 0 for a partial last tile)
  static constexpr bool GDIR = MODE == 6 || MODE == 7;
};
// ---------------------------------------------------------------------------
// preferred number of input stages: Op::NSTP when the Op declares it, else 1
// (measured: more resident CTAs beat a second stage, profiles/r01_tune.log)
template <class Op>
constexpr auto nst_pref_impl(int) -> decltype(Op::NSTP, int()) { return Op::NSTP; }
template <class Op>
constexpr int nst_pref_impl(...) { return 1; }
template <class Op>
constexpr int nst_pref() { return nst_pref_impl<Op>(0); }

// smem stride of one element's staged geometry: Op::GEO_S when the op pads
// it (bank spreading across elements), else GEO
template <class Op>
constexpr auto geo_s_impl(int) -> decltype(Op::GEO_S, int()) { return Op::GEO_S; }
template <class Op>
constexpr int geo_s_impl(...) { return Op::GEO; }

// an Op whose last stage leaves part of its work area free may stage the
// output block there (Op::OUT_OFF, doubles into the work area): one buffer
// fewer, which is what lets the P=4 Helmholtz tile fit four CTAs per SM
template <class Op>
constexpr auto out_off_impl(int) -> decltype(Op::OUT_OFF, int()) { return Op::OUT_OFF; }
template <class Op>
constexpr int out_off_impl(...) { return -1; }

// an Op whose compute() takes a geo_ready hook and calls it before its first
// read of the staged geometry (Op::GEO_HOOK): with one input stage the tile's
// geometry then completes on its own mbarrier, waited for at the pointwise
// stage instead of at the top of the tile — its copy has the first
// contraction stages to land
template <class Op>
constexpr auto geo_hook_impl(int) -> decltype(Op::GEO_HOOK, bool()) { return Op::GEO_HOOK; }
template <class Op>
constexpr bool geo_hook_impl(...) { return false; }

template <class Op, int MODE>
struct Scaffold {
  static constexpr int NE = Op::NE, NT = Op::NT;
  static constexpr bool CLS = ModeTraits<MODE>::CLASS;
  // MODE 5 stages each of the 27 classes in its own slot of NE * size + 2
  // doubles (room for the 16-byte widening of its copy window) rounded up
  // to even (16-byte aligned slots)
  static constexpr int IN_T = CLS ? even_up(NE * Op::IN + 3 * 27) : even_up(NE * Op::IN + 2);
  static constexpr int GEO_S = geo_s_impl<Op>(0);  // even, >= GEO
  // MODE 6 = MODE 5 reading the geometry straight from global memory in the
  // pointwise stage (prefetched into L2 one tile ahead) instead of staging
  // it: no shared-memory copy, more resident CTAs.  Only won at P = 2 with
  // the former skewed Q = 4 plan (0.209 -> 0.198 ms; P = 3..8 lose 10-35 %,
  // tools/time_phases.py); the i-column plan beats both (0.181 ms).  Today
  // MODE 6 serves the k-major K-row order P = 7 (hex_helm.cu: SPHP_CLASS_GDIR)
  static constexpr bool GDIR = ModeTraits<MODE>::GDIR;
  static constexpr int GEO_T = GDIR ? 0 : NE * GEO_S;
  static constexpr int STAGE = IN_T + GEO_T;
  static constexpr int OUT_OFF = out_off_impl<Op>(0);
  // block-input (MODE 0) ops stream the output block back with one TMA bulk
  // store per tile; the buffer is shifted by one double when the tile's
  // global start is odd so both ends share 16-byte alignment (an Op staging
  // it in its work area, OUT_OFF, leaves at least one spare double there)
#ifndef SPHP_NO_BULK_OUT
  static constexpr bool BULK_OUT = ModeTraits<MODE>::LOCAL;
#else
  static constexpr bool BULK_OUT = false;  // tuning build: plain store loop
#endif
  static constexpr int OUT_T = OUT_OFF >= 0 ? 0 : even_up(NE * Op::OUT + (BULK_OUT ? 2 : 0));
  static constexpr int WORK_T = even_up(NE * Op::WORK);
  // assembled-mode integer tables (in doubles): per stage ids + entities,
  // current-tile copies, and the per-mode code table
  static constexpr int ENT = ModeTraits<MODE>::PERIODIC ? 27 : 0;
  static constexpr int ITAB = (ModeTraits<MODE>::LOCAL || CLS) ? 0 : even_up(NE * (2 + ENT)) / 2 + 1;
  // MODE 5 int tables: per-mode input / output positions (2 * IN), per
  // class slot base, Z offset, geometry and first 16-byte chunk (5 * 27 + 1)
  // (PV tile-parity variants of the positions and of the chunk prefix)
  static constexpr int PV = (CLS && (NE & 1)) ? 2 : 1;
  static constexpr int MTAB = ModeTraits<MODE>::PERIODIC ? even_up(Op::IN) / 2 + 1
                              : CLS ? ((PV + PV) * Op::IN + 4 * 27 + PV * 28) / 2 + 1
                                    : 0;
  static constexpr size_t fixed_bytes(int nst) {
    return sizeof(double) * (nst * (STAGE + ITAB) + OUT_T + WORK_T + ITAB + MTAB) + 2 * sizeof(uint64_t);
  }
  // two input stages when they fit in 227 KB, else one (the next tile's copy
  // then overlaps only the part of the compute after the release point)
  static constexpr int NST = (nst_pref<Op>() == 2 && fixed_bytes(2) <= 227 * 1024) ? 2 : 1;
  static constexpr size_t SMEM_BYTES = fixed_bytes(NST);
  // CTAs per SM that shared memory allows (228 KB per SM, 1 KB reserved per
  // CTA)
  static constexpr int SMEM_CTAS = (int)(233472 / (SMEM_BYTES + 1024)) < 1 ? 1 : (int)(233472 / (SMEM_BYTES + 1024));
  static constexpr int MIN_CTAS = CLS ? SPHP_CLASS_MINB : 1;
#ifndef SPHP_NO_GEO_HOOK
  static constexpr bool GHOOK = geo_hook_impl<Op>(0) && NST == 1 && Op::GEO > 0 && !GDIR &&
                                (ModeTraits<MODE>::LOCAL || CLS);
#else
  static constexpr bool GHOOK = false;  // tuning build: geometry waited for at the top of the tile
#endif
};

template <class Op, int MODE>
__global__ void __launch_bounds__(Op::NT, (MODE == 5 ? Scaffold<Op, MODE>::MIN_CTAS : 0)) pipe_kernel(const DevArgs a) {
  using S = Scaffold<Op, MODE>;
  using MT = ModeTraits<MODE>;
  static_assert(S::SMEM_BYTES <= 227 * 1024, "one pipeline stage does not fit in shared memory");
  constexpr int NE = Op::NE, NT = Op::NT, IN = Op::IN, OUT = Op::OUT, GEO = Op::GEO;
  constexpr int GEO_S = S::GEO_S;
  constexpr int NST = S::NST, ENT = S::ENT;
  extern __shared__ __align__(128) double smem[];
  double* stage_base = smem;
  double* work = smem + NST * S::STAGE + S::OUT_T;
  double* out_s = S::OUT_OFF >= 0 ? work + (S::OUT_OFF >= 0 ? S::OUT_OFF : 0) : smem + NST * S::STAGE;
  // MODE 5 stages the tile's class-major results 16-byte aligned (an odd
  // OUT_OFF — odd element strides at odd Q with NE = 1 — moves it by one)
  double* out_c = out_s + (MT::CLASS ? (S::OUT_OFF & 1) : 0);
  int* itab = reinterpret_cast<int*>(work + S::WORK_T);      // NST stages of [ids NE | ent NE*27]
  int* icur = itab + NST * 2 * S::ITAB;                       // current tile copy
  int* mtab = icur + 2 * S::ITAB;                             // per-mode codes (MODE 1)
  uint64_t* bar = reinterpret_cast<uint64_t*>(mtab + 2 * S::MTAB);
  const int tid = threadIdx.x;

  const int64_t count = MT::CONTIG ? a.E : a.nlist;
  const int ntiles = (int)((count + NE - 1) / NE);
  const int G = gridDim.x;

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (MT::PERIODIC)
    for (int i = tid; i < IN; i += NT) mtab[i] = mode_code(Op::M, i);
  // MODE 5 tables: csb[k] = slot of class k in the input stage, ccb[k] =
  // offset of class k in an element's class-major record (sum of sizes),
  // cR / csd[k] = class geometry (region base; size | d << 16 | parity of
  // variant v << (20 + v)), cpre[v][k] = first 16-byte input chunk of class
  // k (cpre[v][27] = count).  Variant v = parity of the tile's first x: with
  // even NE and n it is always 0; with odd NE the classes of odd size start
  // at alternating 16-byte parities, and everything parity-dependent (slot
  // offsets, chunk lists, the interiors' staging shift) exists twice.
  constexpr int PV = S::PV;
  int* ptab = mtab;               // PV x IN: input position word per mode
  int* qtab = mtab + PV * IN;     // PV x IN: output position word per mode
  int* csb = qtab + PV * IN;      // 27
  int* ccb = csb + 27;            // 27
  int* cR = ccb + 27;             // 27
  int* csd = cR + 27;             // 27
  int* cpre = csd + 27;           // PV x 28
  constexpr int B3 = (Op::M - 2) * (Op::M - 2) * (Op::M - 2);
  if constexpr (MT::CLASS) {
    const int b = Op::M - 2;
    if (tid < 32) {  // lane k: class k, exclusive prefix sums by warp scan
      const int k = tid;
      int sz = 0, dx = 0, nch0 = 0, nch1 = 0;
      ClassGeom cg{0, 0, 0};
      if (k < 27) {
        cg = class_geom(k, a.n, Op::M - 1);
        sz = class_size(k, b);
        dx = class_dx(k);
        nch0 = (((sz & 1) & dx) + NE * sz + 1) / 2;
        nch1 = (((sz & 1) & (dx ^ 1)) + NE * sz + 1) / 2;
      }
      const int slot = k < 27 ? even_up(NE * sz + 2) : 0;
      int sb = slot, cb = sz, nc0 = nch0, nc1 = nch1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a1 = __shfl_up_sync(0xffffffffu, sb, o), a2 = __shfl_up_sync(0xffffffffu, cb, o),
                  a3 = __shfl_up_sync(0xffffffffu, nc0, o), a4 = __shfl_up_sync(0xffffffffu, nc1, o);
        if (k >= o) sb += a1, cb += a2, nc0 += a3, nc1 += a4;
      }
      if (k < 27) {
        csb[k] = sb - slot;
        ccb[k] = cb - sz;
        cR[k] = cg.R;
        csd[k] = sz | (cg.d << 16) | (((sz & 1) & dx) << 20) | (((sz & 1) & (dx ^ 1)) << 21);
        cpre[k] = nc0 - nch0;
        if (PV > 1) cpre[28 + k] = nc1 - nch1;
      }
      if (k == 26) {
        cpre[27] = nc0;
        if (PV > 1) cpre[28 + 27] = nc1;
      }
    }
    __syncthreads();
    for (int i = tid; i < IN; i += NT) {
      const int c = mode_code(Op::M, i), k = c & 31, off = c >> 5, sz = class_size(k, b);
      for (int v = 0; v < PV; ++v) {
        // 16-byte parity of the class's first value in variant v
        const int par = (sz & 1) & ((v + class_dx(k)) & 1);
        ptab[v * IN + i] = (csb[k] + par + off) | (sz << 16);
        // the interiors' staging is shifted to the parity of their y range
        const int sh = (k == 26) ? ((v * B3) & 1) : 0;
        qtab[v * IN + i] = (NE * ccb[k] + sh + off) | (sz << 16);
      }
    }
  }
  // MODE 5: this thread's input chunks c = tid + j * NT (j < CPT) of each
  // variant as class | slot offset << 5, resolved once (static lists)
  constexpr int CPT = MT::CLASS ? (NE * IN + 2 * 27 + 2 * NT - 1) / (2 * NT) : 1;
  int chunk[PV][CPT];
  if constexpr (MT::CLASS) {
#pragma unroll
    for (int v = 0; v < PV; ++v)
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int* cp = cpre + 28 * v;
        const int c = tid + j * NT;
        int k = 0;
        while (k < 26 && cp[k + 1] <= c) ++k;
        chunk[v][j] = c < cp[27] ? (k | ((2 * (c - cp[k])) << 5)) : -1;
      }
  }
  constexpr bool PRE = NE * Op::M * Op::M <= NT;
  ClassIO<PRE, PV> cin_io{ptab}, cout_io{qtab};
  cin_io.in_size = cout_io.in_size = IN;
  if constexpr (MT::CLASS && PRE) {
    __syncthreads();
    if (tid < NE * Op::M * Op::M) {
      const int e = tid / (Op::M * Op::M), pq = tid - e * (Op::M * Op::M);
#pragma unroll
      for (int v = 0; v < PV; ++v)
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          cin_io.p[v][r] = ClassIO<PRE, PV>::at(ptab[v * IN + pq * Op::M + r], e);
          cout_io.p[v][r] = ClassIO<PRE, PV>::at(qtab[v * IN + pq * Op::M + r], e);
        }
    }
  }
  __syncthreads();

  // ---- local mode: byte window of tile t's input block, widened to 16-byte
  // boundaries so one bulk copy moves it whatever the element size
  const int64_t in_total = count * (int64_t)IN * (int64_t)sizeof(double);
  auto in_window = [&](int t, int64_t& a0, int64_t& a1, int& off) -> bool {
    const int64_t w0 = (int64_t)t * NE;
    const int64_t r = (count - w0) < NE ? (count - w0) : NE;
    const int64_t s0 = w0 * IN * (int64_t)sizeof(double), s1 = (w0 + r) * IN * (int64_t)sizeof(double);
    a0 = s0 & ~(int64_t)15;
    a1 = (s1 + 15) & ~(int64_t)15;
    off = (int)((s0 - a0) / 8);
    return a.use_tma && a1 <= in_total;
  };

  // schedule slot -> tile (MODE 0 may walk the tiles in reverse)
  auto phys = [&](int ts) { return (MT::LOCAL && a.reverse) ? ntiles - 1 - ts : ts; };
  // thread 0: TMA bulk copies of the tile of schedule slot ts into stage s
  auto issue_local = [&](int ts, int s) {
    if (ts >= ntiles) return;
    const int t = phys(ts);
    double* in_s = stage_base + s * S::STAGE;
    double* geo_s = in_s + S::IN_T;
    const int64_t w0 = (int64_t)t * NE;
    const int r = (int)((count - w0) < NE ? (count - w0) : NE);
    int64_t a0, a1;
    int off;
    if (!in_window(t, a0, a1, off)) return;  // synchronous at consumption
    uint32_t bytes_in = (uint32_t)(a1 - a0);
    uint32_t bytes_g = (uint32_t)(sizeof(double) * r * GEO);
    if constexpr (S::GDIR) {
      mbar_expect_tx(&bar[s], bytes_in);
      bulk_g2s(in_s, reinterpret_cast<const char*>(a.in) + a0, bytes_in, &bar[s]);
      if (GEO > 0) bulk_prefetch_l2(a.geom + w0 * a.gstride, bytes_g);
      return;
    }
    uint64_t* gbar = S::GHOOK ? &bar[1] : &bar[s];  // GHOOK: NST == 1, bar[1] is the geometry's
    if constexpr (S::GHOOK) {
      mbar_expect_tx(&bar[s], bytes_in);
      mbar_expect_tx(gbar, bytes_g);
    } else {
      mbar_expect_tx(&bar[s], bytes_in + bytes_g);
    }
    bulk_g2s(in_s, reinterpret_cast<const char*>(a.in) + a0, bytes_in, &bar[s]);
    if (GEO > 0) {
      if (a.gstride == GEO && a.goff == 0 && GEO_S == GEO) {
        bulk_g2s(geo_s, a.geom + w0 * a.gstride, bytes_g, gbar);
      } else {
        for (int e = 0; e < r; ++e)
          bulk_g2s(geo_s + e * GEO_S, a.geom + (w0 + e) * a.gstride + a.goff,
                   (uint32_t)(sizeof(double) * GEO), gbar);
      }
    }
  };

  // all threads: element ids / entity bases, geometry TMA (thread 0) and the
  // signed gather as cp.async 8-byte copies (assembled modes).  Commits one
  // cp.async group per call, always.
  auto issue_asm = [&](int t, int s) {
    double* in_s = stage_base + s * S::STAGE;
    double* geo_s = in_s + S::IN_T;
    int* ids = itab + s * 2 * S::ITAB;
    int* ent = ids + NE;
    int* crd = ent + NE * ENT;
    const int64_t w0 = (int64_t)t * NE;
    const int r = (t < ntiles) ? (int)((count - w0) < NE ? (count - w0) : NE) : 0;
    if (MODE == 3 && a.ent_g != nullptr) {
      // all elements in order with a precomputed entity table: no index
      // set-up and no barrier — geometry by TMA (thread 0), x by cp.async
      if (tid == 0 && GEO > 0 && r > 0) {
        fence_proxy_async();
        const uint32_t bytes = (uint32_t)(sizeof(double) * r * GEO);
        mbar_expect_tx(&bar[s], bytes);
        if (a.gstride == GEO && a.goff == 0 && GEO_S == GEO) {
          bulk_g2s(geo_s, a.geom + w0 * a.gstride, bytes, &bar[s]);
        } else {
          for (int e = 0; e < r; ++e)
            bulk_g2s(geo_s + e * GEO_S, a.geom + (w0 + e) * a.gstride + a.goff,
                     (uint32_t)(sizeof(double) * GEO), &bar[s]);
        }
      }
      for (int i = tid; i < NE * IN; i += NT) {
        const int e = i / IN, nl = i - e * IN;
        if (e >= r) {
          in_s[i] = 0.0;
          continue;
        }
        const int c = mtab[nl];
        const int gid = __ldg(a.ent_g + (w0 + e) * 27 + (c & 31)) + (c >> 5);
        cp_async8(in_s + i, a.xg + gid);
      }
      cp_async_commit();
      return;
    }
    if (MT::PERIODIC) {
      // element coordinates once per element (packed 10 bits each, n <= 1024),
      // then the 27 entity bases per element
      const int h = a.n >> 1;
      for (int e = tid; e < NE; e += NT) {
        int packed = -1;
        if (e < r) {
          const int w = (int)(w0 + e);
          int ex, ey, ez;
          if (MODE == 1) {
            ex = 2 * (w % h) + (a.colour & 1);
            ey = 2 * ((w / h) % h) + ((a.colour >> 1) & 1);
            ez = 2 * (w / (h * h)) + ((a.colour >> 2) & 1);
          } else {
            ex = w % a.n;
            ey = (w / a.n) % a.n;
            ez = w / (a.n * a.n);
          }
          ids[e] = ex + a.n * (ey + a.n * ez);
          packed = ex | (ey << 10) | (ez << 20);
        }
        crd[e] = packed;
      }
      __syncthreads();
      for (int i = tid; i < NE * 27; i += NT) {
        const int e = i / 27, k = i - e * 27;
        const int c = crd[e];
        ent[i] = c < 0 ? 0 : entity_base(a.n, Op::M - 1, c & 1023, (c >> 10) & 1023, c >> 20, k);
      }
    } else if (MT::CONTIG) {
      for (int e = tid; e < NE; e += NT) ids[e] = (e < r) ? (int)(w0 + e) : -1;
    } else {
      for (int e = tid; e < NE; e += NT) ids[e] = (e < r) ? a.elist[w0 + e] : -1;
    }
    __syncthreads();
    if (tid == 0 && GEO > 0 && r > 0) {
      fence_proxy_async();
      mbar_expect_tx(&bar[s], (uint32_t)(sizeof(double) * r * GEO));
      for (int e = 0; e < r; ++e)
        bulk_g2s(geo_s + e * GEO_S, a.geom + (int64_t)ids[e] * a.gstride + a.goff,
                 (uint32_t)(sizeof(double) * GEO), &bar[s]);
    }
    for (int i = tid; i < NE * IN; i += NT) {
      const int e = i / IN, nl = i - e * IN;
      if (e >= r) {
        in_s[i] = 0.0;
        continue;
      }
      int gid;
      if (MT::PERIODIC) {
        const int c = mtab[nl];
        gid = ent[e * 27 + (c & 31)] + (c >> 5);
      } else {
        const int c = a.codes[(int64_t)ids[e] * IN + nl];
        gid = c >= 0 ? c : (c == -1 ? -1 : -c - 2);
      }
      if (gid >= 0)
        cp_async8(in_s + i, a.xg + gid);
      else
        in_s[i] = 0.0;
    }
    cp_async_commit();
  };

  // MODE 5 input, all threads: the tile's 27 class ranges of x as 16-byte
  // cp.async chunks into the class slots (every chunk's source and slot share
  // their static 16-byte parity).  At the row end the x-shifted classes wrap:
  // the last element's entity comes from x = 0 of the row, and since its
  // slot offset is even no chunk straddles the two pieces.  One cp.async
  // group per call.
  auto issue_x = [&](int ts) {
    if (ts < ntiles) {
      double* in_s = stage_base;
      const int w0 = (int)a.e0 + ts * NE;  // 32-bit: n^3 < 2^31
      const int n = a.n;
      int rowi, ex0, ez, ey;
      fast_divn(w0, n, a.n_magic, rowi, ex0);
      fast_divn(rowi, n, a.n_magic, ez, ey);
      const bool wrap = ex0 + NE == n;
      const int v = PV > 1 ? (ex0 & 1) : 0;
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int w = (PV > 1 && v) ? chunk[PV - 1][j] : chunk[0][j];
        if (w < 0) continue;
        const int k = w & 31, d = w >> 5;
        // volatile: keeps ptxas from hoisting these per-chunk constants out
        // of the tile loop (they would stay live through the pointwise stage)
        const int sd = ld_volatile_s32(csd + k), sz = sd & 0xffff, dx = (sd >> 16) & 1,
                  par = (sd >> (20 + v)) & 1;
        int y = ey + ((sd >> 17) & 1), z = ez + ((sd >> 18) & 1);
        y -= y >= n ? n : 0;
        z -= z >= n ? n : 0;
        const int rb = ld_volatile_s32(cR + k) + sz * n * (y + n * z);  // class region, this row
        const int plast = par + (NE - 1) * sz;        // slot offset of the last element
        const int src = (wrap && dx && d >= plast) ? rb + (d - plast) : rb + sz * (ex0 + dx) + d - par;
        cp_async16(in_s + ld_volatile_s32(csb + k) + d, a.xg + src);
      }
    }
    cp_async_commit();
  };
  // MODE 5 geometry, thread 0: one TMA bulk copy per tile
  auto issue_geo = [&](int ts, int s) {
    if (ts >= ntiles || GEO == 0) return;
    double* geo_s = stage_base + s * S::STAGE + S::IN_T;
    const int64_t w0 = a.e0 + (int64_t)ts * NE;
    if constexpr (S::GDIR) {
      bulk_prefetch_l2(a.geom + w0 * a.gstride, (uint32_t)(sizeof(double) * NE * GEO));
      return;
    }
    uint64_t* gbar = S::GHOOK ? &bar[1] : &bar[s];
    mbar_expect_tx(gbar, (uint32_t)(sizeof(double) * NE * GEO));
    if (a.gstride == GEO && a.goff == 0 && GEO_S == GEO) {
      bulk_g2s(geo_s, a.geom + w0 * a.gstride, (uint32_t)(sizeof(double) * NE * GEO), gbar);
    } else {
      for (int e = 0; e < NE; ++e)
        bulk_g2s(geo_s + e * GEO_S, a.geom + (w0 + e) * a.gstride + a.goff, (uint32_t)(sizeof(double) * GEO),
                 gbar);
    }
  };

  uint32_t phase = 0;  // bit s = parity to wait for on stage s
  if (MT::CLASS) {
    issue_x(blockIdx.x);
    if (tid == 0) issue_geo(blockIdx.x, 0);
  } else if (MT::LOCAL) {
    if (tid == 0) {
      issue_local(blockIdx.x, 0);
      if (NST == 2) issue_local(blockIdx.x + G, 1);
    }
  } else {
    issue_asm(blockIdx.x, 0);
    if (NST == 2) issue_asm(blockIdx.x + G, 1);
  }

  int it = 0;
  for (int ts = blockIdx.x; ts < ntiles; ts += G, ++it) {
    const int t = phys(ts);
    const int s = (NST == 2) ? (it & 1) : 0;
    double* in_s = stage_base + s * S::STAGE;
    double* geo_s = in_s + S::IN_T;
    const int64_t w0 = (int64_t)t * NE;
    const int r = (int)((count - w0) < NE ? (count - w0) : NE);

    // ---- obtain the tile's inputs -------------------------------------
    const double* in_p = in_s;
    bool geo_tma = MT::CLASS;  // GHOOK: this tile's geometry arrives on bar[1]
    if constexpr (MT::CLASS) {
      cp_async_wait<0>();
      if constexpr (!S::GDIR && !S::GHOOK) {
        mbar_wait(&bar[s], (phase >> s) & 1);
        phase ^= (1u << s);
      }
      // the previous tile's bulk stores must have read the output buffer
      if (tid == 0) bulk_wait_read0();
    } else if (MT::LOCAL) {
      int64_t a0, a1;
      int off;
      if (in_window(t, a0, a1, off)) {
        mbar_wait(&bar[s], (phase >> s) & 1);
        phase ^= (1u << s);
        in_p = in_s + off;
        geo_tma = true;
      } else {
        for (int i = tid; i < r * IN; i += NT) in_s[i] = a.in[w0 * IN + i];
        if constexpr (GEO > 0 && !S::GDIR) {
          for (int i = tid; i < r * GEO; i += NT) {
            int e = i / GEO, c = i - e * GEO;
            geo_s[e * GEO_S + c] = a.geom[(w0 + e) * a.gstride + a.goff + c];
          }
        }
      }
      // zero the unused tail of a partial tile (its results are discarded)
      for (int i = r * IN + tid; i < NE * IN; i += NT) in_s[(in_p - in_s) + i] = 0.0;
      if (GEO > 0 && !S::GDIR)
        for (int i = r * GEO_S + tid; i < NE * GEO_S; i += NT) geo_s[i] = 0.0;
      // the previous tile's bulk store must have read the output buffer
      if (S::BULK_OUT && tid == 0) bulk_wait_read0();
    } else {
      cp_async_wait<NST - 1>();
      if (GEO > 0) {
        mbar_wait(&bar[s], (phase >> s) & 1);
        phase ^= (1u << s);
      }
      const int* ids = itab + s * 2 * S::ITAB;
      if (MT::EXPLICIT) {  // sign -1 entries: negate the gathered value (own items)
        for (int i = tid; i < r * IN; i += NT) {
          const int e = i / IN, nl = i - e * IN;
          if (a.codes[(int64_t)ids[e] * IN + nl] <= -2) in_s[i] = -in_s[i];
        }
      }
      if (MT::SCATTER)
        for (int i = tid; i < NE * (1 + ENT); i += NT) icur[i] = ids[i];
      if (GEO > 0)
        for (int i = r * GEO_S + tid; i < NE * GEO_S; i += NT) geo_s[i] = 0.0;
    }
    __syncthreads();

    // ---- compute ---------------------------------------------------------
    auto release = [&]() {
      // all threads call this right after a __syncthreads that follows the
      // last read of the stage: hand the stage to the copy engines
      if (MT::CLASS) {
        if (tid == 0) {
          fence_proxy_async();
          issue_geo(ts + NST * G, s);
        }
      } else if (MT::LOCAL) {
        if (tid == 0) {
          fence_proxy_async();
          issue_local(ts + NST * G, s);
        }
      } else {
        issue_asm(ts + NST * G, s);
      }
    };
    auto pre_out = [&]() {};
    // GHOOK: all threads wait for the tile's geometry right before the
    // pointwise stage (bar[1], parity bit 1 of phase)
    auto geo_ready = [&]() {
      if constexpr (S::GHOOK) {
        if (geo_tma) {
          mbar_wait(&bar[1], (phase >> 1) & 1);
          phase ^= 2u;
        }
      }
    };
    const bool bulk_out = S::BULK_OUT && a.use_tma && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0;
    // out_t + i and a.out + w0 * OUT + i agree mod 16 bytes (the buffer
    // starts OUT_OFF doubles into the 16-byte aligned work area)
    const int head = bulk_out ? (int)((w0 * OUT) & 1) : 0;
    const int sh = bulk_out ? (head + (S::OUT_OFF > 0 ? S::OUT_OFF : 0)) & 1 : 0;
    double* out_t = out_s + sh;
    if constexpr (MT::CLASS) {
      // the class slots are free once S1 has read them: the next tile's x
      // chunks are issued right after S1 (all of S2..S9 to land)
      auto after_in = [&]() { issue_x(ts + G); };
      if constexpr (PV > 1) {
        int qv, rv;
        fast_divn((int)(a.e0 + w0), a.n, a.n_magic, qv, rv);
        const int v = rv & 1;  // parity of the tile's first x
        cin_io.v = cout_io.v = v;
      }
      const double* geo_p = S::GDIR ? a.geom + (a.e0 + w0) * a.gstride : geo_s;
      if constexpr (S::GHOOK)
        Op::compute(in_p, geo_p, work, out_c, a.lam, release, pre_out, c_tab, cin_io, cout_io, after_in, geo_ready);
      else
        Op::compute(in_p, geo_p, work, out_c, a.lam, release, pre_out, c_tab, cin_io, cout_io, after_in);
      fence_proxy_async();
    } else {
      const double* geo_p = S::GDIR ? a.geom + w0 * a.gstride : geo_s;
      if constexpr (S::GHOOK)
        Op::compute(in_p, geo_p, work, out_t, a.lam, release, pre_out, c_tab, BlockIO(), BlockIO(), NoHook(),
                    geo_ready);
      else
        Op::compute(in_p, geo_p, work, out_t, a.lam, release, pre_out, c_tab);
      if (bulk_out) fence_proxy_async();  // this thread's buffer writes -> async proxy
    }
    __syncthreads();

    // ---- write back ------------------------------------------------------
    if constexpr (MT::CLASS) {
      // the tile's results leave in TMA bulk stores: classes 0..25
      // (class-major within the tile) to its record of the tile-major block
      // Z (always 16-byte aligned: ZS is even), the interiors straight into
      // y (or after Z when accumulating); with odd NE and odd (P-1)^3 the
      // interiors' y range starts odd, so their staging is shifted to the
      // same parity (qtab) and the stores split into scalar head / bulk
      // body / scalar tail.  Thread stores when a base is not 16-byte
      // aligned (C-ABI callers may pass offset pointers); keeping that loop
      // in the kernel also keeps ptxas at ~100 registers (without it: ~150,
      // two CTAs per SM at P=4)
      constexpr int b = Op::M - 2, ZS = IN - b * b * b, B3 = b * b * b, NI = NE * B3;
      const int64_t wa = a.e0 + w0, N3 = (int64_t)a.n * a.n * a.n;
      const int sh = (int)((wa * B3) & 1);
      double* zdst = a.zbuf + wa * ZS;
      double* ybase = a.direct_interior ? a.yg + N3 * (1 + 3 * b + 3 * b * b) : a.zbuf + N3 * ZS;
      double* ydst = ybase + wa * B3;
      const double* isrc = out_c + NE * ZS + sh;
      if (((reinterpret_cast<uintptr_t>(zdst) | reinterpret_cast<uintptr_t>(ybase)) & 15) == 0) {
        if (tid == 0) {
          bulk_s2g(zdst, out_c, (uint32_t)(sizeof(double) * NE * ZS));
          const int body = (NI - sh) & ~1;
          if (sh) ydst[0] = isrc[0];
          if (body > 0) bulk_s2g(ydst + sh, isrc + sh, (uint32_t)(sizeof(double) * body));
          if (sh + body < NI) ydst[NI - 1] = isrc[NI - 1];
          bulk_commit();
        }
      } else {
        for (int i = tid; i < NE * IN; i += NT) {
          if (i < NE * ZS)
            zdst[i] = out_c[i];
          else
            ydst[i - NE * ZS] = isrc[i - NE * ZS];
        }
        __syncthreads();  // out_s is rewritten by the next tile
      }
    } else if (bulk_out) {
      const int n = r * OUT, body = (n - head) & ~1;
      double* dst = a.out + w0 * OUT;
      if (tid == 0) {
        if (body > 0) {
          bulk_s2g(dst + head, out_t + head, (uint32_t)(sizeof(double) * body));
          bulk_commit();
        }
        if (head) dst[0] = out_t[0];
      }
      if (tid == NT - 1 && head + body < n) dst[n - 1] = out_t[n - 1];
    } else if (!MT::SCATTER) {
      // element-major local block (a mode-major layout, coalesced for the
      // owner-computes sum, measured slower overall: profiles/r01_bench_*.log)
      for (int i = tid; i < r * OUT; i += NT) a.out[w0 * OUT + i] = out_s[i];
    } else {
      // signed scatter-add of one colour class: every global dof touched by
      // this launch belongs to exactly one element, so plain read-add-write
      // is race free; loads are batched ahead of the stores
      const int* ent = icur + NE;
      constexpr int U = 4;
      for (int i0 = tid; i0 < r * OUT; i0 += U * NT) {
        int g[U];
        double v[U], yv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + u * NT;
          g[u] = -1;
          v[u] = 0.0;
          if (i < r * OUT) {
            const int e = i / OUT, nl = i - e * OUT;
            if (MT::PERIODIC) {
              const int c = mtab[nl];
              g[u] = ent[e * 27 + (c & 31)] + (c >> 5);
              v[u] = out_s[i];
            } else {
              const int c = a.codes[(int64_t)icur[e] * OUT + nl];
              g[u] = c >= 0 ? c : (c == -1 ? -1 : -c - 2);
              v[u] = c >= 0 ? out_s[i] : -out_s[i];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) yv[u] = g[u] >= 0 ? a.yg[g[u]] : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (g[u] >= 0) a.yg[g[u]] = yv[u] + v[u];
      }
      // the next iteration overwrites icur (ids / entity bases) before its
      // first barrier: every thread must be done with this tile's indices
      __syncthreads();
    }
  }
  if (!MT::LOCAL) cp_async_wait<0>();
  if (S::BULK_OUT && tid == 0) bulk_wait0();
  if (MT::CLASS && tid == 0) bulk_wait0();
}

}  // namespace sphp
