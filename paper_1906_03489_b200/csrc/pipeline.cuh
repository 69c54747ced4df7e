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
#include "../../include/spechp_b200.h"

namespace sphp {

__host__ __device__ constexpr int even_up(int x) { return (x + 1) & ~1; }

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
  int n;
  int colour;
};

// periodic n^3 hex numbering (assembly.py:89-133 generalised; identical to
// oracle/assembly.py hex_periodic + build_map for uniform order P)
__device__ __forceinline__ int64_t hex_periodic_gid(int n, int P, int ex, int ey, int ez, int p,
                                                    int q, int r) {
  const int64_t N3 = (int64_t)n * n * n;
  const int64_t b = P - 1;
  int idx[3] = {p, q, r};
  int base[3] = {ex, ey, ez};
  int nb = (p >= 2) + (q >= 2) + (r >= 2);
  auto wrap = [n](int i) { return i >= n ? i - n : i; };
  if (nb == 0) {
    return wrap(ex + p) + (int64_t)n * (wrap(ey + q) + (int64_t)n * wrap(ez + r));
  }
  if (nb == 1) {
    int d = (p >= 2) ? 0 : ((q >= 2) ? 1 : 2);
    int c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) c[a] = wrap(base[a] + (a == d ? 0 : idx[a]));
    int64_t eid = d * N3 + c[0] + (int64_t)n * (c[1] + (int64_t)n * c[2]);
    return N3 + eid * b + (idx[d] - 2);
  }
  if (nb == 2) {
    int d = (p < 2) ? 0 : ((q < 2) ? 1 : 2);
    int c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) c[a] = wrap(base[a] + (a == d ? idx[a] : 0));
    int64_t fid = d * N3 + c[0] + (int64_t)n * (c[1] + (int64_t)n * c[2]);
    int k1 = (d == 0) ? q : p;
    int k2 = (d == 2) ? q : r;
    return N3 + 3 * N3 * b + fid * b * b + (k1 - 2) * b + (k2 - 2);
  }
  int64_t e = ex + (int64_t)n * (ey + (int64_t)n * ez);
  return N3 * (1 + 3 * b + 3 * b * b) + e * b * b * b + ((int64_t)(p - 2) * b + (q - 2)) * b + (r - 2);
}

// element of colour `colour` at list position w (n even): parity colouring
__device__ __forceinline__ void periodic_colour_elem(int n, int colour, int64_t w, int& ex, int& ey,
                                                     int& ez) {
  int h = n >> 1;
  ex = 2 * (int)(w % h) + (colour & 1);
  ey = 2 * (int)((w / h) % h) + ((colour >> 1) & 1);
  ez = 2 * (int)(w / ((int64_t)h * h)) + ((colour >> 2) & 1);
}

__device__ __forceinline__ void decode_code(int c, int64_t& gid, double& sgn) {
  if (c >= 0) {
    gid = c;
    sgn = 1.0;
  } else if (c == -1) {
    gid = -1;
    sgn = 0.0;
  } else {
    gid = -(int64_t)c - 2;
    sgn = -1.0;
  }
}

struct Hooks {
  // set by the scaffold
  int tile_next;  // tile to load into the released stage (or -1)
  int stage;
  bool released;
};

// ---------------------------------------------------------------------------
// The scaffold.  Op supplies: NE, NT, IN, OUT, GEO (staged doubles/element),
// WORK (work doubles/element), NMODE (dofs/element for assembled modes,
// i.e. IN == OUT == NMODE), and
//   template <class R, class W> static void compute(in_s, geo_s, work,
//        out_s, lam, R release, W pre_out)
// ---------------------------------------------------------------------------
template <class Op, int MODE>
struct Scaffold {
  static constexpr int NE = Op::NE, NT = Op::NT;
  static constexpr int IN_T = even_up(NE * Op::IN + 2);
  static constexpr int GEO_T = NE * Op::GEO;  // GEO is even
  static constexpr int STAGE = IN_T + GEO_T;
  static constexpr int OUT_T = even_up(NE * Op::OUT);
  static constexpr int WORK_T = even_up(NE * Op::WORK);
  // two input stages when they fit in 227 KB, else one (the next tile's copy
  // then overlaps only the part of the compute after the release point)
  static constexpr size_t BYTES2 = sizeof(double) * (2 * STAGE + OUT_T + WORK_T) + 2 * sizeof(uint64_t);
  static constexpr int NST = BYTES2 <= 227 * 1024 ? 2 : 1;
  static constexpr size_t SMEM_BYTES = sizeof(double) * (NST * STAGE + OUT_T + WORK_T) + 2 * sizeof(uint64_t);
  static_assert(SMEM_BYTES <= 227 * 1024, "one pipeline stage does not fit in shared memory");
};

template <class Op, int MODE>
__global__ void __launch_bounds__(Op::NT) pipe_kernel(const DevArgs a) {
  using S = Scaffold<Op, MODE>;
  constexpr int NE = Op::NE, NT = Op::NT, IN = Op::IN, OUT = Op::OUT, GEO = Op::GEO;
  extern __shared__ __align__(128) double smem[];
  double* stage_base = smem;
  constexpr int NST = S::NST;
  double* out_s = smem + NST * S::STAGE;
  double* work = out_s + S::OUT_T;
  uint64_t* bar = reinterpret_cast<uint64_t*>(work + S::WORK_T);
  const int tid = threadIdx.x;

  const int64_t count = (MODE == 0) ? a.E : a.nlist;
  const int ntiles = (int)((count + NE - 1) / NE);
  const int G = gridDim.x;

  // element id of list position w (assembled modes) / tile element (local)
  auto elem_of = [&](int64_t w, int& ex, int& ey, int& ez) -> int64_t {
    if (MODE == 1) {
      periodic_colour_elem(a.n, a.colour, w, ex, ey, ez);
      return ex + (int64_t)a.n * (ey + (int64_t)a.n * ez);
    } else if (MODE == 2) {
      return a.elist[w];
    }
    return w;
  };

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // byte window of tile t's input block, widened to 16-byte boundaries so a
  // single bulk copy can move it whatever the element size (the data then
  // starts 0 or 1 doubles into the stage buffer)
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

  // issue the asynchronous part of tile t's input into stage s (thread 0)
  auto issue = [&](int t, int s) {
    if (t >= ntiles) return;
    double* in_s = stage_base + s * S::STAGE;
    double* geo_s = in_s + S::IN_T;
    const int64_t w0 = (int64_t)t * NE;
    const int r = (int)((count - w0) < NE ? (count - w0) : NE);
    if (MODE == 0) {
      int64_t a0, a1;
      int off;
      if (!in_window(t, a0, a1, off)) return;  // synchronous at consumption
      uint32_t bytes_in = (uint32_t)(a1 - a0);
      uint32_t bytes_g = (uint32_t)(sizeof(double) * r * GEO);
      mbar_expect_tx(&bar[s], bytes_in + bytes_g);
      bulk_g2s(in_s, reinterpret_cast<const char*>(a.in) + a0, bytes_in, &bar[s]);
      if (GEO > 0) {
        if (a.gstride == GEO && a.goff == 0) {
          bulk_g2s(geo_s, a.geom + w0 * a.gstride, bytes_g, &bar[s]);
        } else {
          for (int e = 0; e < r; ++e)
            bulk_g2s(geo_s + e * GEO, a.geom + (w0 + e) * a.gstride + a.goff,
                     (uint32_t)(sizeof(double) * GEO), &bar[s]);
        }
      }
    } else {
      if (GEO == 0) return;
      mbar_expect_tx(&bar[s], (uint32_t)(sizeof(double) * r * GEO));
      for (int e = 0; e < r; ++e) {
        int ex, ey, ez;
        int64_t id = elem_of(w0 + e, ex, ey, ez);
        bulk_g2s(geo_s + e * GEO, a.geom + id * a.gstride + a.goff, (uint32_t)(sizeof(double) * GEO),
                 &bar[s]);
      }
    }
  };

  uint32_t phase = 0;  // bit s = parity to wait for on stage s
  if (tid == 0) {
    issue(blockIdx.x, 0);
    if (NST == 2) issue(blockIdx.x + G, 1);
  }

  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += G, ++it) {
    const int s = (NST == 2) ? (it & 1) : 0;
    double* in_s = stage_base + s * S::STAGE;
    double* geo_s = in_s + S::IN_T;
    const int64_t w0 = (int64_t)t * NE;
    const int r = (int)((count - w0) < NE ? (count - w0) : NE);

    // ---- obtain the tile's inputs -------------------------------------
    const double* in_p = in_s;
    if (MODE == 0) {
      int64_t a0, a1;
      int off;
      if (in_window(t, a0, a1, off)) {
        mbar_wait(&bar[s], (phase >> s) & 1);
        phase ^= (1u << s);
        in_p = in_s + off;
      } else {
        for (int i = tid; i < r * IN; i += NT) in_s[i] = a.in[w0 * IN + i];
        if constexpr (GEO > 0) {
          for (int i = tid; i < r * GEO; i += NT) {
            int e = i / GEO, c = i - e * GEO;
            geo_s[i] = a.geom[(w0 + e) * a.gstride + a.goff + c];
          }
        }
      }
      // zero the unused tail of a partial tile (its results are discarded)
      for (int i = r * IN + tid; i < NE * IN; i += NT) in_s[(in_p - in_s) + i] = 0.0;
      if (GEO > 0)
        for (int i = r * GEO + tid; i < NE * GEO; i += NT) geo_s[i] = 0.0;
    } else {
      if (GEO > 0) {
        mbar_wait(&bar[s], (phase >> s) & 1);
        phase ^= (1u << s);
      }
      // signed gather (assembly.py:150-160)
      for (int i = tid; i < NE * IN; i += NT) {
        int e = i / IN, nl = i - e * IN;
        double v = 0.0;
        if (e < r) {
          int ex, ey, ez;
          int64_t id = elem_of(w0 + e, ex, ey, ez);
          if (MODE == 1) {
            int p = nl / (Op::M * Op::M), q = (nl / Op::M) % Op::M, rr = nl % Op::M;
            v = a.xg[hex_periodic_gid(a.n, Op::M - 1, ex, ey, ez, p, q, rr)];
          } else {
            int64_t gid;
            double sg;
            decode_code(a.codes[id * IN + nl], gid, sg);
            v = (gid >= 0) ? sg * a.xg[gid] : 0.0;
          }
        }
        in_s[i] = v;
      }
      if (GEO > 0)
        for (int i = r * GEO + tid; i < NE * GEO; i += NT) geo_s[i] = 0.0;
    }
    __syncthreads();

    // ---- compute ---------------------------------------------------------
    auto release = [&]() {
      // all threads call this right after a __syncthreads that follows the
      // last read of the stage: hand the stage to the copy engine
      if (tid == 0) {
        fence_proxy_async();
        issue(t + NST * G, s);
      }
    };
    auto pre_out = [&]() {};
    Op::compute(in_p, geo_s, work, out_s, a.lam, release, pre_out, c_tab);
    __syncthreads();

    // ---- write back ------------------------------------------------------
    if (MODE == 0) {
      for (int i = tid; i < r * OUT; i += NT) a.out[w0 * OUT + i] = out_s[i];
    } else {
      // signed scatter-add of one colour class: exclusive ownership
      for (int i = tid; i < r * OUT; i += NT) {
        int e = i / OUT, nl = i - e * OUT;
        int ex, ey, ez;
        int64_t id = elem_of(w0 + e, ex, ey, ez);
        if (MODE == 1) {
          int p = nl / (Op::M * Op::M), q = (nl / Op::M) % Op::M, rr = nl % Op::M;
          int64_t gid = hex_periodic_gid(a.n, Op::M - 1, ex, ey, ez, p, q, rr);
          a.yg[gid] += out_s[i];
        } else {
          int64_t gid;
          double sg;
          decode_code(a.codes[id * OUT + nl], gid, sg);
          if (gid >= 0) a.yg[gid] += sg * out_s[i];
        }
      }
    }
  }
}

}  // namespace sphp
