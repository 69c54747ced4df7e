// Hexahedral sum-factorisation operators (the 3D generalisation of
// collections.py:133-185 and geometry.py:145-184).
//
// Per-element layouts (first direction slowest, stdregions.py:1-14):
//   coefficients c[(p*M + q)*M + r], points u[(i*Q + j)*Q + k].
// Shared-memory work tensors use an odd row pitch QK = Q|1 in the fastest
// direction so pencil reads along k are bank-conflict free for FP64.
//
// Tables (B, Bd = dB/dxi, D, w) are read from __constant__ memory with
// compile-time indices (c_tab must be declared by the including TU).
#pragma once
#include <type_traits>

#ifndef SPHP_JEO_S5_BYCOMP
#define SPHP_JEO_S5_BYCOMP 1  // 0 (tuning): J-pencil plan's pointwise stage point by point (P=6: 1.506 vs 1.488 ms local, 1.745 vs 1.688 assembled)
#endif
#ifndef SPHP_GDIR_LOCAL
#define SPHP_GDIR_LOCAL 1  // tuning: 0 = k-major orders still stage their geometry (MODE 0)
#endif
#ifndef SPHP_SI_Q
#define SPHP_SI_Q 0  // tuning: another Q with the padded dense plane pitch
#endif

#include "pipeline.cuh"
#include "eo.cuh"

namespace sphp {

__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
// smallest v >= lo with v = Q (mod 16)
__host__ __device__ constexpr int pitch_mod16(int lo, int Q) {
  int v = lo;
  while (v % 16 != Q % 16) ++v;
  return v;
}

// per-element geometry record sizes (see sphp_geom_stride)
__host__ __device__ constexpr int pt_stride(int npts) { return even_up(npts); }

// work-item loop: items are distributed over the CTA's NT threads
#define SPHP_FOR_ITEMS(NITEMS, w) for (int w = threadIdx.x; w < (NITEMS); w += NT)

// ---------------------------------------------------------------------------
// contiguous row helpers: Q doubles at a 16-byte aligned address move as
// LDS.128 / STS.128 when Q is even (row stride Q then makes 8-lane phases
// bank-conflict free), as scalar accesses otherwise (odd stride: also free)
// ---------------------------------------------------------------------------
template <int Q>
__device__ __forceinline__ void load_row(const double* __restrict__ p, double* x) {
  if constexpr (Q % 2 == 0) {
    const double2* v = reinterpret_cast<const double2*>(p);
#pragma unroll
    for (int h = 0; h < Q / 2; ++h) {
      const double2 t = v[h];
      x[2 * h] = t.x;
      x[2 * h + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < Q; ++k) x[k] = p[k];
  }
}
template <int Q>
__device__ __forceinline__ void store_row(double* __restrict__ p, const double* x) {
  if constexpr (Q % 2 == 0) {
    double2* v = reinterpret_cast<double2*>(p);
#pragma unroll
    for (int h = 0; h < Q / 2; ++h) v[h] = make_double2(x[2 * h], x[2 * h + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < Q; ++k) p[k] = x[k];
  }
}


// ---------------------------------------------------------------------------
// Element-block rows (M contiguous doubles, one lane per row R of the tile):
// lane R hits bank R*M + r.  For even M consecutive rows share banks (4-way
// at M = 4, 8-way at M = 8 in the Helmholtz S1/S9 stages).  Reading /
// writing the row in the order r = (it + s) mod M with s = (R / PER) & MASK,
// PER = 16 / gcd(M, 16), makes the 16 lanes of a half-warp distinct; the
// registers are put back in order by log2(MASK + 1) conditional rotations.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int gcd16(int m) { return (m % 16 == 0) ? 16 : (m % 8 == 0) ? 8 : (m % 4 == 0) ? 4 : (m % 2 == 0) ? 2 : 1; }
template <int M>
struct RowRot {
  static constexpr int PER = 16 / gcd16(M);
  static constexpr int NV = 16 / PER;  // distinct rotations needed in a half-warp
  static constexpr int MASK = NV - 1;  // NV is 1, 2, 4, 8 or 16 (<= M for M in 2..10)
  __device__ static __forceinline__ int shift(int R) { return (R / PER) & MASK; }
  // y[r] = x[(r + SH) % M] where the bit is set
  template <int SH>
  __device__ static __forceinline__ void rotl_if(double* x, bool c) {
    double t[M];
#pragma unroll
    for (int r = 0; r < M; ++r) t[r] = x[(r + SH) % M];
#pragma unroll
    for (int r = 0; r < M; ++r) x[r] = c ? t[r] : x[r];
  }
  // x <- rotate left by s (x[r] = old[(r + s) % M]), s in [0, NV)
  __device__ static __forceinline__ void rotl(double* x, int s) {
    if constexpr (NV > 1) rotl_if<1 % M>(x, s & 1);
    if constexpr (NV > 2) rotl_if<2 % M>(x, s & 2);
    if constexpr (NV > 4) rotl_if<4 % M>(x, s & 4);
    if constexpr (NV > 8) rotl_if<8 % M>(x, s & 8);
  }
  template <int SH>
  __device__ static __forceinline__ void rotr_if(double* x, bool c) {
    double t[M];
#pragma unroll
    for (int r = 0; r < M; ++r) t[r] = x[(r - SH % M + M) % M];
#pragma unroll
    for (int r = 0; r < M; ++r) x[r] = c ? t[r] : x[r];
  }
  __device__ static __forceinline__ void rotr(double* x, int s) {
    if constexpr (NV > 1) rotr_if<1>(x, s & 1);
    if constexpr (NV > 2) rotr_if<2>(x, s & 2);
    if constexpr (NV > 4) rotr_if<4>(x, s & 4);
    if constexpr (NV > 8) rotr_if<8>(x, s & 8);
  }
  // p[(it + s) % M] = c[(it + s) % M]: stores in rotated order
  __device__ static __forceinline__ void store(double* __restrict__ p, int R, const double* c) {
    if constexpr (NV == 1) {
#pragma unroll
      for (int r = 0; r < M; ++r) p[r] = c[r];
    } else {
      const int s = shift(R);
      double cr[M];
#pragma unroll
      for (int r = 0; r < M; ++r) cr[r] = c[r];
      rotl(cr, s);  // cr[it] = c[(it + s) % M]
#pragma unroll
      for (int it = 0; it < M; ++it) {
        int r = it + s;
        r -= r >= M ? M : 0;
        p[r] = cr[it];
      }
    }
  }
  __device__ static __forceinline__ void load(const double* __restrict__ p, int R, double* x) {
    if constexpr (NV == 1) {
#pragma unroll
      for (int r = 0; r < M; ++r) x[r] = p[r];
    } else {
      const int s = shift(R);
      double xr[M];
#pragma unroll
      for (int it = 0; it < M; ++it) {
        int r = it + s;
        r -= r >= M ? M : 0;
        xr[it] = p[r];  // xr[it] = x[(it + s) % M]
      }
      // x[r] = xr[(r - s) mod M]: undo the left rotation by s
      rotr(xr, s);
#pragma unroll
      for (int r = 0; r < M; ++r) x[r] = xr[r];
    }
  }
};


// ===========================================================================
// Fused matrix-free Helmholtz (K4): y = sum_ab B_a^T G_ab B_b uhat + lam B^T wJ B uhat
// (geometry.py:171-184 as one sum-factorised pass; no quadrature data
// leaves shared memory).  GK: SPHP_GEOM_METRIC (7 per-point comps, point
// order (i,j,k)) or SPHP_GEOM_AFFINE (det, inv per element).
//
// Stages (m = M modes, Q points per direction; e = element of the tile):
//   S1 r->k   c[p,q,r]  -> T1[p,q,k]            pencils (p,q)
//   S2 q->j   T1        -> T2[p,j,k]            pencils (p,k)
//   S3 p->i   T2        -> u, d0 = d/dxi0 u     pencils (j,k)   (dense Q^3)
//   S4 j      u         -> d1                   pencils (i,k)
//   S5 k      row (i,j): d2 = D u in registers, f = G grad u, mass term,
//             t = lam wJ u + D2^T f2; writes t, f0, f1 (contiguous rows,
//             128-bit accesses, geometry rows read straight from the stage)
//   S6 j      t += D1^T f1                      pencils (i,k)
//   S7 i->p   T2'[p,j,k] = B t + dB f0          pencils (j,k)
//   S8 j->q, S9 k->r    -> y[p,q,r]
// ===========================================================================

// ===========================================================================
// Fused Helmholtz, K-row plan (HexHelmEO): the stages above, every 1D
// contraction evaluated through eo.cuh (half the DFMAs and table loads of
// the plain pencil form).
// ===========================================================================
template <int M_, int Q_, int GK, int NE_, int NT_, int NSTP_ = 2>
struct HexHelmEO {
  static constexpr int M = M_, Q = Q_, NE = NE_, NT = NT_;
  static constexpr int NSTP = NSTP_;
  static constexpr bool GEO_HOOK = true;  // compute() calls geo_ready() before its first geometry read
  static constexpr int M3 = M * M * M, Q3 = Q * Q * Q;
  static constexpr int IN = M3, OUT = M3;
  static constexpr int CS = pt_stride(Q3);
  static constexpr int GEO = (GK == SPHP_GEOM_METRIC) ? 7 * CS : 10;
  static constexpr int QK = odd_up(Q);
  // pitches = Q (mod 16): the (p, k) lanes of the j-pencil stages land on
  // consecutive banks
  static constexpr int PP1 = pitch_mod16(M * QK, Q);
  static constexpr int PP2 = pitch_mod16(Q * Q, Q);
  // plane pitch of the dense (i, j, k) work tensors: Q^2 (contiguous), except
  // Q = 10 where Q^2 = 4 mod 16 puts the j-pencil lanes (i, k) on banks
  // 4i + k (ncu P=8: 105 M of 144 M excess wavefronts); SI = Q mod 16 makes
  // them consecutive while the 128-bit k-rows stay conflict free but for the
  // phases that cross an i.  Measured: P=8 3.341 -> 3.256 ms.  (Odd Q: the
  // scalar k-rows would conflict instead.)
  static constexpr int SI = (Q == 10 || Q == SPHP_SI_Q) ? pitch_mod16(Q * Q, Q) : Q * Q;
  // W2 (d0 / f0) never meets a j-pencil: it keeps the contiguous pitch, so
  // its k-rows stay conflict free (wavefront model: -10 % on these accesses)
  static constexpr int SI2 = Q * Q;
  static constexpr int SE = even_up(cmax(Q * SI, cmax(M * PP1, M * PP2)));
  static_assert(SE >= Q * SI && SE >= M * PP1 && SE >= M * PP2, "element tensors overlap");
  static_assert(Q % 2 == 1 || SE % 2 == 0, "128-bit rows need an even element stride");
  static constexpr int WORK = 3 * SE;
  static constexpr int OUT_OFF = NE * SE;  // S9 writes the block into W1 (free after S8)
  // (j-pencil stages S4/S6 in a rotated order per lane: modelled fewer
  // wavefronts, measured slower at Q = 10 — P=8 3.34 -> 3.66 ms, the rotation
  // selects cost more than the conflicts; natural order)
  // k-major METRIC points (metric_slot): the local operator then reads the
  // geometry from global memory (pipeline MODE 7) instead of staging it
  static constexpr bool KMAJ = GK == SPHP_GEOM_METRIC && metric_kmajor(Q);
  static constexpr bool GDIR_LOCAL = KMAJ && SPHP_GDIR_LOCAL;
  using T = Tab<M, Q>;
  using X = EO<M, Q>;

  template <class R, class W, class IO = BlockIO, class H = NoHook, class GH = NoHook>
  __device__ static void compute(const double* __restrict__ cin, const double* __restrict__ geo,
                                 double* __restrict__ work, double* __restrict__ out, double lam,
                                 R release, W pre_out, const double* tab, IO io = IO(),
                                 IO oio = IO(), H after_in = H(), GH geo_ready = GH()) {
    double* W0 = work;
    double* W1 = work + NE * SE;
    double* W2 = work + 2 * NE * SE;
    // S1: r -> k
    SPHP_FOR_ITEMS(NE * M * M, w) {
      int e = w / (M * M), pq = w - e * (M * M), p = pq / M, q = pq - p * M;
      double x[M], u[Q];
      if constexpr (IO::DENSE)
        RowRot<M>::load(cin + e * M3 + pq * M, w, x);
      else
        io.template load_row<M>(cin, e, pq, x);
      X::interp(tab, x, u);
      st_pencil<Q, 1>(W0 + e * SE + p * PP1 + q * QK, u);
    }
    __syncthreads();
    after_in();
    // S2: q -> j
    SPHP_FOR_ITEMS(NE * M * Q, w) {
      int e = w / (M * Q), rem = w - e * (M * Q), p = rem / Q, k = rem - p * Q;
      double x[M], u[Q];
      ld_pencil<M, QK>(W0 + e * SE + p * PP1 + k, x);
      X::interp(tab, x, u);
      st_pencil<Q, Q>(W1 + e * SE + p * PP2 + k, u);
    }
    __syncthreads();
    // S3: p -> i, u and d0
    SPHP_FOR_ITEMS(NE * Q * Q, w) {
      int e = w / (Q * Q), jk = w - e * (Q * Q);
      double x[M], u[Q], d[Q];
      ld_pencil<M, PP2>(W1 + e * SE + jk, x);
      X::interp_and_deriv(tab, x, u, d);
      st_pencil<Q, SI>(W0 + e * SE + jk, u);
      st_pencil<Q, SI2>(W2 + e * SE + jk, d);
    }
    __syncthreads();
    // S4: d1 = D along j
    SPHP_FOR_ITEMS(NE * Q * Q, w) {
      const int e = w / (Q * Q), ik = w - e * (Q * Q), i = ik / Q, k = ik - i * Q;
      double v[Q], r[Q];
      ld_pencil<Q, Q>(W0 + e * SE + i * SI + k, v);
      X::template deriv<false, false>(tab, v, r);
      st_pencil<Q, Q>(W1 + e * SE + i * SI + k, r);
    }
    __syncthreads();
    geo_ready();  // the staged geometry is first read here (pipeline: GEO_HOOK)
    // S5: k rows
    SPHP_FOR_ITEMS(NE * Q * Q, w) {
      int e = w / (Q * Q), ij = w - e * (Q * Q), i = ij / Q, j = ij - i * Q;
      const int row = e * SE + i * SI + j * Q;
      const int row2 = e * SE + i * SI2 + j * Q;
      double u[Q], d[Q], f0[Q], f1[Q], f2[Q], g[Q], d2[Q];
      load_row<Q>(W0 + row, u);
      X::template deriv<false, false>(tab, u, d2);
      if constexpr (GK == SPHP_GEOM_METRIC) {
        // the (i, j) row of metric component c: contiguous in point order, or
        // one value per k plane (k-major, metric_slot): lanes on consecutive
        // (i, j) then read consecutive doubles (coalesced from global memory)
        const double* gr = geo + e * GEO + (KMAJ ? ij : ij * Q);
        auto geo_row = [&](int c, double* x) {
          if constexpr (KMAJ) {
#pragma unroll
            for (int k = 0; k < Q; ++k) x[k] = gr[c * CS + k * Q * Q];
          } else {
            load_row<Q>(gr + c * CS, x);
          }
        };
        load_row<Q>(W2 + row2, d);
        geo_row(0, g);
#pragma unroll
        for (int k = 0; k < Q; ++k) f0[k] = g[k] * d[k];
        geo_row(1, g);
#pragma unroll
        for (int k = 0; k < Q; ++k) f1[k] = g[k] * d[k];
        double h[Q];
        load_row<Q>(W1 + row, h);
#pragma unroll
        for (int k = 0; k < Q; ++k) f0[k] = fma(g[k], h[k], f0[k]);
        geo_row(2, g);
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          f2[k] = g[k] * d[k];
          f0[k] = fma(g[k], d2[k], f0[k]);
        }
        geo_row(3, g);
#pragma unroll
        for (int k = 0; k < Q; ++k) f1[k] = fma(g[k], h[k], f1[k]);
        geo_row(4, g);
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          f1[k] = fma(g[k], d2[k], f1[k]);
          f2[k] = fma(g[k], h[k], f2[k]);
        }
        geo_row(5, g);
#pragma unroll
        for (int k = 0; k < Q; ++k) f2[k] = fma(g[k], d2[k], f2[k]);
        geo_row(6, g);
#pragma unroll
        for (int k = 0; k < Q; ++k) u[k] = lam * g[k] * u[k];
      } else {
        const double* gg = geo + e * GEO;
        const double det = gg[0];
        const double* iv = gg + 1;
        const double a00 = det * (iv[0] * iv[0] + iv[1] * iv[1] + iv[2] * iv[2]);
        const double a01 = det * (iv[0] * iv[3] + iv[1] * iv[4] + iv[2] * iv[5]);
        const double a02 = det * (iv[0] * iv[6] + iv[1] * iv[7] + iv[2] * iv[8]);
        const double a11 = det * (iv[3] * iv[3] + iv[4] * iv[4] + iv[5] * iv[5]);
        const double a12 = det * (iv[3] * iv[6] + iv[4] * iv[7] + iv[5] * iv[8]);
        const double a22 = det * (iv[6] * iv[6] + iv[7] * iv[7] + iv[8] * iv[8]);
        const double wij = tab[T::W + i] * tab[T::W + j];
        load_row<Q>(W2 + row2, d);
        double h[Q];
        load_row<Q>(W1 + row, h);
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          const double wq = wij * tab[T::W + k];
          f0[k] = wq * (a00 * d[k] + a01 * h[k] + a02 * d2[k]);
          f1[k] = wq * (a01 * d[k] + a11 * h[k] + a12 * d2[k]);
          f2[k] = wq * (a02 * d[k] + a12 * h[k] + a22 * d2[k]);
          u[k] = lam * (wq * det) * u[k];
        }
      }
      X::template deriv<true, true>(tab, f2, u);  // t = mass + D2^T f2
      store_row<Q>(W0 + row, u);
      store_row<Q>(W2 + row2, f0);
      store_row<Q>(W1 + row, f1);
    }
    __syncthreads();
    release();
    // S6: t += D1^T f1 along j
    SPHP_FOR_ITEMS(NE * Q * Q, w) {
      const int e = w / (Q * Q), ik = w - e * (Q * Q), i = ik / Q, k = ik - i * Q;
      double f[Q], t[Q];
      ld_pencil<Q, Q>(W1 + e * SE + i * SI + k, f);
      ld_pencil<Q, Q>(W0 + e * SE + i * SI + k, t);
      X::template deriv<true, true>(tab, f, t);
      st_pencil<Q, Q>(W0 + e * SE + i * SI + k, t);
    }
    __syncthreads();
    // S7: i -> p, B t + dB f0
    SPHP_FOR_ITEMS(NE * Q * Q, w) {
      int e = w / (Q * Q), jk = w - e * (Q * Q);
      double t[Q], f0[Q], c[M];
      ld_pencil<Q, SI>(W0 + e * SE + jk, t);
      ld_pencil<Q, SI2>(W2 + e * SE + jk, f0);
      X::project2(tab, t, f0, c);
      st_pencil<M, PP2>(W1 + e * SE + jk, c);
    }
    __syncthreads();
    // S8: j -> q
    SPHP_FOR_ITEMS(NE * M * Q, w) {
      int e = w / (M * Q), rem = w - e * (M * Q), p = rem / Q, k = rem - p * Q;
      double v[Q], c[M];
      ld_pencil<Q, Q>(W1 + e * SE + p * PP2 + k, v);
      X::project(tab, v, c);
      st_pencil<M, QK>(W0 + e * SE + p * PP1 + k, c);
    }
    pre_out();
    __syncthreads();
    // S9: k -> r
    SPHP_FOR_ITEMS(NE * M * M, w) {
      int e = w / (M * M), pq = w - e * (M * M), p = pq / M, q = pq - p * M;
      double v[Q], c[M];
      ld_pencil<Q, 1>(W0 + e * SE + p * PP1 + q * QK, v);
      X::project(tab, v, c);
      if constexpr (IO::DENSE)
        RowRot<M>::store(out + e * M3 + pq * M, w, c);
      else
        oio.template store_row<M>(out, e, pq, c);
    }
  }
};

// ===========================================================================
// Fused Helmholtz, J-pencil plan with even-odd contractions (Q % 4 == 0,
// where contiguous k-rows of Q doubles would map every 128-bit access of an
// 8-lane phase to two bank groups): the pointwise stage runs on pencils
// along j; 1D contractions through eo.cuh.
// ===========================================================================
template <int M_, int Q_, int GK, int NE_, int NT_, int NSTP_ = 2>
struct HexHelmJEO {
  static constexpr int M = M_, Q = Q_, NE = NE_, NT = NT_;
  static constexpr int NSTP = NSTP_;
  static constexpr bool GEO_HOOK = true;  // compute() calls geo_ready() before its first geometry read
  static constexpr int M3 = M * M * M, Q3 = Q * Q * Q;
  static constexpr int IN = M3, OUT = M3;
  static constexpr int CS = pt_stride(Q3);
  static constexpr int GEO = (GK == SPHP_GEOM_METRIC) ? 7 * CS : 10;
  static constexpr int QK = odd_up(Q);
  static constexpr int SW = odd_up(Q * Q * QK);
  static constexpr int WORK = 3 * SW;
  static constexpr int OUT_OFF = NE * SW;  // the last stage writes the block into W1 (free)
  using T = Tab<M, Q>;
  using X = EO<M, Q>;

  template <class R, class W, class IO = BlockIO, class H = NoHook, class GH = NoHook>
  __device__ static void compute(const double* __restrict__ cin, const double* __restrict__ geo,
                                 double* __restrict__ work, double* __restrict__ out, double lam,
                                 R release, W pre_out, const double* tab, IO io = IO(),
                                 IO oio = IO(), H after_in = H(), GH geo_ready = GH()) {
    double* W0 = work;
    double* W1 = work + NE * SW;
    double* W2 = work + 2 * NE * SW;
    SPHP_FOR_ITEMS(NE * M * M, w) {  // S1 r -> k
      int e = w / (M * M), pq = w - e * (M * M);
      double x[M], u[Q];
      if constexpr (IO::DENSE)
        ld_pencil<M, 1>(cin + e * M3 + pq * M, x);
      else
        io.template load_row<M>(cin, e, pq, x);
      X::interp(tab, x, u);
      st_pencil<Q, 1>(W0 + e * SW + pq * QK, u);
    }
    __syncthreads();
    after_in();
    SPHP_FOR_ITEMS(NE * M * Q, w) {  // S2 q -> j
      int e = w / (M * Q), rem = w - e * (M * Q), p = rem / Q, k = rem - p * Q;
      double x[M], u[Q];
      ld_pencil<M, QK>(W0 + e * SW + p * M * QK + k, x);
      X::interp(tab, x, u);
      st_pencil<Q, QK>(W1 + e * SW + p * Q * QK + k, u);
    }
    __syncthreads();
    SPHP_FOR_ITEMS(NE * Q * Q, w) {  // S3 p -> i: u, d0
      int e = w / (Q * Q), jk = w - e * (Q * Q), j = jk / Q, k = jk - j * Q;
      double x[M], u[Q], d[Q];
      ld_pencil<M, Q * QK>(W1 + e * SW + j * QK + k, x);
      X::interp_and_deriv(tab, x, u, d);
      st_pencil<Q, Q * QK>(W0 + e * SW + j * QK + k, u);
      st_pencil<Q, Q * QK>(W2 + e * SW + j * QK + k, d);
    }
    __syncthreads();
    SPHP_FOR_ITEMS(NE * Q * Q, w) {  // S4 d2 = D along k
      int e = w / (Q * Q), ij = w - e * (Q * Q);
      double v[Q], r[Q];
      ld_pencil<Q, 1>(W0 + e * SW + ij * QK, v);
      X::template deriv<false, false>(tab, v, r);
      st_pencil<Q, 1>(W1 + e * SW + ij * QK, r);
    }
    __syncthreads();
    geo_ready();  // the staged geometry is first read here (pipeline: GEO_HOOK)
    SPHP_FOR_ITEMS(NE * Q * Q, w) {  // S5 pencil along j: pointwise, t = mass + D1^T f1
      int e = w / (Q * Q), ik = w - e * (Q * Q), i = ik / Q, k = ik - i * Q;
      const int base = e * SW + i * Q * QK + k;
      double u[Q], d1v[Q], f1[Q];
      ld_pencil<Q, QK>(W0 + base, u);
      X::template deriv<false, false>(tab, u, d1v);
      const double* g = geo + e * GEO;
      double a00, a01, a02, a11, a12, a22, adet;
      if (GK == SPHP_GEOM_AFFINE) {
        const double det = g[0];
        const double* iv = g + 1;
        a00 = det * (iv[0] * iv[0] + iv[1] * iv[1] + iv[2] * iv[2]);
        a01 = det * (iv[0] * iv[3] + iv[1] * iv[4] + iv[2] * iv[5]);
        a02 = det * (iv[0] * iv[6] + iv[1] * iv[7] + iv[2] * iv[8]);
        a11 = det * (iv[3] * iv[3] + iv[4] * iv[4] + iv[5] * iv[5]);
        a12 = det * (iv[3] * iv[6] + iv[4] * iv[7] + iv[5] * iv[8]);
        a22 = det * (iv[6] * iv[6] + iv[7] * iv[7] + iv[8] * iv[8]);
        adet = det;
      }
      if constexpr (GK == SPHP_GEOM_METRIC && SPHP_JEO_S5_BYCOMP) {
        // one metric component at a time (Q independent loads in flight,
        // then their FMAs), as in the column plan's pointwise stage
        double d0[Q], d2[Q], f0[Q], f2[Q], gc[Q];
        ld_pencil<Q, QK>(W2 + base, d0);
        ld_pencil<Q, QK>(W1 + base, d2);
        auto comp = [&](int c) {
#pragma unroll
          for (int j = 0; j < Q; ++j) gc[j] = g[c * CS + metric_slot(3, Q, (i * Q + j) * Q + k)];
        };
        comp(0);
#pragma unroll
        for (int j = 0; j < Q; ++j) f0[j] = gc[j] * d0[j];
        comp(1);
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          f1[j] = gc[j] * d0[j];
          f0[j] = fma(gc[j], d1v[j], f0[j]);
        }
        comp(2);
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          f2[j] = gc[j] * d0[j];
          f0[j] = fma(gc[j], d2[j], f0[j]);
        }
        comp(3);
#pragma unroll
        for (int j = 0; j < Q; ++j) f1[j] = fma(gc[j], d1v[j], f1[j]);
        comp(4);
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          f1[j] = fma(gc[j], d2[j], f1[j]);
          f2[j] = fma(gc[j], d1v[j], f2[j]);
        }
        comp(5);
#pragma unroll
        for (int j = 0; j < Q; ++j) f2[j] = fma(gc[j], d2[j], f2[j]);
        comp(6);
#pragma unroll
        for (int j = 0; j < Q; ++j) u[j] = lam * gc[j] * u[j];
        st_pencil<Q, QK>(W2 + base, f0);
        st_pencil<Q, QK>(W1 + base, f2);
      } else {
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        const double d1 = d1v[j];
        const double d0 = W2[base + j * QK];
        const double d2 = W1[base + j * QK];
        double G00, G01, G02, G11, G12, G22, wj;
        if (GK == SPHP_GEOM_METRIC) {
          const int pt = metric_slot(3, Q, (i * Q + j) * Q + k);
          G00 = g[0 * CS + pt];
          G01 = g[1 * CS + pt];
          G02 = g[2 * CS + pt];
          G11 = g[3 * CS + pt];
          G12 = g[4 * CS + pt];
          G22 = g[5 * CS + pt];
          wj = g[6 * CS + pt];
        } else {
          const double wq = tab[T::W + i] * tab[T::W + j] * tab[T::W + k];
          G00 = wq * a00;
          G01 = wq * a01;
          G02 = wq * a02;
          G11 = wq * a11;
          G12 = wq * a12;
          G22 = wq * a22;
          wj = wq * adet;
        }
        W2[base + j * QK] = G00 * d0 + G01 * d1 + G02 * d2;
        f1[j] = G01 * d0 + G11 * d1 + G12 * d2;
        W1[base + j * QK] = G02 * d0 + G12 * d1 + G22 * d2;
        u[j] = lam * wj * u[j];
      }
      }
      X::template deriv<true, true>(tab, f1, u);
      st_pencil<Q, QK>(W0 + base, u);
    }
    __syncthreads();
    release();
    SPHP_FOR_ITEMS(NE * Q * Q, w) {  // S6 t += D2^T f2 along k
      int e = w / (Q * Q), ij = w - e * (Q * Q);
      double f[Q], t[Q];
      ld_pencil<Q, 1>(W1 + e * SW + ij * QK, f);
      ld_pencil<Q, 1>(W0 + e * SW + ij * QK, t);
      X::template deriv<true, true>(tab, f, t);
      st_pencil<Q, 1>(W0 + e * SW + ij * QK, t);
    }
    __syncthreads();
    SPHP_FOR_ITEMS(NE * Q * Q, w) {  // S7 i -> p
      int e = w / (Q * Q), jk = w - e * (Q * Q), j = jk / Q, k = jk - j * Q;
      double t[Q], f0[Q], c[M];
      ld_pencil<Q, Q * QK>(W0 + e * SW + j * QK + k, t);
      ld_pencil<Q, Q * QK>(W2 + e * SW + j * QK + k, f0);
      X::project2(tab, t, f0, c);
      st_pencil<M, Q * QK>(W1 + e * SW + j * QK + k, c);
    }
    __syncthreads();
    SPHP_FOR_ITEMS(NE * M * Q, w) {  // S8 j -> q
      int e = w / (M * Q), rem = w - e * (M * Q), p = rem / Q, k = rem - p * Q;
      double v[Q], c[M];
      ld_pencil<Q, QK>(W1 + e * SW + p * Q * QK + k, v);
      X::project(tab, v, c);
      st_pencil<M, QK>(W0 + e * SW + p * M * QK + k, c);
    }
    pre_out();
    __syncthreads();
    SPHP_FOR_ITEMS(NE * M * M, w) {  // S9 k -> r
      int e = w / (M * M), pq = w - e * (M * M);
      double v[Q], c[M];
      ld_pencil<Q, 1>(W0 + e * SW + pq * QK, v);
      X::project(tab, v, c);
      if constexpr (IO::DENSE)
        st_pencil<M, 1>(out + e * M3 + pq * M, c);
      else
        oio.template store_row<M>(out, e, pq, c);
    }
  }
};

// ===========================================================================
// Fused Helmholtz, i-column plan (HexHelmCol): the direction i never goes
// through shared memory.  Sum factorisation runs k, then j, on the small
// mode-sized tensors; the pointwise stage owns one (j, k) column of the
// element, interpolates u and the three reference derivatives along i in
// registers (dB = D B exactly, the modes being polynomials of degree < Q),
// applies the metric and projects its results back along i before they
// leave the thread.  No dense Q^3 work tensor exists:
//   S1 r->k   c[p,q,:]  -> T1 = B_k c, T1d = dB_k c           items (p, q)   A tensors [p][q][k]
//   S2 q->j   T1, T1d   -> T2 = B_j T1, T2e = dB_j T1, T2f = B_j T1d
//                                                             items (p, k)   B tensors [p][j][k]
//   S5 i      u = B_i T2, d0 = dB_i T2, d1 = B_i T2e, d2 = B_i T2f; f = G grad u;
//             U0 = B_i^T(lam wJ u) + dB_i^T f0, U1 = B_i^T f1, U2 = B_i^T f2
//                                                             items (j, k)   in place in the B tensors
//   B1 j->q   V0 = B_j^T U0 + dB_j^T U1, V1 = B_j^T U2         items (p, k)   A tensors
//   B2 k->r   y = B_k^T V0 + dB_k^T V1                         items (p, q)
// Shared-memory traffic per element: 2 M^3 + 8 M^2 Q + 12 M Q^2 + 7 Q^3
// doubles against 2 M^3 + 4 M^2 Q + 4 M Q^2 + 22 Q^3 of the K-row plan
// (P = 3: -21 %, P = 5: -18 %, P = 8: -15 %), five barriers instead of nine,
// and every column access of the pointwise stage (work tensors and the
// staged metric in natural point order) is conflict free at any Q.  Lanes
// run element-fastest over tiles of NE = 2, 4, 8 elements whose strides are
// 16 / NE (mod 16) doubles apart: a half-warp is then 16 / NE consecutive
// items of NE elements, so pitches only need the right residue mod 16 / NE
// (tools/layout_search_col.py).  More FP64 work (+25 %: four interpolations
// and three projections per column); the kernels are bound by the
// shared-memory pipe and HBM, not FP64.
// ===========================================================================
#ifndef SPHP_COL_S5_BYCOMP
#define SPHP_COL_S5_BYCOMP 1  // 0 (tuning): metric read point by point instead of one component at a time
#endif
struct ColLay {
  int RA, PA, SEA;  // A tensors: row pitch (k rows), p pitch, element stride
  int PB, SEB;      // B tensors: p pitch (rows of Q contiguous), element stride
  int GS;           // staged METRIC stride per element
  int O2, O5;       // lane orders of S2 / B1 and S5: 0 element-major, 1 element-fastest, 2 (O2) p-fastest
};
__host__ __device__ constexpr int with_res16(int lo, int res) {
  int v = lo;
  while (((v % 16) + 16) % 16 != res) ++v;
  return v;
}
__host__ __device__ constexpr bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }
__host__ __device__ constexpr ColLay col_layout(int M, int Q, int NE, int GEO) {
  ColLay L{};
  const bool ef = NE > 1 && NE <= 8 && is_pow2(NE);
  const int g = ef ? 16 / NE : 16;
  L.O2 = L.O5 = ef ? 1 : 0;
  L.RA = Q;
  // (p, k) -> p * PA + k and p * PB + k stay consecutive mod g
  L.PA = M * L.RA;
  while (L.PA % g != Q % g) ++L.PA;
  L.PB = Q * Q;
  while (L.PB % g != Q % g) ++L.PB;
  L.SEA = ef ? with_res16(2 * M * L.PA, g) : 2 * M * L.PA;
  L.SEB = ef ? with_res16(3 * M * L.PB, g) : 3 * M * L.PB;
  L.GS = (ef && GEO > 16) ? with_res16(GEO, g) : GEO;
  // searched (tools/layout_search_col.py)
#ifndef SPHP_COL_GENERIC
  if (M == 4 && Q == 5 && NE == 4) L.PA = 20, L.SEA = 164, L.PB = 25, L.SEB = 300;
  if (M == 4 && Q == 5 && NE == 8) L.PA = 20, L.SEA = 162, L.PB = 25, L.SEB = 302;
  if (M == 6 && Q == 7 && NE == 2) L.PA = 47, L.SEA = 568, L.PB = 55, L.SEB = 1000;
  if (M == 8 && Q == 9 && NE == 1) L.RA = 10, L.PA = 89, L.SEA = 1424, L.PB = 89, L.SEB = 2136;
  if (M == 9 && Q == 10 && NE == 1) L.RA = 10, L.PA = 105, L.SEA = 1890, L.PB = 105, L.SEB = 2835, L.O2 = 2;
  if (M == 5 && Q == 6 && NE == 4) L.RA = 7, L.PA = 35, L.SEA = 356, L.PB = 38, L.SEB = 572;
  // (M = 5, Q = 6, NE = 2: the searched pitches (RA 9, PA 45, PB 45: 1.07x the ideal wavefronts) cost a
  // resident CTA against the rule above, 4 instead of 5 per SM: class P = 4 0.700 vs 0.665 ms)
#endif
  return L;
}

template <int M_, int Q_, int GK, int NE_, int NT_, int NSTP_ = 2>
struct HexHelmCol {
  static constexpr int M = M_, Q = Q_, NE = NE_, NT = NT_;
  static constexpr int NSTP = NSTP_;
  static constexpr bool GEO_HOOK = true;  // compute() calls geo_ready() before its first geometry read
  static constexpr int M3 = M * M * M, Q3 = Q * Q * Q;
  static constexpr int IN = M3, OUT = M3;
  static constexpr int CS = pt_stride(Q3);
  static constexpr int GEO = (GK == SPHP_GEOM_METRIC) ? 7 * CS : 10;
  static constexpr ColLay L = col_layout(M, Q, NE, GEO);
  static constexpr int RA = L.RA, PA = L.PA, SEA = L.SEA, PB = L.PB, SEB = L.SEB;
  static constexpr int TA = M * PA, TB = M * PB;  // tensor strides inside an element's region
  static constexpr int GEO_S = L.GS;
  static_assert(RA >= Q && PA >= M * RA && SEA >= 2 * TA && PB >= Q * Q && SEB >= 3 * TB, "tensors overlap");
  static_assert(GEO_S % 2 == 0 && GEO_S >= GEO, "staged geometry stride");
  static constexpr int WORK = SEA + SEB;
  static constexpr int OUT_OFF = NE * SEA;  // B2 writes the block into the B region (free after B1)
  static_assert(NE * SEB >= NE * M3 + 4, "output block does not fit the B region");
  using T = Tab<M, Q>;
  using X = EO<M, Q>;

  // item w of a stage over (e, a, b), b in [0, NB): element-major (b
  // fastest), element-fastest, or element-major with a fastest
  template <int ORDER, int NA, int NB>
  __device__ static __forceinline__ void item(int w, int& e, int& a, int& b) {
    if constexpr (ORDER == 1) {
      e = w % NE;
      const int ab = w / NE;
      a = ab / NB, b = ab - a * NB;
    } else if constexpr (ORDER == 2) {
      e = w / (NA * NB);
      const int ab = w - e * (NA * NB);
      b = ab / NA, a = ab - b * NA;
    } else {
      e = w / (NA * NB);
      const int ab = w - e * (NA * NB);
      a = ab / NB, b = ab - a * NB;
    }
  }

  template <class R, class W, class IO = BlockIO, class H = NoHook, class GH = NoHook>
  __device__ static void compute(const double* __restrict__ cin, const double* __restrict__ geo,
                                 double* __restrict__ work, double* __restrict__ out, double lam,
                                 R release, W pre_out, const double* tab, IO io = IO(),
                                 IO oio = IO(), H after_in = H(), GH geo_ready = GH()) {
    double* WA = work;
    double* WB = work + NE * SEA;
    // S1: r -> k, value and k-derivative
    SPHP_FOR_ITEMS(NE * M * M, w) {
      const int e = w / (M * M), pq = w - e * (M * M), p = pq / M, q = pq - p * M;
      double x[M], u[Q], d[Q];
      if constexpr (IO::DENSE)
        RowRot<M>::load(cin + e * M3 + pq * M, w, x);
      else
        io.template load_row<M>(cin, e, pq, x);
      X::interp_and_deriv(tab, x, u, d);
      double* a = WA + e * SEA + p * PA + q * RA;
      st_pencil<Q, 1>(a, u);
      st_pencil<Q, 1>(a + TA, d);
    }
    __syncthreads();
    after_in();
    // S2: q -> j
    SPHP_FOR_ITEMS(NE * M * Q, w) {
      int e, p, k;
      item<L.O2, M, Q>(w, e, p, k);
      const double* a = WA + e * SEA + p * PA + k;
      double* b = WB + e * SEB + p * PB + k;
      double x[M], xd[M], u[Q], d[Q];
      // both pencils before any store (the compiler cannot move a load of the
      // A tensors above a store to the B tensors: same work area)
      ld_pencil<M, RA>(a, x);
      ld_pencil<M, RA>(a + TA, xd);
      X::interp_and_deriv(tab, x, u, d);
      st_pencil<Q, Q>(b, u);
      st_pencil<Q, Q>(b + TB, d);
      X::interp(tab, xd, u);
      st_pencil<Q, Q>(b + 2 * TB, u);
    }
    __syncthreads();
    geo_ready();  // the staged geometry is first read here (pipeline: GEO_HOOK)
    // S5: columns along i
    SPHP_FOR_ITEMS(NE * Q * Q, w) {
      int e, j, k;
      item<L.O5, Q, Q>(w, e, j, k);
      const int jk = j * Q + k;
      double* b = WB + e * SEB + jk;
      double x[M], u[Q], d0[Q], d1[Q], d2[Q], f0[Q], f1[Q], f2[Q];
      double g[Q];
      const double* gr = geo + e * GEO_S + jk;
      auto comp = [&](int c) {
#pragma unroll
        for (int i = 0; i < Q; ++i) g[i] = gr[c * CS + i * Q * Q];
      };
      ld_pencil<M, PB>(b, x);
      X::interp_and_deriv(tab, x, u, d0);
      ld_pencil<M, PB>(b + TB, x);
      X::interp(tab, x, d1);
      ld_pencil<M, PB>(b + 2 * TB, x);
      X::interp(tab, x, d2);
      if constexpr (GK == SPHP_GEOM_METRIC && SPHP_COL_S5_BYCOMP) {
        // one metric component at a time: Q independent loads in flight,
        // then their FMAs (point by point, 7 loads then 9 FMAs, measured
        // slower: P=4 assembled 0.666 vs 0.646 ms, P=5 local 1.02 vs 0.97;
        // hoisting the column loads and the first component above the
        // interpolations as well: no further gain)
        comp(0);
#pragma unroll
        for (int i = 0; i < Q; ++i) f0[i] = g[i] * d0[i];
        comp(1);
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          f1[i] = g[i] * d0[i];
          f0[i] = fma(g[i], d1[i], f0[i]);
        }
        comp(2);
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          f2[i] = g[i] * d0[i];
          f0[i] = fma(g[i], d2[i], f0[i]);
        }
        comp(3);
#pragma unroll
        for (int i = 0; i < Q; ++i) f1[i] = fma(g[i], d1[i], f1[i]);
        comp(4);
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          f1[i] = fma(g[i], d2[i], f1[i]);
          f2[i] = fma(g[i], d1[i], f2[i]);
        }
        comp(5);
#pragma unroll
        for (int i = 0; i < Q; ++i) f2[i] = fma(g[i], d2[i], f2[i]);
        comp(6);
#pragma unroll
        for (int i = 0; i < Q; ++i) u[i] = lam * g[i] * u[i];
      } else if constexpr (GK == SPHP_GEOM_METRIC) {
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          const double g0 = gr[0 * CS + i * Q * Q], g1 = gr[1 * CS + i * Q * Q], g2 = gr[2 * CS + i * Q * Q];
          f0[i] = fma(g2, d2[i], fma(g1, d1[i], g0 * d0[i]));
          const double g3 = gr[3 * CS + i * Q * Q], g4 = gr[4 * CS + i * Q * Q];
          f1[i] = fma(g4, d2[i], fma(g3, d1[i], g1 * d0[i]));
          const double g5 = gr[5 * CS + i * Q * Q];
          f2[i] = fma(g5, d2[i], fma(g4, d1[i], g2 * d0[i]));
          u[i] = lam * gr[6 * CS + i * Q * Q] * u[i];
        }
      } else {
        const double* gg = geo + e * GEO_S;
        const double det = gg[0];
        const double* iv = gg + 1;
        const double a00 = det * (iv[0] * iv[0] + iv[1] * iv[1] + iv[2] * iv[2]);
        const double a01 = det * (iv[0] * iv[3] + iv[1] * iv[4] + iv[2] * iv[5]);
        const double a02 = det * (iv[0] * iv[6] + iv[1] * iv[7] + iv[2] * iv[8]);
        const double a11 = det * (iv[3] * iv[3] + iv[4] * iv[4] + iv[5] * iv[5]);
        const double a12 = det * (iv[3] * iv[6] + iv[4] * iv[7] + iv[5] * iv[8]);
        const double a22 = det * (iv[6] * iv[6] + iv[7] * iv[7] + iv[8] * iv[8]);
        const double wjk = tab[T::W + j] * tab[T::W + k];
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          const double wq = wjk * tab[T::W + i];
          f0[i] = wq * (a00 * d0[i] + a01 * d1[i] + a02 * d2[i]);
          f1[i] = wq * (a01 * d0[i] + a11 * d1[i] + a12 * d2[i]);
          f2[i] = wq * (a02 * d0[i] + a12 * d1[i] + a22 * d2[i]);
          u[i] = lam * (wq * det) * u[i];
        }
      }
      double c[M];
      X::project2(tab, u, f0, c);
      st_pencil<M, PB>(b, c);
      X::project(tab, f1, c);
      st_pencil<M, PB>(b + TB, c);
      X::project(tab, f2, c);
      st_pencil<M, PB>(b + 2 * TB, c);
    }
    __syncthreads();
    release();
    // B1: j -> q
    SPHP_FOR_ITEMS(NE * M * Q, w) {
      int e, p, k;
      item<L.O2, M, Q>(w, e, p, k);
      const double* b = WB + e * SEB + p * PB + k;
      double* a = WA + e * SEA + p * PA + k;
      double t[Q], f[Q], g[Q], c[M];
      ld_pencil<Q, Q>(b, t);
      ld_pencil<Q, Q>(b + TB, f);
      ld_pencil<Q, Q>(b + 2 * TB, g);  // before the first store, as in S2
      X::project2(tab, t, f, c);
      st_pencil<M, RA>(a, c);
      X::project(tab, g, c);
      st_pencil<M, RA>(a + TA, c);
    }
    pre_out();
    __syncthreads();
    // B2: k -> r
    SPHP_FOR_ITEMS(NE * M * M, w) {
      const int e = w / (M * M), pq = w - e * (M * M), p = pq / M, q = pq - p * M;
      const double* a = WA + e * SEA + p * PA + q * RA;
      double t[Q], f[Q], c[M];
      ld_pencil<Q, 1>(a, t);
      ld_pencil<Q, 1>(a + TA, f);
      X::project2(tab, t, f, c);
      if constexpr (IO::DENSE)
        RowRot<M>::store(out + e * M3 + pq * M, w, c);
      else
        oio.template store_row<M>(out, e, pq, c);
    }
  }
};

// variant selection: i-column plan where col_plan(Q) (common.cuh), else
// j-pencil plan at Q % 4 == 0, k-row plan otherwise
template <int M_, int Q_, int GK, int NE_, int NT_, int NSTP_, bool COL>
using HexHelmSel = typename std::conditional<
    COL, HexHelmCol<M_, Q_, GK, NE_, NT_, NSTP_>,
    typename std::conditional<(Q_ % 4 == 0), HexHelmJEO<M_, Q_, GK, NE_, NT_, NSTP_>,
                              HexHelmEO<M_, Q_, GK, NE_, NT_, NSTP_>>::type>::type;

template <int M_, int Q_, int GK, int NE_, int NT_, int NSTP_ = 2>
using HexHelm = HexHelmSel<M_, Q_, GK, NE_, NT_, NSTP_, col_plan(Q_)>;

// ===========================================================================
// BwdTrans (K1): u = (B x B x B)^T c   (collections.py:133-150)
// ===========================================================================
template <int M_, int Q_, int NE_, int NT_>
struct HexBwd {
  static constexpr int M = M_, Q = Q_, NE = NE_, NT = NT_;
  static constexpr int M3 = M * M * M, Q3 = Q * Q * Q;
  static constexpr int IN = M3, OUT = Q3, GEO = 0;
  static constexpr int QK = odd_up(Q);
  // B[p][j][k]: contiguous rows, plane pitch = Q (mod 16) so the (p, k)
  // lanes of the j-stage hit consecutive banks (wavefront model,
  // tools/layout_search_bwd.py: -18 % at P=4 and fewer at every fast key)
  static constexpr int PB = pitch_mod16(Q * Q, Q);
  static constexpr int SA = odd_up(M * M * QK), SB = M * PB;
  static constexpr int WORK = SA + SB;
  using T = Tab<M, Q>;

  template <class R, class W>
  __device__ static void compute(const double* __restrict__ cin, const double* __restrict__,
                                 double* __restrict__ work, double* __restrict__ out, double,
                                 R release, W pre_out, const double* tab) {
    double* A = work;
    double* Bb = work + NE * SA;
    SPHP_FOR_ITEMS(NE * M * M, w) {
      int e = w / (M * M), pq = w - e * (M * M);
      eo_interp<M, Q, 1, 1>(tab, cin + e * M3 + pq * M, A + e * SA + pq * QK);
    }
    __syncthreads();
    release();
    SPHP_FOR_ITEMS(NE * M * Q, w) {
      int e = w / (M * Q), rem = w - e * (M * Q), p = rem / Q, k = rem - p * Q;
      eo_interp<M, Q, QK, Q>(tab, A + e * SA + p * M * QK + k, Bb + e * SB + p * PB + k);
    }
    pre_out();
    __syncthreads();
    SPHP_FOR_ITEMS(NE * Q * Q, w) {
      int e = w / (Q * Q), jk = w - e * (Q * Q), j = jk / Q, k = jk - j * Q;
      eo_interp<M, Q, PB, Q * Q>(tab, Bb + e * SB + j * Q + k, out + e * Q3 + j * Q + k);
    }
  }
};

// ===========================================================================
// IProductWRTBase (K2): c = (B x B x B) (W u)   (collections.py:152-167, 215-224)
// GK: NONE (reference weights), AFFINE (w * det_e), POINT (staged wJ comp)
// ===========================================================================
template <int M_, int Q_, int GK, int NE_, int NT_>
struct HexIprod {
  static constexpr int M = M_, Q = Q_, NE = NE_, NT = NT_;
  static constexpr int M3 = M * M * M, Q3 = Q * Q * Q;
  static constexpr int IN = Q3, OUT = M3;
  static constexpr int CS = pt_stride(Q3);
  static constexpr int GEO = (GK == SPHP_GEOM_POINT) ? CS : (GK == SPHP_GEOM_AFFINE ? 10 : 0);
  static constexpr int QK = odd_up(Q);
  // B[p][j][k] as in HexBwd: contiguous rows, plane pitch = Q (mod 16)
  static constexpr int PB = pitch_mod16(Q * Q, Q);
  static constexpr int SA = odd_up(M * M * QK), SB = M * PB;
  static constexpr int WORK = SA + SB;
  static constexpr int OUT_OFF = NE * SA;  // the last stage reads A: the block is staged in B
  using T = Tab<M, Q>;

  template <class R, class W>
  __device__ static void compute(const double* __restrict__ uin, const double* __restrict__ geo,
                                 double* __restrict__ work, double* __restrict__ out, double,
                                 R release, W pre_out, const double* tab) {
    double* A = work;
    double* Bb = work + NE * SA;
    // i -> p with the weights folded in (wu = W*u, collections.py:216)
    SPHP_FOR_ITEMS(NE * Q * Q, w) {
      int e = w / (Q * Q), jk = w - e * (Q * Q), j = jk / Q, k = jk - j * Q;
      double x[Q];
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        const int pt = (i * Q + j) * Q + k;
        double wt;
        if (GK == SPHP_GEOM_POINT)
          wt = geo[e * GEO + pt];
        else if (GK == SPHP_GEOM_AFFINE)
          wt = tab[T::W + i] * tab[T::W + j] * tab[T::W + k] * geo[e * GEO];
        else
          wt = tab[T::W + i] * tab[T::W + j] * tab[T::W + k];
        x[i] = wt * uin[e * Q3 + pt];
      }
#pragma unroll
      for (int p = 0; p < M; ++p) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < Q; ++i) acc = fma(tab[T::B + p * Q + i], x[i], acc);
        Bb[e * SB + p * PB + j * Q + k] = acc;
      }
    }
    __syncthreads();
    release();
    SPHP_FOR_ITEMS(NE * M * Q, w) {
      int e = w / (M * Q), rem = w - e * (M * Q), p = rem / Q, k = rem - p * Q;
      eo_project<M, Q, Q, QK>(tab, Bb + e * SB + p * PB + k, A + e * SA + p * M * QK + k);
    }
    pre_out();
    __syncthreads();
    SPHP_FOR_ITEMS(NE * M * M, w) {
      int e = w / (M * M), pq = w - e * (M * M);
      eo_project<M, Q, 1, 1>(tab, A + e * SA + pq * QK, out + e * M3 + pq * M);
    }
  }
};

// ===========================================================================
// PhysDeriv (K3): d_a = D_a u ; world dx_k = sum_a inv[a,k] d_a
// (collections.py:169-185, 226-241).  Output (3, Q3) per element.
// GK: NONE (reference components), AFFINE, POINT (staged inv comps 1..9)
// ===========================================================================
template <int M_, int Q_, int GK, int NE_, int NT_>
struct HexPhysDeriv {
  static constexpr int M = M_, Q = Q_, NE = NE_, NT = NT_;
  static constexpr int Q3 = Q * Q * Q;
  static constexpr int IN = Q3, OUT = 3 * Q3;
  static constexpr int CS = pt_stride(Q3);
  static constexpr int GEO = (GK == SPHP_GEOM_POINT) ? 9 * CS : (GK == SPHP_GEOM_AFFINE ? 10 : 0);
  static constexpr int QK = odd_up(Q);
  static constexpr int SW = odd_up(Q * Q * QK);
  static constexpr int WORK = 2 * SW;
  static constexpr bool ROWROT = (Q % 4 == 0);
  using T = Tab<M, Q>;

  template <class R, class W>
  __device__ static void compute(const double* __restrict__ uin, const double* __restrict__ geo,
                                 double* __restrict__ work, double* __restrict__ out, double,
                                 R release, W pre_out, const double* tab) {
    double* W0 = work;
    double* W1 = work + NE * SW;
    // d0 (pencils along i) and d1 (pencils along j) in one stage
    SPHP_FOR_ITEMS(2 * NE * Q * Q, w) {
      const int half = w >= NE * Q * Q;
      const int v = half ? w - NE * Q * Q : w;
      int e = v / (Q * Q), ab = v - e * (Q * Q), a = ab / Q, b = ab - a * Q;
      if (!half) {  // pencil along i at (j=a, k=b)
        eo_deriv<M, Q, false, false, Q * Q, Q * Q * QK / Q>(
            tab, uin + e * Q3 + a * Q + b, W0 + e * SW + a * QK + b);
      } else {  // pencil along j at (i=a, k=b)
        eo_deriv<M, Q, false, false, Q, QK>(tab, uin + e * Q3 + a * Q * Q + b,
                                               W1 + e * SW + a * Q * QK + b);
      }
    }
    pre_out();
    __syncthreads();
    // pencil along k: d2 in registers, metric transform, write 3 comps
    SPHP_FOR_ITEMS(NE * Q * Q, w) {
      int e = w / (Q * Q), ij = w - e * (Q * Q), i = ij / Q, j = ij - i * Q;
      double x[Q], r0[Q], r1[Q], r2[Q];
      // rows of Q doubles one lane each: rotated order (RowRot) when Q = 0
      // mod 4 (4-8-way conflicts otherwise; P=6: 908 -> 697 us); at Q = 2
      // mod 4 the 2-way conflicts cost less than the rotation (measured)
      if constexpr (ROWROT) {
        RowRot<Q>::load(uin + e * Q3 + ij * Q, w, x);
      } else {
#pragma unroll
        for (int k = 0; k < Q; ++k) x[k] = uin[e * Q3 + ij * Q + k];
      }
      const double* g = geo + e * GEO;
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        double d2 = 0.0;
#pragma unroll
        for (int l = 0; l < Q; ++l) d2 = fma(tab[T::D + k * Q + l], x[l], d2);
        const double d0 = W0[e * SW + ij * QK + k];
        const double d1 = W1[e * SW + ij * QK + k];
        const int pt = ij * Q + k;
        double o0 = d0, o1 = d1, o2 = d2;
        if (GK != SPHP_GEOM_NONE) {
          double iv[9];
#pragma unroll
          for (int c = 0; c < 9; ++c) iv[c] = (GK == SPHP_GEOM_POINT) ? g[c * CS + pt] : g[1 + c];
          // dx_k = sum_a inv[a,k] d_a ; inv row-major [a*3 + k]
          o0 = iv[0] * d0 + iv[3] * d1 + iv[6] * d2;
          o1 = iv[1] * d0 + iv[4] * d1 + iv[7] * d2;
          o2 = iv[2] * d0 + iv[5] * d1 + iv[8] * d2;
        }
        r0[k] = o0;
        r1[k] = o1;
        r2[k] = o2;
      }
      const int row = e * 3 * Q * Q + ij;  // row index of component 0 in the output block
      if constexpr (ROWROT) {
        RowRot<Q>::store(out + e * OUT + 0 * Q3 + ij * Q, row, r0);
        RowRot<Q>::store(out + e * OUT + 1 * Q3 + ij * Q, row + Q * Q, r1);
        RowRot<Q>::store(out + e * OUT + 2 * Q3 + ij * Q, row + 2 * Q * Q, r2);
      } else {
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          out[e * OUT + 0 * Q3 + ij * Q + k] = r0[k];
          out[e * OUT + 1 * Q3 + ij * Q + k] = r1[k];
          out[e * OUT + 2 * Q3 + ij * Q + k] = r2[k];
        }
      }
    }
    __syncthreads();
    release();
  }
};

// ===========================================================================
// IProductWRTDerivBase: c = sum_a B_a [ wJ sum_k inv[a,k] f_k ]
// (geometry.py:163-168; batched form solvers.py:361-365).  Input (3, Q3).
// GK: NONE (g_a = w f_a), AFFINE, POINT (staged comps 0..9 = wJ, inv)
// ===========================================================================
template <int M_, int Q_, int GK, int NE_, int NT_>
struct HexIPDeriv {
  static constexpr int M = M_, Q = Q_, NE = NE_, NT = NT_;
  static constexpr int M3 = M * M * M, Q3 = Q * Q * Q;
  static constexpr int IN = 3 * Q3, OUT = M3;
  static constexpr int CS = pt_stride(Q3);
  static constexpr int GEO = (GK == SPHP_GEOM_POINT) ? 10 * CS : (GK == SPHP_GEOM_AFFINE ? 10 : 0);
  static constexpr int QK = odd_up(Q);
  static constexpr int SW = odd_up(Q * Q * QK);
  static constexpr int WORK = 3 * SW;
  static constexpr int OUT_OFF = NE * SW;  // the last stage reads W0: the block is staged in W1
  using T = Tab<M, Q>;

  template <class R, class W>
  __device__ static void compute(const double* __restrict__ fin, const double* __restrict__ geo,
                                 double* __restrict__ work, double* __restrict__ out, double,
                                 R release, W pre_out, const double* tab) {
    double* W0 = work;            // t
    double* W1 = work + NE * SW;  // g0 | later T2'
    double* W2 = work + 2 * NE * SW;  // g1 | later T1'
    // pencil along k: g = wJ inv f ; t = D2^T g2
    SPHP_FOR_ITEMS(NE * Q * Q, w) {
      int e = w / (Q * Q), ij = w - e * (Q * Q), i = ij / Q, j = ij - i * Q;
      const double* g = geo + e * GEO;
      double g2[Q], rx[Q], ry[Q], rz[Q];
      // the three input rows, in rotated order when Q = 0 mod 4 (RowRot;
      // see HexPhysDeriv)
      if constexpr (Q % 4 == 0) {
        const int row = e * 3 * Q * Q + ij;
        RowRot<Q>::load(fin + e * IN + ij * Q, row, rx);
        RowRot<Q>::load(fin + e * IN + Q3 + ij * Q, row + Q * Q, ry);
        RowRot<Q>::load(fin + e * IN + 2 * Q3 + ij * Q, row + 2 * Q * Q, rz);
      } else {
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          rx[k] = fin[e * IN + ij * Q + k];
          ry[k] = fin[e * IN + Q3 + ij * Q + k];
          rz[k] = fin[e * IN + 2 * Q3 + ij * Q + k];
        }
      }
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        const int pt = ij * Q + k;
        const double fx = rx[k], fy = ry[k], fz = rz[k];
        double a0, a1, a2;
        if (GK == SPHP_GEOM_NONE) {
          const double wq = tab[T::W + i] * tab[T::W + j] * tab[T::W + k];
          a0 = wq * fx;
          a1 = wq * fy;
          a2 = wq * fz;
        } else {
          double wj;
          double iv[9];
          if (GK == SPHP_GEOM_POINT) {
            wj = g[pt];
#pragma unroll
            for (int c = 0; c < 9; ++c) iv[c] = g[(1 + c) * CS + pt];
          } else {
            wj = tab[T::W + i] * tab[T::W + j] * tab[T::W + k] * g[0];
#pragma unroll
            for (int c = 0; c < 9; ++c) iv[c] = g[1 + c];
          }
          a0 = wj * (iv[0] * fx + iv[1] * fy + iv[2] * fz);
          a1 = wj * (iv[3] * fx + iv[4] * fy + iv[5] * fz);
          a2 = wj * (iv[6] * fx + iv[7] * fy + iv[8] * fz);
        }
        W1[e * SW + ij * QK + k] = a0;
        W2[e * SW + ij * QK + k] = a1;
        g2[k] = a2;
      }
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        double t = 0.0;
#pragma unroll
        for (int l = 0; l < Q; ++l) t = fma(tab[T::D + l * Q + k], g2[l], t);
        W0[e * SW + ij * QK + k] = t;
      }
    }
    __syncthreads();
    release();
    // t += D1^T g1 along j
    SPHP_FOR_ITEMS(NE * Q * Q, w) {
      int e = w / (Q * Q), ik = w - e * (Q * Q), i = ik / Q, k = ik - i * Q;
      eo_deriv<M, Q, true, true, QK, QK>(tab, W2 + e * SW + i * Q * QK + k,
                                             W0 + e * SW + i * Q * QK + k);
    }
    __syncthreads();
    // i -> p : T2'[p,j,k] = sum_i B t + Bd g0  (into W2)
    SPHP_FOR_ITEMS(NE * Q * Q, w) {
      int e = w / (Q * Q), jk = w - e * (Q * Q), j = jk / Q, k = jk - j * Q;
      const int base = e * SW + j * QK + k;
      double t[Q], g0[Q];
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        t[i] = W0[base + i * Q * QK];
        g0[i] = W1[base + i * Q * QK];
      }
#pragma unroll
      for (int p = 0; p < M; ++p) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          acc = fma(tab[T::B + p * Q + i], t[i], acc);
          acc = fma(tab[T::BD + p * Q + i], g0[i], acc);
        }
        W2[e * SW + (p * Q + j) * QK + k] = acc;
      }
    }
    __syncthreads();
    SPHP_FOR_ITEMS(NE * M * Q, w) {
      int e = w / (M * Q), rem = w - e * (M * Q), p = rem / Q, k = rem - p * Q;
      eo_project<M, Q, QK, QK>(tab, W2 + e * SW + p * Q * QK + k,
                                              W0 + e * SW + p * M * QK + k);
    }
    pre_out();
    __syncthreads();
    SPHP_FOR_ITEMS(NE * M * M, w) {
      int e = w / (M * M), pq = w - e * (M * M);
      eo_project<M, Q, 1, 1>(tab, W0 + e * SW + pq * QK, out + e * M3 + pq * M);
    }
  }
};

}  // namespace sphp
