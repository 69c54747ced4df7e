// Quadrilateral sum-factorisation operators: collections.py:133-185 for
// Shape.QUAD, plus IProductWRTDerivBase (geometry.py:163-168) and the fused
// Helmholtz operator (geometry.py:171-184).
// Layouts: coefficient c[p*M + q], point u[i*Q + j] (stdregions.py:5-13).
#pragma once
#ifndef SPHP_QUAD_NST
#define SPHP_QUAD_NST 1  // quad tile pipeline input stages (tuning)
#endif
#include "hex_ops.cuh"

namespace sphp {

// 2D geometry records: AFFINE [det, inv00, inv01, inv10, inv11, pad];
// POINT [wJ, inv00, inv01, inv10, inv11] x CS; METRIC [G00, G01, G11, wJ] x CS
// smallest stride >= x that is = 2 (mod 16) doubles: eight elements at that
// stride start on eight distinct even bank pairs (and on eight distinct
// 16-byte slots of a 128-byte line), so a half-warp of 8 elements x 2
// positions that differ by an odd offset is conflict free
__host__ __device__ constexpr int spread16(int x) { return x + ((2 - x % 16) + 16) % 16; }

// Fused Helmholtz on quads.  Work items are ordered element-fastest (item w:
// element w % NE, position w / NE) with NE = 8, and the per-element strides
// of the work buffers (SW) and of the staged geometry (GEO_S) are = 2 (mod
// 16): every stage's half-warp (8 elements x 2 positions, odd position
// offset) and every geometry row read (a quarter-warp of 8 elements, same
// row: LDS.128) then touch distinct banks.  (The first layout, positions
// fastest with SW = odd, measured 59 % bank-conflict excess at cfg2.)
template <int M_, int Q_, int GK, int NE_, int NT_>
struct QuadHelm {
  static constexpr int M = M_, Q = Q_, NE = NE_, NT = NT_;
  static constexpr int NSTP = SPHP_QUAD_NST;  // preferred input stages
  static constexpr int M2 = M * M, Q2 = Q * Q;
  static constexpr int IN = M2, OUT = M2;
  static constexpr int CS = pt_stride(Q2);
  static constexpr int GEO = (GK == SPHP_GEOM_METRIC) ? 4 * CS : 6;
  static constexpr int GEO_S = (GK == SPHP_GEOM_METRIC) ? spread16(GEO) : GEO;
  static constexpr int QK = odd_up(Q);
  static constexpr int SW = spread16(Q * QK);
  static constexpr int WORK = 3 * SW;
  // the last stage reads only W0: the output block is staged in W1 (one
  // buffer fewer per CTA -> more resident CTAs; the kernel is latency bound)
  static constexpr int OUT_OFF = NE * SW;
  using T = Tab<M, Q>;
  using X = EO<M, Q>;

  template <class R, class W>
  __device__ static void compute(const double* __restrict__ cin, const double* __restrict__ geo,
                                 double* __restrict__ work, double* __restrict__ out, double lam,
                                 R release, W pre_out, const double* tab) {
    double* W0 = work;
    double* W1 = work + NE * SW;
    double* W2 = work + 2 * NE * SW;
    SPHP_FOR_ITEMS(NE * M, w) {  // q -> j
      const int e = w % NE, p = w / NE;
      eo_interp<M, Q, 1, 1>(tab, cin + e * M2 + p * M, W0 + e * SW + p * QK);
    }
    __syncthreads();
    SPHP_FOR_ITEMS(NE * Q, w) {  // p -> i, u and d0 (even-odd form)
      const int e = w % NE, j = w / NE;
      double x[M], u[Q], d[Q];
#pragma unroll
      for (int p = 0; p < M; ++p) x[p] = W0[e * SW + p * QK + j];
      X::interp_and_deriv(tab, x, u, d);
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        W1[e * SW + i * QK + j] = u[i];
        W2[e * SW + i * QK + j] = d[i];
      }
    }
    __syncthreads();
    SPHP_FOR_ITEMS(NE * Q, w) {  // pencil along j: d1, fluxes, t = mass + D1^T f1
      const int e = w % NE, i = w / NE;
      const int base = e * SW + i * QK;
      double u[Q], f1[Q];
#pragma unroll
      for (int j = 0; j < Q; ++j) u[j] = W1[base + j];
      const double* g = geo + e * GEO_S;
      double a00, a01, a11, adet;
      if (GK == SPHP_GEOM_AFFINE) {
        const double det = g[0];
        a00 = det * (g[1] * g[1] + g[2] * g[2]);
        a01 = det * (g[1] * g[3] + g[2] * g[4]);
        a11 = det * (g[3] * g[3] + g[4] * g[4]);
        adet = det;
      }
      double d1v[Q];
      X::template deriv<false, false>(tab, u, d1v);
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        const double d1 = d1v[j];
        const double d0 = W2[base + j];
        double G00, G01, G11, wj;
        if (GK == SPHP_GEOM_METRIC) {
          const int pt = i * Q + j;
          G00 = g[pt];
          G01 = g[CS + pt];
          G11 = g[2 * CS + pt];
          wj = g[3 * CS + pt];
        } else {
          const double wq = tab[T::W + i] * tab[T::W + j];
          G00 = wq * a00;
          G01 = wq * a01;
          G11 = wq * a11;
          wj = wq * adet;
        }
        W2[base + j] = G00 * d0 + G01 * d1;
        f1[j] = G01 * d0 + G11 * d1;
        u[j] = lam * wj * u[j];
      }
      X::template deriv<true, true>(tab, f1, u);  // t = mass + D1^T f1
#pragma unroll
      for (int j = 0; j < Q; ++j) W1[base + j] = u[j];
    }
    __syncthreads();
    release();
    SPHP_FOR_ITEMS(NE * Q, w) {  // i -> p : B t + Bd f0
      const int e = w % NE, j = w / NE;
      double t[Q], f0[Q], c[M];
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        t[i] = W1[e * SW + i * QK + j];
        f0[i] = W2[e * SW + i * QK + j];
      }
      X::project2(tab, t, f0, c);
#pragma unroll
      for (int p = 0; p < M; ++p) W0[e * SW + p * QK + j] = c[p];
    }
    pre_out();
    __syncthreads();
    SPHP_FOR_ITEMS(NE * M, w) {  // j -> q
      const int e = w % NE, p = w / NE;
      eo_project<M, Q, 1, 1>(tab, W0 + e * SW + p * QK, out + e * M2 + p * M);
    }
  }
};

template <int M_, int Q_, int NE_, int NT_>
struct QuadBwd {
  static constexpr int M = M_, Q = Q_, NE = NE_, NT = NT_;
  static constexpr int NSTP = SPHP_QUAD_NST;
  static constexpr int M2 = M * M, Q2 = Q * Q;
  static constexpr int IN = M2, OUT = Q2, GEO = 0;
  static constexpr int QK = odd_up(Q);
  static constexpr int SW = odd_up(M * QK);
  static constexpr int WORK = SW;
  using T = Tab<M, Q>;

  template <class R, class W>
  __device__ static void compute(const double* __restrict__ cin, const double* __restrict__,
                                 double* __restrict__ work, double* __restrict__ out, double,
                                 R release, W pre_out, const double* tab) {
    SPHP_FOR_ITEMS(NE * M, w) {
      int e = w / M, p = w - e * M;
      eo_interp<M, Q, 1, 1>(tab, cin + e * M2 + p * M, work + e * SW + p * QK);
    }
    pre_out();
    __syncthreads();
    release();
    SPHP_FOR_ITEMS(NE * Q, w) {
      int e = w / Q, j = w - e * Q;
      eo_interp<M, Q, QK, Q>(tab, work + e * SW + j, out + e * Q2 + j);
    }
  }
};

template <int M_, int Q_, int GK, int NE_, int NT_>
struct QuadIprod {
  static constexpr int M = M_, Q = Q_, NE = NE_, NT = NT_;
  static constexpr int NSTP = SPHP_QUAD_NST;
  static constexpr int M2 = M * M, Q2 = Q * Q;
  static constexpr int IN = Q2, OUT = M2;
  static constexpr int CS = pt_stride(Q2);
  static constexpr int GEO = (GK == SPHP_GEOM_POINT) ? CS : (GK == SPHP_GEOM_AFFINE ? 6 : 0);
  static constexpr int QK = odd_up(Q);
  static constexpr int SW = odd_up(M * QK);
  static constexpr int WORK = SW;
  using T = Tab<M, Q>;

  template <class R, class W>
  __device__ static void compute(const double* __restrict__ uin, const double* __restrict__ geo,
                                 double* __restrict__ work, double* __restrict__ out, double,
                                 R release, W pre_out, const double* tab) {
    SPHP_FOR_ITEMS(NE * Q, w) {  // i -> p with weights
      int e = w / Q, j = w - e * Q;
      double x[Q];
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        const int pt = i * Q + j;
        double wt;
        if (GK == SPHP_GEOM_POINT)
          wt = geo[e * GEO + pt];
        else if (GK == SPHP_GEOM_AFFINE)
          wt = tab[T::W + i] * tab[T::W + j] * geo[e * GEO];
        else
          wt = tab[T::W + i] * tab[T::W + j];
        x[i] = wt * uin[e * Q2 + pt];
      }
#pragma unroll
      for (int p = 0; p < M; ++p) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < Q; ++i) acc = fma(tab[T::B + p * Q + i], x[i], acc);
        work[e * SW + p * QK + j] = acc;
      }
    }
    pre_out();
    __syncthreads();
    release();
    SPHP_FOR_ITEMS(NE * M, w) {
      int e = w / M, p = w - e * M;
      eo_project<M, Q, 1, 1>(tab, work + e * SW + p * QK, out + e * M2 + p * M);
    }
  }
};

template <int M_, int Q_, int GK, int NE_, int NT_>
struct QuadPhysDeriv {
  static constexpr int M = M_, Q = Q_, NE = NE_, NT = NT_;
  static constexpr int NSTP = SPHP_QUAD_NST;
  static constexpr int Q2 = Q * Q;
  static constexpr int IN = Q2, OUT = 2 * Q2;
  static constexpr int CS = pt_stride(Q2);
  static constexpr int GEO = (GK == SPHP_GEOM_POINT) ? 4 * CS : (GK == SPHP_GEOM_AFFINE ? 6 : 0);
  static constexpr int QK = odd_up(Q);
  static constexpr int SW = odd_up(Q * QK);
  static constexpr int WORK = SW;
  using T = Tab<M, Q>;

  template <class R, class W>
  __device__ static void compute(const double* __restrict__ uin, const double* __restrict__ geo,
                                 double* __restrict__ work, double* __restrict__ out, double,
                                 R release, W pre_out, const double* tab) {
    SPHP_FOR_ITEMS(NE * Q, w) {  // d0 along i
      int e = w / Q, j = w - e * Q;
      eo_deriv<M, Q, false, false, Q, QK>(tab, uin + e * Q2 + j, work + e * SW + j);
    }
    pre_out();
    __syncthreads();
    SPHP_FOR_ITEMS(NE * Q, w) {  // along j: d1, metric (collections.py:181-185)
      int e = w / Q, i = w - e * Q;
      // rows of Q doubles one lane each (input, 4 metric rows, 2 output
      // rows): rotated order for Q = 0 mod 4 (RowRot, 4-8-way conflicts
      // otherwise), plain order at Q = 2 mod 4
      constexpr bool ROT = (Q % 4 == 0) && (CS % Q == 0) && (GEO % Q == 0);
      double x[Q], gi[4][Q], o0[Q], o1[Q];
      if constexpr (ROT) {
        RowRot<Q>::load(uin + e * Q2 + i * Q, w, x);
      } else {
#pragma unroll
        for (int j = 0; j < Q; ++j) x[j] = uin[e * Q2 + i * Q + j];
      }
      const double* g = geo + e * GEO;
      if constexpr (GK == SPHP_GEOM_POINT) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if constexpr (ROT) {
            RowRot<Q>::load(g + c * CS + i * Q, (e * GEO + c * CS) / Q + i, gi[c]);
          } else {
#pragma unroll
            for (int j = 0; j < Q; ++j) gi[c][j] = g[c * CS + i * Q + j];
          }
        }
      }
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        double d1 = 0.0;
#pragma unroll
        for (int l = 0; l < Q; ++l) d1 = fma(tab[T::D + j * Q + l], x[l], d1);
        const double d0 = work[e * SW + i * QK + j];
        double r0 = d0, r1 = d1;
        if (GK != SPHP_GEOM_NONE) {
          double i00, i01, i10, i11;
          if (GK == SPHP_GEOM_POINT) {
            i00 = gi[0][j];
            i01 = gi[1][j];
            i10 = gi[2][j];
            i11 = gi[3][j];
          } else {
            i00 = g[1];
            i01 = g[2];
            i10 = g[3];
            i11 = g[4];
          }
          r0 = i00 * d0 + i10 * d1;
          r1 = i01 * d0 + i11 * d1;
        }
        o0[j] = r0;
        o1[j] = r1;
      }
      if constexpr (ROT) {
        RowRot<Q>::store(out + e * OUT + i * Q, e * 2 * Q + i, o0);
        RowRot<Q>::store(out + e * OUT + Q2 + i * Q, e * 2 * Q + Q + i, o1);
      } else {
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          out[e * OUT + i * Q + j] = o0[j];
          out[e * OUT + Q2 + i * Q + j] = o1[j];
        }
      }
    }
    __syncthreads();
    release();
  }
};

template <int M_, int Q_, int GK, int NE_, int NT_>
struct QuadIPDeriv {
  static constexpr int M = M_, Q = Q_, NE = NE_, NT = NT_;
  static constexpr int NSTP = SPHP_QUAD_NST;
  static constexpr int M2 = M * M, Q2 = Q * Q;
  static constexpr int IN = 2 * Q2, OUT = M2;
  static constexpr int CS = pt_stride(Q2);
  static constexpr int GEO = (GK == SPHP_GEOM_POINT) ? 5 * CS : (GK == SPHP_GEOM_AFFINE ? 6 : 0);
  static constexpr int QK = odd_up(Q);
  static constexpr int SW = odd_up(Q * QK);
  static constexpr int WORK = 3 * SW;
  using T = Tab<M, Q>;

  template <class R, class W>
  __device__ static void compute(const double* __restrict__ fin, const double* __restrict__ geo,
                                 double* __restrict__ work, double* __restrict__ out, double,
                                 R release, W pre_out, const double* tab) {
    double* W0 = work;
    double* W1 = work + NE * SW;
    double* W2 = work + 2 * NE * SW;
    SPHP_FOR_ITEMS(NE * Q, w) {  // along j: g = wJ inv f ; t = D1^T g1
      int e = w / Q, i = w - e * Q;
      const double* g = geo + e * GEO;
      double g1[Q];
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        const int pt = i * Q + j;
        const double fx = fin[e * IN + pt], fy = fin[e * IN + Q2 + pt];
        double a0, a1;
        if (GK == SPHP_GEOM_NONE) {
          const double wq = tab[T::W + i] * tab[T::W + j];
          a0 = wq * fx;
          a1 = wq * fy;
        } else {
          double wj, i00, i01, i10, i11;
          if (GK == SPHP_GEOM_POINT) {
            wj = g[pt];
            i00 = g[CS + pt];
            i01 = g[2 * CS + pt];
            i10 = g[3 * CS + pt];
            i11 = g[4 * CS + pt];
          } else {
            wj = tab[T::W + i] * tab[T::W + j] * g[0];
            i00 = g[1];
            i01 = g[2];
            i10 = g[3];
            i11 = g[4];
          }
          a0 = wj * (i00 * fx + i01 * fy);
          a1 = wj * (i10 * fx + i11 * fy);
        }
        W1[e * SW + i * QK + j] = a0;
        g1[j] = a1;
      }
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        double t = 0.0;
#pragma unroll
        for (int l = 0; l < Q; ++l) t = fma(tab[T::D + l * Q + j], g1[l], t);
        W0[e * SW + i * QK + j] = t;
      }
    }
    __syncthreads();
    release();
    SPHP_FOR_ITEMS(NE * Q, w) {  // i -> p
      int e = w / Q, j = w - e * Q;
      double t[Q], g0[Q];
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        t[i] = W0[e * SW + i * QK + j];
        g0[i] = W1[e * SW + i * QK + j];
      }
#pragma unroll
      for (int p = 0; p < M; ++p) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          acc = fma(tab[T::B + p * Q + i], t[i], acc);
          acc = fma(tab[T::BD + p * Q + i], g0[i], acc);
        }
        W2[e * SW + p * QK + j] = acc;
      }
    }
    pre_out();
    __syncthreads();
    SPHP_FOR_ITEMS(NE * M, w) {
      int e = w / M, p = w - e * M;
      eo_project<M, Q, 1, 1>(tab, W2 + e * SW + p * QK, out + e * M2 + p * M);
    }
  }
};

}  // namespace sphp
