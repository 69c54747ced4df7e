// Even-odd (parity) evaluation of the 1D operators.
//
// On symmetric GLL points (z[Q-1-i] = -z[i]) the boundary-first Modified_A
// table has mirror structure — rows 0 and 1 swap under z -> -z, bubble k
// has parity (-1)^k — and the collocation derivative is centro-antisymmetric
// (D[Q-1-i][Q-1-j] = -D[i][j]).  Splitting inputs into parity parts halves
// every contraction: an M x Q interpolation becomes (ME + MO) x ceil(Q/2),
// a Q x Q derivative two ceil(Q/2) x ceil(Q/2) products.  Tables: Tab<M,Q>
// BE/BO/BDE/BDO/DE/DO/DTE/DTO (built on the host, api.cu fast_table_pool).
//
//   modes -> parity   xe = [c0+c1, c2, c4, ...], xo = [c1-c0, c3, c5, ...]
//   points -> parity  ve[i] = v[i] + v[Q-1-i] (ve[mid] = v[mid]),
//                     vo[i] = v[i] - v[Q-1-i]
//   merge points      out[i] = E[i] + O[i], out[Q-1-i] = E[i] - O[i]
//   merge modes       c0 = e[0] - o[0], c1 = e[0] + o[0], bubbles by parity
#pragma once
#include "common.cuh"

namespace sphp {

template <int M, int Q>
struct EO {
  using T = Tab<M, Q>;
  static constexpr int H = T::H, HF = T::HF, ME = T::ME, MO = T::MO;

  __device__ static __forceinline__ void split_modes(const double* x, double* xe, double* xo) {
    xe[0] = x[0] + x[1];
    xo[0] = x[1] - x[0];
#pragma unroll
    for (int k = 2; k < M; ++k) {
      if (k % 2 == 0)
        xe[k / 2] = x[k];
      else
        xo[(k - 1) / 2] = x[k];
    }
  }
  __device__ static __forceinline__ void merge_modes(const double* e, const double* o, double* x) {
    x[0] = e[0] - o[0];
    x[1] = e[0] + o[0];
#pragma unroll
    for (int k = 2; k < M; ++k) x[k] = (k % 2 == 0) ? e[k / 2] : o[(k - 1) / 2];
  }
  __device__ static __forceinline__ void split_points(const double* v, double* ve, double* vo) {
#pragma unroll
    for (int i = 0; i < HF; ++i) {
      ve[i] = v[i] + v[Q - 1 - i];
      vo[i] = v[i] - v[Q - 1 - i];
    }
    if constexpr (Q % 2) ve[HF] = v[HF];
  }
  __device__ static __forceinline__ void merge_points(const double* E, const double* O, double* v) {
#pragma unroll
    for (int i = 0; i < HF; ++i) {
      v[i] = E[i] + O[i];
      v[Q - 1 - i] = E[i] - O[i];
    }
    if constexpr (Q % 2) v[HF] = E[HF] + O[HF];
  }

  // u = B^T c (modes -> points)
  __device__ static __forceinline__ void interp(const double* tab, const double* c, double* u) {
    double xe[ME], xo[MO], E[H], O[H];
    split_modes(c, xe, xo);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int r = 0; r < ME; ++r) a = fma(tab[T::BE + r * H + i], xe[r], a);
#pragma unroll
      for (int r = 0; r < MO; ++r) b = fma(tab[T::BO + r * H + i], xo[r], b);
      E[i] = a;
      O[i] = b;
    }
    merge_points(E, O, u);
  }
  // u = B^T c and d = dB^T c from one split
  __device__ static __forceinline__ void interp_and_deriv(const double* tab, const double* c, double* u,
                                                          double* d) {
    double xe[ME], xo[MO], E[H], O[H];
    split_modes(c, xe, xo);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int r = 0; r < ME; ++r) a = fma(tab[T::BE + r * H + i], xe[r], a);
#pragma unroll
      for (int r = 0; r < MO; ++r) b = fma(tab[T::BO + r * H + i], xo[r], b);
      E[i] = a;
      O[i] = b;
    }
    merge_points(E, O, u);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      double a = 0.0, b = 0.0;  // even part from odd inputs, odd part from even inputs
#pragma unroll
      for (int r = 0; r < MO; ++r) a = fma(tab[T::BDO + r * H + i], xo[r], a);
#pragma unroll
      for (int r = 1; r < ME; ++r) b = fma(tab[T::BDE + r * H + i], xe[r], b);
      E[i] = a;
      O[i] = b;
    }
    merge_points(E, O, d);
  }
  // c = B v (points -> modes)
  __device__ static __forceinline__ void project(const double* tab, const double* v, double* c) {
    double ve[H], vo[HF > 0 ? HF : 1], e[ME], o[MO];
    split_points(v, ve, vo);
#pragma unroll
    for (int r = 0; r < ME; ++r) {
      double a = 0.0;
#pragma unroll
      for (int i = 0; i < H; ++i) a = fma(tab[T::BE + r * H + i], ve[i], a);
      e[r] = a;
    }
#pragma unroll
    for (int r = 0; r < MO; ++r) {
      double a = 0.0;
#pragma unroll
      for (int i = 0; i < HF; ++i) a = fma(tab[T::BO + r * H + i], vo[i], a);
      o[r] = a;
    }
    merge_modes(e, o, c);
  }
  // c = B t + dB f (points -> modes, value and derivative tables)
  __device__ static __forceinline__ void project2(const double* tab, const double* t, const double* f,
                                                  double* c) {
    double te[H], to[HF > 0 ? HF : 1], fe[H], fo[HF > 0 ? HF : 1], e[ME], o[MO];
    split_points(t, te, to);
    split_points(f, fe, fo);
#pragma unroll
    for (int r = 0; r < ME; ++r) {
      double a = 0.0;
#pragma unroll
      for (int i = 0; i < H; ++i) a = fma(tab[T::BE + r * H + i], te[i], a);
      if (r > 0) {
#pragma unroll
        for (int i = 0; i < HF; ++i) a = fma(tab[T::BDE + r * H + i], fo[i], a);
      }
      e[r] = a;
    }
#pragma unroll
    for (int r = 0; r < MO; ++r) {
      double a = 0.0;
#pragma unroll
      for (int i = 0; i < HF; ++i) a = fma(tab[T::BO + r * H + i], to[i], a);
#pragma unroll
      for (int i = 0; i < H; ++i) a = fma(tab[T::BDO + r * H + i], fe[i], a);
      o[r] = a;
    }
    merge_modes(e, o, c);
  }
  // out = D v (TR = false) or D^T v (TR = true); ACC adds into out
  template <bool TR, bool ACC>
  __device__ static __forceinline__ void deriv(const double* tab, const double* v, double* out) {
    constexpr int TE = TR ? T::DTE : T::DE;
    constexpr int TO = TR ? T::DTO : T::DO;
    double ve[H], vo[HF > 0 ? HF : 1], E[H], O[H];
    split_points(v, ve, vo);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int j = 0; j < HF; ++j) a = fma(tab[TE + i * HF + j], vo[j], a);
#pragma unroll
      for (int j = 0; j < H; ++j) b = fma(tab[TO + i * H + j], ve[j], b);
      E[i] = a;
      O[i] = b;
    }
    if constexpr (ACC) {
      double r[Q];
      merge_points(E, O, r);
#pragma unroll
      for (int i = 0; i < Q; ++i) out[i] += r[i];
    } else {
      merge_points(E, O, out);
    }
  }
};

// load / store a strided pencil to registers
template <int N, int S>
__device__ __forceinline__ void ld_pencil(const double* __restrict__ p, double* x) {
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] = p[i * S];
}
template <int N, int S>
__device__ __forceinline__ void st_pencil(double* __restrict__ p, const double* x) {
#pragma unroll
  for (int i = 0; i < N; ++i) p[i * S] = x[i];
}


// pencil-level wrappers (drop-in for common.cuh pencil<> with the B / B^T /
// D / D^T tables): load a strided pencil, parity contraction, store
template <int M, int Q, int IS, int OS>
__device__ __forceinline__ void eo_interp(const double* tab, const double* __restrict__ in,
                                          double* __restrict__ out) {
  double x[M], u[Q];
  ld_pencil<M, IS>(in, x);
  EO<M, Q>::interp(tab, x, u);
  st_pencil<Q, OS>(out, u);
}
template <int M, int Q, int IS, int OS>
__device__ __forceinline__ void eo_project(const double* tab, const double* __restrict__ in,
                                           double* __restrict__ out) {
  double v[Q], c[M];
  ld_pencil<Q, IS>(in, v);
  EO<M, Q>::project(tab, v, c);
  st_pencil<M, OS>(out, c);
}
template <int M, int Q, bool TR, bool ACC, int IS, int OS>
__device__ __forceinline__ void eo_deriv(const double* tab, const double* __restrict__ in,
                                         double* __restrict__ out) {
  double v[Q], r[Q];
  ld_pencil<Q, IS>(in, v);
  if constexpr (ACC) ld_pencil<Q, OS>(out, r);
  EO<M, Q>::template deriv<TR, ACC>(tab, v, r);
  st_pencil<Q, OS>(out, r);
}

}  // namespace sphp
