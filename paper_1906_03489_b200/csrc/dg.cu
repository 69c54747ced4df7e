// DG primitives on the device: the batched pieces of
// the reference's DGSystem / AdvectionOperator / ape_rhs that are not
// Collections operators — per-element mass solve, trace extraction, the
// deterministic trace lift, and the pointwise volume / trace fluxes of the
// acoustic (APE) and advection systems.  The Collections operators (BwdTrans,
// IProductWRTBase, IProductWRTDerivBase) come from the fused tile kernels.
//
// All kernels are one thread per output value with a fixed summation order,
// so results are bitwise reproducible.  These are small, latency-bound
// kernels at the reference's DG sizes (E <= 65k quads); they exist to keep
// the DG right-hand side on the device, not as roofline targets.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dg.h"

namespace sphp {

namespace {

constexpr int kBlock = 256;

unsigned blocks_for(int64_t n) { return (unsigned)((n + kBlock - 1) / kBlock); }

// y[e, i] = alpha * sum_j A[e, i, j] (s[e] x[e, j]) (+ y[e, i])
// DGSystem.mass_solve (solvers.py:353-354): einsum("emn,en->em", minv, b)
__global__ void batched_matvec_kernel(int64_t E, int m, int n, const double* __restrict__ A,
                                      const double* __restrict__ x, const double* __restrict__ s,
                                      double alpha, int accumulate, double* __restrict__ y) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= E * m) return;
  const int64_t e = k / m;
  const int i = (int)(k - e * m);
  const double* a = A + (e * m + i) * n;
  const double* xe = x + e * n;
  double acc = 0.0;
  if (s) {
    const double se = s[e];
    for (int j = 0; j < n; ++j) acc = fma(a[j], se * xe[j], acc);
  } else {
    for (int j = 0; j < n; ++j) acc = fma(a[j], xe[j], acc);
  }
  const double v = alpha * acc;
  y[k] = accumulate ? y[k] + v : v;
}

// out[t, q] = sum_n ex[t, q, n] phys[idx[t], n]  (solvers.py:366-372)
__global__ void trace_extract_kernel(int64_t T, int nq, int np, const double* __restrict__ ex,
                                     const int64_t* __restrict__ idx,
                                     const double* __restrict__ phys, double* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= T * nq) return;
  const int64_t t = k / nq;
  const double* row = ex + k * np;
  const double* u = phys + idx[t] * np;
  double acc = 0.0;
  for (int j = 0; j < np; ++j) acc = fma(row[j], u[j], acc);
  out[k] = acc;
}

// b[r, e, n] (+/-)= sum_q L[t, n, q] (w[t, q]) s[r, t, q] over the CSR list
// of element e, in list order (np.add.at order, solvers.py:374-389)
__global__ void trace_lift_kernel(int nrhs, int64_t E, int nm, int nq, int64_t T,
                                  const int64_t* __restrict__ rowp, const int64_t* __restrict__ codes,
                                  const double* __restrict__ Lm, const double* __restrict__ Lp,
                                  const double* __restrict__ w, const double* __restrict__ s,
                                  double* __restrict__ b) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (int64_t)nrhs * E * nm) return;
  const int64_t r = k / (E * nm);
  const int64_t rem = k - r * E * nm;
  const int64_t e = rem / nm;
  const int n = (int)(rem - e * nm);
  const double* sr = s + r * T * nq;
  double acc = b[k];
  for (int64_t c = rowp[e]; c < rowp[e + 1]; ++c) {
    const int64_t code = codes[c];
    const int64_t t = code >> 2;
    const double* L = ((code & 2) ? Lp : Lm) + (t * nm + n) * nq;
    const double* st = sr + t * nq;
    double v = 0.0;
    if (w) {
      const double* wt = w + t * nq;
      for (int q = 0; q < nq; ++q) v = fma(L[q], wt[q] * st[q], v);
    } else {
      for (int q = 0; q < nq; ++q) v = fma(L[q], st[q], v);
    }
    acc = (code & 1) ? acc - v : acc + v;
  }
  b[k] = acc;
}

__device__ __forceinline__ double sgn(double x) { return (double)((x > 0.0) - (x < 0.0)); }

// F(q) . n for the acoustic system (solvers.py:131-139)
__device__ __forceinline__ void ape_fn(double p, double ux, double uy, double nx, double ny,
                                       double bux, double buy, double rho, double c2, double* f) {
  const double un = ux * nx + uy * ny;
  const double ubn = bux * nx + buy * ny;
  const double h = bux * ux + buy * uy + p / rho;
  f[0] = c2 * rho * un + ubn * p;
  f[1] = h * nx;
  f[2] = h * ny;
}

// riemann_flux (solvers.py:142-181) with the ghost states of _ghost_state
// (solvers.py:498-517) for boundary traces; writes sp, sx, sy planes
__global__ void ape_trace_flux_kernel(int64_t npts, int riemann, int bc,
                                      const double* __restrict__ qm, const double* __restrict__ qp,
                                      const double* __restrict__ gv, const double* __restrict__ nrm,
                                      const double* __restrict__ base, const double* __restrict__ w,
                                      double* __restrict__ out, int64_t ostride) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= npts) return;
  const double m0 = qm[k], m1 = qm[npts + k], m2 = qm[2 * npts + k];
  const double nx = nrm[2 * k], ny = nrm[2 * k + 1];
  double p0, p1, p2;
  if (bc == SPHP_BC_INTERIOR) {
    p0 = qp[k];
    p1 = qp[npts + k];
    p2 = qp[2 * npts + k];
  } else if (bc == SPHP_BC_RIGID_WALL) {
    const double un = m1 * nx + m2 * ny;
    p0 = m0;
    p1 = m1 - 2.0 * un * nx;
    p2 = m2 - 2.0 * un * ny;
  } else if (bc == SPHP_BC_FARFIELD) {
    p0 = p1 = p2 = 0.0;
  } else {  // dirichlet on the pressure
    p0 = 2.0 * gv[k] - m0;
    p1 = m1;
    p2 = m2;
  }
  const double bux = base[k], buy = base[npts + k], rho = base[2 * npts + k], c2 = base[3 * npts + k];
  double fm[3], fp[3], out3[3];
  ape_fn(m0, m1, m2, nx, ny, bux, buy, rho, c2, fm);
  ape_fn(p0, p1, p2, nx, ny, bux, buy, rho, c2, fp);
  const double cbar = sqrt(c2);
  const double ubn = bux * nx + buy * ny;
  const double c0 = 0.5 * (fm[0] + fp[0]), c1 = 0.5 * (fm[1] + fp[1]), cc2 = 0.5 * (fm[2] + fp[2]);
  if (riemann == SPHP_RIEMANN_LAXFRIEDRICHS) {
    const double lam = fabs(ubn) + cbar;
    out3[0] = c0 - 0.5 * lam * (p0 - m0);
    out3[1] = c1 - 0.5 * lam * (p1 - m1);
    out3[2] = cc2 - 0.5 * lam * (p2 - m2);
  } else {
    const double tx = -ny, ty = nx;
    const double ubt = bux * tx + buy * ty;
    const double dp = p0 - m0, dux = p1 - m1, duy = p2 - m2;
    const double dun = dux * nx + duy * ny;
    const double dut = dux * tx + duy * ty;
    const double z = rho * cbar;
    const double mu_p = ubn + cbar, mu_m = ubn - cbar;
    const double a_p = fabs(mu_p) * (dp + z * dun) / (2 * z) + sgn(mu_p) * ubt * dut / 2;
    const double a_m = fabs(mu_m) * (dp - z * dun) / (2 * z) - sgn(mu_m) * ubt * dut / 2;
    const double diss_p = a_p * z + a_m * z;
    const double diss_un = a_p - a_m;
    out3[0] = c0 - 0.5 * diss_p;
    out3[1] = c1 - 0.5 * diss_un * nx;
    out3[2] = cc2 - 0.5 * diss_un * ny;
  }
  const double wk = w[k];
  // interior: warc * (F_p / c2) (solvers.py:573-574); boundary:
  // warc * F_p / c2 evaluated left to right (solvers.py:603)
  out[k] = bc == SPHP_BC_INTERIOR ? wk * (out3[0] / c2) : wk * out3[0] / c2;
  out[ostride + k] = wk * out3[1];
  out[2 * ostride + k] = wk * out3[2];
}

// APE volume fluxes (solvers.py:563-569), negated for the three
// -iproduct_deriv calls: G = -(gx, gy), HX = -(h, 0), HY = -(0, h), each
// in the (E, 2, np) layout of IProductWRTDerivBase
__global__ void ape_volume_kernel(int64_t E, int np, const double* __restrict__ q,
                                  const double* __restrict__ base, double* __restrict__ G,
                                  double* __restrict__ HX, double* __restrict__ HY) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t npts = E * np;
  if (k >= npts) return;
  const int64_t e = k / np;
  const int i = (int)(k - e * np);
  const double p = q[k], ux = q[npts + k], uy = q[2 * npts + k];
  const double bux = base[k], buy = base[npts + k], rho = base[2 * npts + k], c2 = base[3 * npts + k];
  const double gx = rho * ux + bux * p / c2;
  const double gy = rho * uy + buy * p / c2;
  const double h = bux * ux + buy * uy + p / rho;
  const int64_t o0 = (e * 2) * np + i, o1 = o0 + np;
  G[o0] = -gx;
  G[o1] = -gy;
  HX[o0] = -h;
  HX[o1] = 0.0;
  HY[o0] = 0.0;
  HY[o1] = -h;
}

// advection volume flux (ax u, ay u) in the (E, 2, np) layout
// (AdvectionOperator.rhs, solvers.py:428-430)
__global__ void advect_volume_kernel(int64_t E, int np, const double* __restrict__ ax,
                                     const double* __restrict__ ay, const double* __restrict__ u,
                                     double* __restrict__ F) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= E * np) return;
  const int64_t e = k / np;
  const int i = (int)(k - e * np);
  F[(e * 2) * np + i] = ax[k] * u[k];
  F[(e * 2 + 1) * np + i] = ay[k] * u[k];
}

// upwind advection trace flux an * (an >= 0 ? um : up) with the boundary
// ghost values of solvers.py:441-455 (dirichlet 2g - um, farfield 0)
__global__ void advect_trace_flux_kernel(int64_t npts, int bc, const double* __restrict__ an,
                                         const double* __restrict__ um,
                                         const double* __restrict__ up,
                                         const double* __restrict__ gv, double* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= npts) return;
  const double m = um[k];
  double p;
  if (bc == SPHP_BC_INTERIOR)
    p = up[k];
  else if (bc == SPHP_BC_DIRICHLET)
    p = 2.0 * gv[k] - m;
  else
    p = 0.0;
  const double a = an[k];
  out[k] = a * (a >= 0 ? m : p);
}

// rp = c[k] * v[k] (+ src[k]): the pointwise c2 branch of ape_rhs
// (solvers.py:621-624) with c = -c2
__global__ void scale_points_kernel(int64_t n, const double* __restrict__ c,
                                    const double* __restrict__ v, const double* __restrict__ src,
                                    double* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double r = c[k] * v[k];
  out[k] = src ? r + src[k] : r;
}

}  // namespace

cudaError_t batched_matvec(int64_t E, int m, int n, const double* A, const double* x,
                           const double* s, double alpha, int accumulate, double* y,
                           cudaStream_t st) {
  if (E * m == 0) return cudaSuccess;
  batched_matvec_kernel<<<blocks_for(E * m), kBlock, 0, st>>>(E, m, n, A, x, s, alpha, accumulate, y);
  return cudaGetLastError();
}

cudaError_t trace_extract(int64_t T, int nq, int np, const double* ex, const int64_t* idx,
                          const double* phys, double* out, cudaStream_t st) {
  if (T * nq == 0) return cudaSuccess;
  trace_extract_kernel<<<blocks_for(T * nq), kBlock, 0, st>>>(T, nq, np, ex, idx, phys, out);
  return cudaGetLastError();
}

cudaError_t trace_lift(int nrhs, int64_t E, int nm, int nq, int64_t T, const int64_t* rowp,
                       const int64_t* codes, const double* Lm, const double* Lp, const double* w,
                       const double* s, double* b, cudaStream_t st) {
  const int64_t n = (int64_t)nrhs * E * nm;
  if (n == 0) return cudaSuccess;
  trace_lift_kernel<<<blocks_for(n), kBlock, 0, st>>>(nrhs, E, nm, nq, T, rowp, codes, Lm, Lp, w, s, b);
  return cudaGetLastError();
}

cudaError_t ape_trace_flux(int64_t npts, int riemann, int bc, const double* qm, const double* qp,
                           const double* gv, const double* nrm, const double* base,
                           const double* w, double* out, int64_t ostride, cudaStream_t st) {
  if (npts == 0) return cudaSuccess;
  ape_trace_flux_kernel<<<blocks_for(npts), kBlock, 0, st>>>(npts, riemann, bc, qm, qp, gv, nrm,
                                                             base, w, out, ostride);
  return cudaGetLastError();
}

cudaError_t ape_volume(int64_t E, int np, const double* q, const double* base, double* G,
                       double* HX, double* HY, cudaStream_t st) {
  if (E * np == 0) return cudaSuccess;
  ape_volume_kernel<<<blocks_for(E * np), kBlock, 0, st>>>(E, np, q, base, G, HX, HY);
  return cudaGetLastError();
}

cudaError_t advect_volume(int64_t E, int np, const double* ax, const double* ay, const double* u,
                          double* F, cudaStream_t st) {
  if (E * np == 0) return cudaSuccess;
  advect_volume_kernel<<<blocks_for(E * np), kBlock, 0, st>>>(E, np, ax, ay, u, F);
  return cudaGetLastError();
}

cudaError_t advect_trace_flux(int64_t npts, int bc, const double* an, const double* um,
                              const double* up, const double* gv, double* out, cudaStream_t st) {
  if (npts == 0) return cudaSuccess;
  advect_trace_flux_kernel<<<blocks_for(npts), kBlock, 0, st>>>(npts, bc, an, um, up, gv, out);
  return cudaGetLastError();
}

cudaError_t scale_points(int64_t n, const double* c, const double* v, const double* src, double* out,
                         cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  scale_points_kernel<<<blocks_for(n), kBlock, 0, st>>>(n, c, v, src, out);
  return cudaGetLastError();
}

}  // namespace sphp
