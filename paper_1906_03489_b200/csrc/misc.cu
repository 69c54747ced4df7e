// Non-sum-factorisation device code:
//   * analytic geometric factors (geometry.py:115-142 semantics) for the
//     structured BASELINE meshes, and conversion of reference GeomFactors;
//   * signed scatter / colour-ordered assemble (assembly.py:141-160);
//   * the StdMat strategy (collections.py:203-229): a register-tiled FP64
//     GEMM for the dense elemental operators, plus the pointwise helpers and
//     the per-element matrix-vector product of the dense Helmholtz operator.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/spechp_b200.h"
#include "common.cuh"
#include "misc.h"
#include "periodic.cuh"

namespace sphp {

// ---------------------------------------------------------------------------
// geometry
// ---------------------------------------------------------------------------
__device__ __forceinline__ void affine_index(int64_t id, int n, int dim, int* idx) {
  for (int a = 0; a < dim; ++a) {
    idx[a] = (int)(id % n);
    id /= n;
  }
}

__global__ void geom_analytic_kernel(GeomJob j, int* bad) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int dim = j.dim;
  const int64_t npts = j.npts;
  const int64_t total = (j.kind == SPHP_GEOM_AFFINE) ? j.E : j.E * npts;
  if (tid >= total) return;
  const int64_t el = (j.kind == SPHP_GEOM_AFFINE) ? tid : tid / npts;
  const int pt = (j.kind == SPHP_GEOM_AFFINE) ? 0 : (int)(tid - el * npts);
  const int64_t id = j.ids ? j.ids[el] : j.e0 + el;
  int idx[3] = {0, 0, 0};
  affine_index(id, j.n, dim, idx);
  // point (i, j[, k]) with the first direction slowest
  int pi[3] = {0, 0, 0};
  {
    int rem = pt;
    for (int a = dim - 1; a >= 0; --a) {
      pi[a] = rem % j.Q;
      rem /= j.Q;
    }
  }
  double x[3], h[3], wq = 1.0;
  for (int a = 0; a < dim; ++a) {
    h[a] = j.L[a] / j.n;
    const double z = (j.kind == SPHP_GEOM_AFFINE) ? 0.0 : j.z[pi[a]];
    x[a] = (idx[a] + 0.5 * (z + 1.0)) * h[a];
    wq *= j.w[pi[a]];
  }
  // jac[k][a] = dx_k / dxi_a
  double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int a = 0; a < dim; ++a) J[a][a] = 0.5 * h[a];
  const double tp = 6.283185307179586;
  if (j.mapping == SPHP_MAP_QUAD_SINE) {
    J[0][1] = j.amp * tp * cos(tp * x[1]) * 0.5 * h[1];
    J[1][0] = j.amp * tp * cos(tp * x[0]) * 0.5 * h[0];
  } else if (j.mapping == SPHP_MAP_HEX_SINE) {
    J[0][1] = j.amp * tp * cos(tp * x[1]) * sin(tp * x[2]) * 0.5 * h[1];
    J[0][2] = j.amp * tp * sin(tp * x[1]) * cos(tp * x[2]) * 0.5 * h[2];
  }
  double det, inv[3][3];
  if (dim == 2) {
    det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    inv[0][0] = J[1][1] / det;
    inv[0][1] = -J[0][1] / det;
    inv[1][0] = -J[1][0] / det;
    inv[1][1] = J[0][0] / det;
  } else {
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    inv[0][0] = c00 / det;
    inv[1][0] = c01 / det;
    inv[2][0] = c02 / det;
    inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
    inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
    inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
    inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
    inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
    inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  }
  if (!(det > 0.0)) atomicExch(bad, 1);
  double* rec = j.out + el * j.stride;
  const int64_t cs = j.cs;
  if (j.kind == SPHP_GEOM_AFFINE) {
    rec[0] = det;
    int c = 1;
    for (int a = 0; a < dim; ++a)
      for (int k = 0; k < dim; ++k) rec[c++] = inv[a][k];
    for (; c < j.stride; ++c) rec[c] = 0.0;
  } else if (j.kind == SPHP_GEOM_POINT) {
    rec[pt] = wq * det;
    int c = 1;
    for (int a = 0; a < dim; ++a)
      for (int k = 0; k < dim; ++k) rec[(c++) * cs + pt] = inv[a][k];
  } else {  // METRIC: G_ab = wJ sum_k inv[a,k] inv[b,k]
    const double wj = wq * det;
    const int ms = metric_slot(dim, j.Q, pt);
    int c = 0;
    for (int a = 0; a < dim; ++a)
      for (int b = a; b < dim; ++b) {
        double g = 0.0;
        for (int k = 0; k < dim; ++k) g += inv[a][k] * inv[b][k];
        rec[(c++) * cs + ms] = wj * g;
      }
    rec[c * cs + ms] = wj;
  }
}

cudaError_t geom_analytic(const GeomJob& j, int* bad, cudaStream_t s) {
  const int64_t total = (j.kind == SPHP_GEOM_AFFINE) ? j.E : j.E * j.npts;
  if (total == 0) return cudaSuccess;
  const int T = 256;
  geom_analytic_kernel<<<(unsigned)((total + T - 1) / T), T, 0, s>>>(j, bad);
  return cudaGetLastError();
}

// reference GeomFactors arrays (wj (E,np), inv (E,np,d,d)) -> encoding
__global__ void geom_convert_kernel(GeomJob j, const double* wj, const double* inv, int* bad) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int dim = j.dim;
  const int64_t np = j.npts;
  if (tid >= j.E * np) return;
  const int64_t el = tid / np;
  const int pt = (int)(tid - el * np);
  const double w = wj[tid];
  const double* iv = inv + tid * dim * dim;
  if (!(w > 0.0)) atomicExch(bad, 1);
  double* rec = j.out + el * j.stride;
  const int64_t cs = j.cs;
  if (j.kind == SPHP_GEOM_POINT) {
    rec[pt] = w;
    for (int c = 0; c < dim * dim; ++c) rec[(1 + c) * cs + pt] = iv[c];
  } else {
    const int ms = metric_slot(dim, j.Q, pt);
    int c = 0;
    for (int a = 0; a < dim; ++a)
      for (int b = a; b < dim; ++b) {
        double g = 0.0;
        for (int k = 0; k < dim; ++k) g += iv[a * dim + k] * iv[b * dim + k];
        rec[(c++) * cs + ms] = w * g;
      }
    rec[c * cs + ms] = w;
  }
}

cudaError_t geom_convert(const GeomJob& j, const double* wj, const double* inv, int* bad,
                         cudaStream_t s) {
  const int64_t total = j.E * j.npts;
  if (total == 0) return cudaSuccess;
  geom_convert_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(j, wj, inv, bad);
  return cudaGetLastError();
}

// geometry.geom_factors (geometry.py:125-142) from the reference-direction
// derivatives of the coordinate map at the quadrature points: jac[k][a] =
// dx_k / dxi_a, det, inv[a][k] = dxi_a / dx_k, wj = w det.  bad[0] counts
// points with det <= 0, bad[1] keeps the first such element.
__global__ void jacobian_factors_kernel(int64_t E, int64_t np, const double* __restrict__ dx,
                                        const double* __restrict__ dy, const double* __restrict__ w,
                                        double* __restrict__ wj, double* __restrict__ inv,
                                        unsigned long long* bad) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= E * np) return;
  const int64_t e = tid / np, i = tid - e * np;
  const double j00 = dx[(e * 2) * np + i], j01 = dx[(e * 2 + 1) * np + i];
  const double j10 = dy[(e * 2) * np + i], j11 = dy[(e * 2 + 1) * np + i];
  const double det = j00 * j11 - j01 * j10;
  if (!(det > 0.0)) {
    atomicAdd(&bad[0], 1ull);
    atomicMin(&bad[1], (unsigned long long)e);
  }
  double* iv = inv + tid * 4;
  iv[0] = j11 / det;
  iv[1] = -j01 / det;
  iv[2] = -j10 / det;
  iv[3] = j00 / det;
  wj[tid] = w[i] * det;
}

cudaError_t jacobian_factors(int64_t E, int64_t np, const double* dx, const double* dy,
                             const double* w, double* wj, double* inv, unsigned long long* bad,
                             cudaStream_t s) {
  const int64_t total = E * np;
  if (total == 0) return cudaSuccess;
  jacobian_factors_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(E, np, dx, dy, w, wj, inv, bad);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// assembly: scatter (global -> local) and colour-ordered assemble
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t hexp_gid(int n, int P, int64_t e, int nl) {
  const int m = P + 1;
  const int p = nl / (m * m), q = (nl / m) % m, r = nl % m;
  const int ex = (int)(e % n), ey = (int)((e / n) % n), ez = (int)(e / ((int64_t)n * n));
  const int64_t N3 = (int64_t)n * n * n;
  const int64_t b = P - 1;
  int idx[3] = {p, q, r};
  int base[3] = {ex, ey, ez};
  const int nb = (p >= 2) + (q >= 2) + (r >= 2);
  auto wrap = [n](int i) { return i >= n ? i - n : i; };
  if (nb == 0) return wrap(ex + p) + (int64_t)n * (wrap(ey + q) + (int64_t)n * wrap(ez + r));
  if (nb == 1) {
    const int d = (p >= 2) ? 0 : ((q >= 2) ? 1 : 2);
    int c[3];
    for (int a = 0; a < 3; ++a) c[a] = wrap(base[a] + (a == d ? 0 : idx[a]));
    return N3 + (d * N3 + c[0] + (int64_t)n * (c[1] + (int64_t)n * c[2])) * b + (idx[d] - 2);
  }
  if (nb == 2) {
    const int d = (p < 2) ? 0 : ((q < 2) ? 1 : 2);
    int c[3];
    for (int a = 0; a < 3; ++a) c[a] = wrap(base[a] + (a == d ? idx[a] : 0));
    const int k1 = (d == 0) ? q : p, k2 = (d == 2) ? q : r;
    return N3 + 3 * N3 * b + (d * N3 + c[0] + (int64_t)n * (c[1] + (int64_t)n * c[2])) * b * b +
           (k1 - 2) * b + (k2 - 2);
  }
  return N3 * (1 + 3 * b + 3 * b * b) + e * b * b * b + ((int64_t)(p - 2) * b + (q - 2)) * b + (r - 2);
}

__device__ __forceinline__ void map_entry(const AmapDev& m, int64_t e, int nl, int64_t& gid,
                                          double& sg) {
  if (m.periodic) {
    gid = hexp_gid(m.n, m.P, e, nl);
    sg = 1.0;
    return;
  }
  const int c = m.codes[e * m.nm + nl];
  if (c >= 0) {
    gid = c;
    sg = 1.0;
  } else if (c == -1) {
    gid = -1;
    sg = 0.0;
  } else {
    gid = -(int64_t)c - 2;
    sg = -1.0;
  }
}

cudaError_t periodic_scatter(int n, int P, const double* g, double* loc, cudaStream_t s);

__global__ void scatter_kernel(AmapDev m, const double* __restrict__ g, double* __restrict__ loc) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= m.E * m.nm) return;
  const int64_t e = tid / m.nm;
  const int nl = (int)(tid - e * m.nm);
  int64_t gid;
  double sg;
  map_entry(m, e, nl, gid, sg);
  loc[tid] = gid >= 0 ? sg * g[gid] : 0.0;
}

// explicit maps: local entry i maps to code i (element-major), so the
// scatter is a flat signed gather; 4 entries per thread (one 16-byte code
// load, four independent gathers in flight, two 16-byte stores)
__device__ __forceinline__ double signed_gather(const double* __restrict__ g, int c) {
  return c >= 0 ? __ldg(g + c) : (c == -1 ? 0.0 : -__ldg(g + (-(int64_t)c - 2)));
}
__global__ void __launch_bounds__(256) scatter_explicit_kernel(int64_t total, const int* __restrict__ codes,
                                                               const double* __restrict__ g,
                                                               double* __restrict__ loc) {
  const int64_t n4 = total >> 2;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
    const int4 c = __ldg(reinterpret_cast<const int4*>(codes) + q);
    const double v0 = signed_gather(g, c.x), v1 = signed_gather(g, c.y);
    const double v2 = signed_gather(g, c.z), v3 = signed_gather(g, c.w);
    reinterpret_cast<double2*>(loc)[2 * q] = make_double2(v0, v1);
    reinterpret_cast<double2*>(loc)[2 * q + 1] = make_double2(v2, v3);
  }
  const int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) loc[i] = signed_gather(g, codes[i]);
}

// one colour class: exclusive ownership of every touched global dof
__global__ void assemble_colour_kernel(AmapDev m, const double* __restrict__ loc,
                                       double* __restrict__ g, int colour, const int* elist,
                                       int64_t nlist) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= nlist * m.nm) return;
  const int64_t w = tid / m.nm;
  const int nl = (int)(tid - w * m.nm);
  int64_t e;
  if (m.periodic) {
    const int h = m.n >> 1;
    const int ex = 2 * (int)(w % h) + (colour & 1);
    const int ey = 2 * (int)((w / h) % h) + ((colour >> 1) & 1);
    const int ez = 2 * (int)(w / ((int64_t)h * h)) + ((colour >> 2) & 1);
    e = ex + (int64_t)m.n * (ey + (int64_t)m.n * ez);
  } else {
    e = elist[w];
  }
  int64_t gid;
  double sg;
  map_entry(m, e, nl, gid, sg);
  if (gid >= 0) g[gid] += sg * loc[e * m.nm + nl];
}

cudaError_t amap_scatter(const AmapDev& m, const double* g, double* loc, cudaStream_t s, int* ctr) {
  if (m.periodic) {
    cudaError_t e = periodic_scatter_v2(m.n, m.P, g, loc, s, 0, -1, ctr);
    return e == cudaErrorNotSupported ? periodic_scatter(m.n, m.P, g, loc, s) : e;
  }
  const int64_t total = m.E * m.nm;
  if (total == 0) return cudaSuccess;
  if ((reinterpret_cast<uintptr_t>(loc) & 15) == 0 && (reinterpret_cast<uintptr_t>(m.codes) & 15) == 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (total / 4 + 255) / 256;
    const int64_t cap = (int64_t)sms * 8;
    scatter_explicit_kernel<<<(unsigned)(want < cap ? (want > 0 ? want : 1) : cap), 256, 0, s>>>(
        total, m.codes, g, loc);
    return cudaGetLastError();
  }
  scatter_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(m, g, loc);
  return cudaGetLastError();
}

cudaError_t amap_assemble(const AmapDev& m, const double* loc, double* g, int ncolours,
                          const int* elist_dev, const int64_t* colour_off, int accumulate,
                          cudaStream_t s) {
  cudaError_t err = cudaSuccess;
  if (!accumulate) {
    err = cudaMemsetAsync(g, 0, sizeof(double) * m.num_global, s);
    if (err != cudaSuccess) return err;
  }
  for (int c = 0; c < ncolours; ++c) {
    int64_t nlist;
    const int* el = nullptr;
    if (m.periodic) {
      nlist = (int64_t)(m.n / 2) * (m.n / 2) * (m.n / 2);
    } else {
      nlist = colour_off[c + 1] - colour_off[c];
      el = elist_dev + colour_off[c];
    }
    const int64_t total = nlist * m.nm;
    if (total == 0) continue;
    assemble_colour_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(m, loc, g, c, el, nlist);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// StdMat: C (R x N) = A (R x K) * B (K x N), all row-major FP64.
// 64x64 CTA tiles, K chunks of 16, 256 threads x (4x4) register tile.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) dgemm_kernel(int64_t R, int N, int K, const double* __restrict__ A,
                                                    const double* __restrict__ B, double* __restrict__ C) {
  __shared__ double As[16][64 + 1];
  __shared__ double Bs[16][64];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t row0 = (int64_t)blockIdx.y * 64;
  const int col0 = blockIdx.x * 64;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int r = i / 16, kk = i % 16;
      const int64_t gr = row0 + r;
      As[kk][r] = (gr < R && k0 + kk < K) ? A[gr * K + k0 + kk] : 0.0;
      const int kb = i / 64, c = i % 64;
      Bs[kb][c] = (k0 + kb < K && col0 + c < N) ? B[(int64_t)(k0 + kb) * N + col0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) b[jj] = Bs[kk][tx + 16 * jj];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj] = fma(a[i], b[jj], acc[i][jj]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = row0 + ty + 16 * i;
    if (r >= R) continue;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int c = col0 + tx + 16 * jj;
      if (c < N) C[r * N + c] = acc[i][jj];
    }
  }
}

cudaError_t dgemm(int64_t R, int N, int K, const double* A, const double* B, double* C,
                  cudaStream_t s) {
  if (R == 0) return cudaSuccess;
  const int64_t gy = (R + 63) / 64;
  if (gy > 65535) {
    // split rows into chunks the grid can address
    for (int64_t r0 = 0; r0 < R; r0 += 65535 * 64) {
      const int64_t rr = (R - r0) < 65535 * 64 ? (R - r0) : 65535 * 64;
      cudaError_t err = dgemm(rr, N, K, A + r0 * K, B, C + r0 * N, s);
      if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
  }
  dim3 grid((N + 63) / 64, (unsigned)gy);
  dgemm_kernel<<<grid, 256, 0, s>>>(R, N, K, A, B, C);
  return cudaGetLastError();
}

// pointwise helpers of the StdMat strategy ---------------------------------
// IProduct: W u with W from the geometry encoding (collections.py:216)
__global__ void weight_kernel(PointJob j, const double* __restrict__ u, double* __restrict__ o) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= j.E * j.np) return;
  const int64_t e = tid / j.np;
  const int pt = (int)(tid - e * j.np);
  double w;
  if (j.kind == SPHP_GEOM_POINT)
    w = j.geom[e * j.stride + pt];
  else if (j.kind == SPHP_GEOM_AFFINE)
    w = j.wstd[pt] * j.geom[e * j.stride];
  else
    w = j.wstd[pt];
  o[tid] = w * u[tid];
}

// PhysDeriv metric transform in place on (E, d, np) (collections.py:181-185)
__global__ void metric_kernel(PointJob j, double* __restrict__ d) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= j.E * j.np) return;
  const int64_t e = tid / j.np;
  const int pt = (int)(tid - e * j.np);
  const int dim = j.dim;
  double v[3], o[3], iv[9];
  for (int a = 0; a < dim; ++a) v[a] = d[(e * dim + a) * j.np + pt];
  for (int c = 0; c < dim * dim; ++c)
    iv[c] = (j.kind == SPHP_GEOM_POINT) ? j.geom[e * j.stride + (1 + c) * j.cs + pt]
                                        : j.geom[e * j.stride + 1 + c];
  for (int k = 0; k < dim; ++k) {
    double s = 0.0;
    for (int a = 0; a < dim; ++a) s += iv[a * dim + k] * v[a];
    o[k] = s;
  }
  for (int k = 0; k < dim; ++k) d[(e * dim + k) * j.np + pt] = o[k];
}

// IProductWRTDerivBase pointwise: g_a = wJ sum_k inv[a,k] f_k  (geometry.py:166-167)
__global__ void flux_kernel(PointJob j, const double* __restrict__ f, double* __restrict__ g) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= j.E * j.np) return;
  const int64_t e = tid / j.np;
  const int pt = (int)(tid - e * j.np);
  const int dim = j.dim;
  double v[3];
  for (int k = 0; k < dim; ++k) v[k] = f[(e * dim + k) * j.np + pt];
  double w, iv[9];
  if (j.kind == SPHP_GEOM_POINT) {
    w = j.geom[e * j.stride + pt];
    for (int c = 0; c < dim * dim; ++c) iv[c] = j.geom[e * j.stride + (1 + c) * j.cs + pt];
  } else if (j.kind == SPHP_GEOM_AFFINE) {
    w = j.wstd[pt] * j.geom[e * j.stride];
    for (int c = 0; c < dim * dim; ++c) iv[c] = j.geom[e * j.stride + 1 + c];
  } else {
    w = j.wstd[pt];
    for (int c = 0; c < dim * dim; ++c) iv[c] = (c / dim == c % dim) ? 1.0 : 0.0;
  }
  for (int a = 0; a < dim; ++a) {
    double s = 0.0;
    for (int k = 0; k < dim; ++k) s += iv[a * dim + k] * v[k];
    g[(e * dim + a) * j.np + pt] = w * s;
  }
}

cudaError_t pointwise(int which, const PointJob& j, const double* in, double* out,
                      cudaStream_t s) {
  const int64_t total = j.E * j.np;
  if (total == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((total + 255) / 256);
  if (which == 0)
    weight_kernel<<<grid, 256, 0, s>>>(j, in, out);
  else if (which == 1)
    metric_kernel<<<grid, 256, 0, s>>>(j, out);
  else
    flux_kernel<<<grid, 256, 0, s>>>(j, in, out);
  return cudaGetLastError();
}

// dense elemental Helmholtz: y_e = H_e x_e, H_e symmetric (nm x nm)
__global__ void elem_matvec_kernel(int64_t E, int nm, const double* __restrict__ H,
                                   const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ double xs[];
  const int64_t e = blockIdx.x;
  for (int i = threadIdx.x; i < nm; i += blockDim.x) xs[i] = x[e * nm + i];
  __syncthreads();
  const double* He = H + e * (int64_t)nm * nm;
  for (int r = threadIdx.x; r < nm; r += blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < nm; ++c) acc = fma(He[(int64_t)c * nm + r], xs[c], acc);  // H sym: column read
    y[e * nm + r] = acc;
  }
}

cudaError_t elem_matvec(int64_t E, int nm, const double* H, const double* x, double* y,
                        cudaStream_t s) {
  if (E == 0) return cudaSuccess;
  int T = nm < 32 ? 32 : (nm > 256 ? 256 : ((nm + 31) / 32) * 32);
  elem_matvec_kernel<<<(unsigned)E, T, sizeof(double) * nm, s>>>(E, nm, H, x, y);
  return cudaGetLastError();
}

// unit-vector input for column n of every element, and symmetrisation
__global__ void unit_kernel(int64_t E, int nm, int n, double* x) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= E * nm) return;
  x[tid] = ((int)(tid % nm) == n) ? 1.0 : 0.0;
}
__global__ void column_kernel(int64_t E, int nm, int n, const double* y, double* H) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= E * nm) return;
  const int64_t e = tid / nm;
  const int r = (int)(tid - e * nm);
  H[e * (int64_t)nm * nm + (int64_t)n * nm + r] = y[tid];  // column n stored contiguously
}
__global__ void symmetrise_kernel(int64_t E, int nm, double* H) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= E * nm * nm) return;
  const int64_t e = tid / ((int64_t)nm * nm);
  const int rc = (int)(tid - e * nm * nm);
  const int r = rc / nm, c = rc % nm;
  if (c <= r) return;
  double* He = H + e * (int64_t)nm * nm;
  const double v = 0.5 * (He[r * nm + c] + He[c * nm + r]);
  He[r * nm + c] = v;
  He[c * nm + r] = v;
}

cudaError_t unit_block(int64_t E, int nm, int n, double* x, cudaStream_t s) {
  unit_kernel<<<(unsigned)((E * nm + 255) / 256), 256, 0, s>>>(E, nm, n, x);
  return cudaGetLastError();
}
cudaError_t store_column(int64_t E, int nm, int n, const double* y, double* H, cudaStream_t s) {
  column_kernel<<<(unsigned)((E * nm + 255) / 256), 256, 0, s>>>(E, nm, n, y, H);
  return cudaGetLastError();
}
cudaError_t symmetrise(int64_t E, int nm, double* H, cudaStream_t s) {
  const int64_t total = E * (int64_t)nm * nm;
  symmetrise_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(E, nm, H);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// owner-computes assembly (deterministic, no atomics, no colour passes):
// every global dof is summed by one thread from its contributing local
// entries in a fixed order.  Periodic hex: element (ex,ey,ez) owns its
// lower vertex, the 3 edges and 3 faces leaving it, and its interior —
// P^3 dofs — and threads walk elements in id order so the neighbour
// blocks they read stay in L2.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 6) owner_periodic_kernel(int n, int P, const double* __restrict__ loc,
                                                             double* __restrict__ y, int accumulate,
                                                             int mode_major) {
  // block = 32 consecutive elements along x (lanes) for one (ey, ez) row
  // segment; warp w walks owned dofs o = w, w+8, ...: every warp-level branch
  // below is uniform, and the neighbour blocks a CTA reads stay in L1/L2
  const int segs = (n + 31) / 32;
  const int seg = blockIdx.x % segs;
  const int row = blockIdx.x / segs;  // ey + n*ez
  const int ey = row % n, ez = row / n;
  const int ex = seg * 32 + (threadIdx.x & 31);
  if (ex >= n) return;
  const int N3 = n * n * n, b = P - 1, m = P + 1, nm = m * m * m, per = P * P * P;
  const int e = ex + n * row;
  auto wrapm = [n](int i) { return i < 0 ? i + n : i; };
  auto eid = [&](int i, int j, int k) { return wrapm(i) + n * (wrapm(j) + n * wrapm(k)); };
  auto flat = [m](int p, int q, int r) { return (p * m + q) * m + r; };
  // local entry (element, mode): element-major e*nm + nl, or mode-major
  // nl*N3 + e (written by the gathering fused kernel; coalesced here)
  auto at = [&](int el, int nl) -> double {
    return mode_major ? loc[(size_t)nl * N3 + el] : loc[(size_t)el * nm + nl];
  };
  const int base[3] = {ex, ey, ez};
  for (int o = threadIdx.x >> 5; o < per; o += blockDim.x >> 5) {
    double acc = 0.0;
    int gid;
    int oo = o;
    if (oo == 0) {  // vertex: 8 elements, local corner (a, bb, c)
      gid = e;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
#pragma unroll
          for (int c = 0; c < 2; ++c)
            acc += at(eid(ex - a, ey - bb, ez - c), flat(a, bb, c));
    } else if ((oo -= 1) < 3 * b) {  // edge leaving the vertex along d, degree k
      const int d = oo / b, k = oo - d * b + 2;
      gid = N3 + (d * N3 + e) * b + (k - 2);
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          int c[3], idx[3];
          const int st[2] = {s, t};
          int w = 0;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            if (a == d) {
              c[a] = base[a];
              idx[a] = k;
            } else {
              c[a] = base[a] - st[w];
              idx[a] = st[w++];
            }
          }
          acc += at(eid(c[0], c[1], c[2]), flat(idx[0], idx[1], idx[2]));
        }
    } else if ((oo -= 3 * b) < 3 * b * b) {  // face normal d at the vertex
      const int d = oo / (b * b), r2 = oo - d * b * b;
      const int k1 = r2 / b + 2, k2 = r2 - (k1 - 2) * b + 2;
      gid = N3 + 3 * N3 * b + (d * N3 + e) * b * b + (k1 - 2) * b + (k2 - 2);
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        int c[3], idx[3];
        const int kk[2] = {k1, k2};
        int w = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (a == d) {
            c[a] = base[a] - side;
            idx[a] = side;
          } else {
            c[a] = base[a];
            idx[a] = kk[w++];
          }
        }
        acc += at(eid(c[0], c[1], c[2]), flat(idx[0], idx[1], idx[2]));
      }
    } else {  // interior, owned by the element alone
      oo -= 3 * b * b;
      const int p = oo / (b * b) + 2, q = (oo / b) % b + 2, r = oo % b + 2;
      gid = N3 * (1 + 3 * b + 3 * b * b) + e * b * b * b + oo;
      acc = at(e, flat(p, q, r));
    }
    y[gid] = accumulate ? y[gid] + acc : acc;
  }
}

// explicit maps: CSR rows over global dofs, entries = local index, negative
// (-(idx+1)) for sign -1; rows sorted by local index (element order)
__global__ void owner_csr_kernel(int64_t ng, const int64_t* __restrict__ rowp,
                                 const int* __restrict__ ent, const double* __restrict__ loc,
                                 double* __restrict__ y, int accumulate, int nm, int64_t E,
                                 int mode_major) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  double acc = 0.0;
  for (int64_t k = rowp[g]; k < rowp[g + 1]; ++k) {
    const int c = ent[k];
    const int64_t i = c >= 0 ? c : -(int64_t)c - 1;  // element-major local index
    const int64_t j = mode_major ? (i % nm) * E + i / nm : i;
    acc += c >= 0 ? loc[j] : -loc[j];
  }
  y[g] = accumulate ? y[g] + acc : acc;
}

cudaError_t owner_assemble_periodic(int n, int P, const double* loc, double* y, int accumulate,
                                    int mode_major, cudaStream_t s, int* ctr) {
  if (!mode_major) {
    cudaError_t e = owner_periodic_v3(n, P, loc, y, accumulate, s, 0, -1, ctr);
    if (e != cudaErrorNotSupported) return e;
  }
  if (n == 0) return cudaSuccess;
  const int64_t blocks = (int64_t)((n + 31) / 32) * n * n;
  owner_periodic_kernel<<<(unsigned)blocks, 256, 0, s>>>(n, P, loc, y, accumulate, mode_major);
  return cudaGetLastError();
}

// several batches: entries index the concatenation of the batches' local
// blocks (int32 rows and entries); one pass over the global dofs
__global__ void owner_csr32_kernel(int64_t ng, const int* __restrict__ rowp, const int* __restrict__ ent,
                                   const double* __restrict__ loc, double* __restrict__ y) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int k0 = __ldg(rowp + g), k1 = __ldg(rowp + g + 1);
  double acc = 0.0;
  for (int k = k0; k < k1; ++k) {
    const int c = __ldg(ent + k);
    acc += c >= 0 ? __ldg(loc + c) : -__ldg(loc + (-(int64_t)c - 1));
  }
  y[g] = acc;
}

cudaError_t owner_assemble_csr32(int64_t ng, const int* rowp, const int* ent, const double* loc, double* y,
                                 cudaStream_t s) {
  if (ng == 0) return cudaSuccess;
  owner_csr32_kernel<<<(unsigned)((ng + 255) / 256), 256, 0, s>>>(ng, rowp, ent, loc, y);
  return cudaGetLastError();
}

cudaError_t owner_assemble_csr(int64_t ng, const int64_t* rowp, const int* ent, const double* loc,
                               double* y, int accumulate, int nm, int64_t E, int mode_major,
                               cudaStream_t s) {
  if (ng == 0) return cudaSuccess;
  owner_csr_kernel<<<(unsigned)((ng + 255) / 256), 256, 0, s>>>(ng, rowp, ent, loc, y, accumulate, nm,
                                                                E, mode_major);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// periodic scatter (global -> local block), entity-based int32 indexing:
// a CTA takes EB consecutive elements, builds their 27 entity bases and the
// per-mode code table in shared memory, then writes the local block in
// order (coalesced stores; the x reads hit L2 for neighbouring elements)
// ---------------------------------------------------------------------------
constexpr int SC_EB = 8;
__global__ void __launch_bounds__(256) periodic_scatter_kernel(int n, int P, const double* __restrict__ g,
                                                               double* __restrict__ loc) {
  extern __shared__ int sh[];
  const int m = P + 1, nm = m * m * m;
  int* ent = sh;                // SC_EB * 27
  int* mtab = sh + SC_EB * 27;  // nm
  const int N3 = n * n * n;
  const int e0 = blockIdx.x * SC_EB;
  for (int i = threadIdx.x; i < nm; i += blockDim.x) mtab[i] = mode_code(m, i);
  for (int i = threadIdx.x; i < SC_EB * 27; i += blockDim.x) {
    const int e = e0 + i / 27, k = i % 27;
    int v = 0;
    if (e < N3) v = entity_base(n, P, e % n, (e / n) % n, e / (n * n), k);
    ent[i] = v;
  }
  __syncthreads();
  const int cnt = (N3 - e0 < SC_EB ? N3 - e0 : SC_EB) * nm;
  double* out = loc + (size_t)e0 * nm;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const int e = i / nm, nl = i - e * nm;
    const int c = mtab[nl];
    out[i] = g[ent[e * 27 + (c & 31)] + (c >> 5)];
  }
}

cudaError_t periodic_scatter(int n, int P, const double* g, double* loc, cudaStream_t s) {
  const int N3 = n * n * n;
  const int nm = (P + 1) * (P + 1) * (P + 1);
  const int blocks = (N3 + SC_EB - 1) / SC_EB;
  if (blocks == 0) return cudaSuccess;
  periodic_scatter_kernel<<<blocks, 256, sizeof(int) * (SC_EB * 27 + nm), s>>>(n, P, g, loc);
  return cudaGetLastError();
}

// (E, 27) entity bases of the periodic map, built once per map
__global__ void entity_table_kernel(int n, int P, int* ent) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t N3 = (int64_t)n * n * n;
  if (tid >= N3 * 27) return;
  const int e = (int)(tid / 27), k = (int)(tid % 27);
  ent[tid] = entity_base(n, P, e % n, (e / n) % n, e / (n * n), k);
}

cudaError_t periodic_entity_table(int n, int P, int* ent, cudaStream_t s) {
  const int64_t total = (int64_t)n * n * n * 27;
  if (total == 0) return cudaSuccess;
  entity_table_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(n, P, ent);
  return cudaGetLastError();
}

// sharded operator's interface exchange (distributed.py): pack the
// interface entries into a send buffer, and combine the two copies in rank
// order (lo + hi: identical bits on both sides of the interface)
__global__ void index_gather_kernel(int64_t n, const int64_t* __restrict__ idx, const double* __restrict__ src,
                                    double* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}
__global__ void index_sum2_kernel(int64_t n, const int64_t* __restrict__ idx, const double* __restrict__ lo,
                                  const double* __restrict__ hi, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[idx[i]] = lo[i] + hi[i];
}
static unsigned grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (unsigned)(b < 1 ? 1 : (b > 65535 ? 65535 : b));
}
cudaError_t index_gather(int64_t n, const int64_t* idx, const double* src, double* dst, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  index_gather_kernel<<<grid_for(n), 256, 0, s>>>(n, idx, src, dst);
  return cudaGetLastError();
}
cudaError_t index_sum2(int64_t n, const int64_t* idx, const double* lo, const double* hi, double* y,
                       cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  index_sum2_kernel<<<grid_for(n), 256, 0, s>>>(n, idx, lo, hi, y);
  return cudaGetLastError();
}

}  // namespace sphp
