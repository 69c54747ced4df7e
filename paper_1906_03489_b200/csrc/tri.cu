// Triangle (collapsed-coordinate) sum-factorisation kernels (SURVEY §8(f)
// row 3): BwdTrans, IProductWRTBase and PhysDeriv of collections.py:141-148,
// :161-167, :175-177 on Modified_A (direction 1, GLL) x Modified_B
// (direction 2, Gauss-Radau) expansions (basis.py:117-157).
//
//   BwdTrans   tmp[p, j] = sum_{n in block p} c[n] B2[n, j]
//                          (+ c[1] B2[1, j] for p = 1: the collapsed vertex)
//              u[i, j]   = sum_p A1[p, i] tmp[p, j]
//   IProduct   tmp[p, j] = sum_i A1[p, i] W[i, j] u[i, j]
//              b[n]      = sum_j tmp[p(n), j] B2[n, j] (+ tmp[1, j] B2[1, j] for n = 1)
//   PhysDeriv  d1 = D1 along i, d2 = D2 along j; d1' = f d1, d2' = g d1 + d2
//              (collapse factors f = 2/(1-eta2), g = (1+eta1)/(1-eta2),
//              stdregions.py:210-235), then the world transform with inv.
//
// Persistent CTAs hold the tables in shared memory and walk elements; the
// sizes are runtime values (the reference's triangle orders are small and
// any P is accepted), so these are generic loops, not the unrolled
// constant-table contractions of the quad/hex kernels.
#include <cuda_runtime.h>
#include <stdint.h>

#include "tri.h"

namespace sphp {

namespace {

constexpr int kThreads = 128;

__global__ void __launch_bounds__(kThreads) tri_kernel(const TriJob j) {
  extern __shared__ __align__(16) double sm[];
  const int m1 = j.m1, nm = j.nm, Q1 = j.Q1, Q2 = j.Q2, np = Q1 * Q2;
  const int ntab = j.ntab;
  double* tab = sm;                 // A1 | B2 | D1 | D2 | f | g | w
  double* u = tab + ntab;           // np (or nm) input
  double* tmp = u + np;             // max(m1 * Q2, np)
  double* tmp2 = tmp + (m1 * Q2 > np ? m1 * Q2 : np);
  int* pidx = reinterpret_cast<int*>(tmp2 + np);  // nm
  int* bstart = pidx + nm;                        // m1 + 1
  for (int i = threadIdx.x; i < ntab; i += kThreads) tab[i] = j.tab[i];
  for (int i = threadIdx.x; i < nm; i += kThreads) pidx[i] = j.itab[i];
  for (int i = threadIdx.x; i <= m1; i += kThreads) bstart[i] = j.itab[nm + i];
  const double* A1 = tab;
  const double* B2 = A1 + m1 * Q1;
  const double* D1 = B2 + nm * Q2;
  const double* D2 = D1 + Q1 * Q1;
  const double* f = D2 + Q2 * Q2;
  const double* g = f + Q2;
  const double* w = g + np;
  const int64_t cs = j.cs;
  for (int64_t e = blockIdx.x; e < j.E; e += gridDim.x) {
    __syncthreads();  // tables ready / previous element done
    const double* ge = j.geom ? j.geom + e * j.gstride : nullptr;
    if (j.op == SPHP_OP_BWD_TRANS) {
      const double* c = j.in + e * nm;
      for (int i = threadIdx.x; i < nm; i += kThreads) u[i] = c[i];
      __syncthreads();
      for (int k = threadIdx.x; k < m1 * Q2; k += kThreads) {
        const int p = k / Q2, jj = k - p * Q2;
        double acc = 0.0;
        for (int n = bstart[p]; n < bstart[p + 1]; ++n) acc = fma(u[n], B2[n * Q2 + jj], acc);
        if (p == 1) acc = fma(u[1], B2[1 * Q2 + jj], acc);
        tmp[k] = acc;
      }
      __syncthreads();
      double* out = j.out + e * np;
      for (int k = threadIdx.x; k < np; k += kThreads) {
        const int i = k / Q2, jj = k - i * Q2;
        double acc = 0.0;
        for (int p = 0; p < m1; ++p) acc = fma(A1[p * Q1 + i], tmp[p * Q2 + jj], acc);
        out[k] = acc;
      }
    } else if (j.op == SPHP_OP_IPRODUCT_WRT_BASE) {
      const double* in = j.in + e * np;
      for (int k = threadIdx.x; k < np; k += kThreads) {
        double wk;
        if (j.geom_kind == SPHP_GEOM_POINT)
          wk = ge[k];
        else if (j.geom_kind == SPHP_GEOM_AFFINE)
          wk = w[k] * ge[0];
        else
          wk = w[k];
        u[k] = wk * in[k];
      }
      __syncthreads();
      for (int k = threadIdx.x; k < m1 * Q2; k += kThreads) {
        const int p = k / Q2, jj = k - p * Q2;
        double acc = 0.0;
        for (int i = 0; i < Q1; ++i) acc = fma(A1[p * Q1 + i], u[i * Q2 + jj], acc);
        tmp[k] = acc;
      }
      __syncthreads();
      double* out = j.out + e * nm;
      for (int n = threadIdx.x; n < nm; n += kThreads) {
        const int p = pidx[n];
        double acc = 0.0;
        for (int jj = 0; jj < Q2; ++jj) acc = fma(tmp[p * Q2 + jj], B2[n * Q2 + jj], acc);
        if (n == 1)
          for (int jj = 0; jj < Q2; ++jj) acc = fma(tmp[1 * Q2 + jj], B2[1 * Q2 + jj], acc);
        out[n] = acc;
      }
    } else {  // PhysDeriv
      const double* in = j.in + e * np;
      for (int k = threadIdx.x; k < np; k += kThreads) u[k] = in[k];
      __syncthreads();
      double* out = j.out + e * 2 * np;
      for (int k = threadIdx.x; k < np; k += kThreads) {
        const int i = k / Q2, jj = k - i * Q2;
        double d1 = 0.0, d2 = 0.0;
        for (int l = 0; l < Q1; ++l) d1 = fma(D1[i * Q1 + l], u[l * Q2 + jj], d1);
        for (int l = 0; l < Q2; ++l) d2 = fma(D2[jj * Q2 + l], u[i * Q2 + l], d2);
        const double a = f[jj] * d1, b = g[k] * d1 + d2;
        if (j.geom_kind == SPHP_GEOM_NONE) {
          out[k] = a;
          out[np + k] = b;
        } else {
          double i00, i01, i10, i11;  // inv[a][k] = d xi_a / d x_k
          if (j.geom_kind == SPHP_GEOM_POINT) {
            i00 = ge[cs + k];
            i01 = ge[2 * cs + k];
            i10 = ge[3 * cs + k];
            i11 = ge[4 * cs + k];
          } else {
            i00 = ge[1];
            i01 = ge[2];
            i10 = ge[3];
            i11 = ge[4];
          }
          out[k] = i00 * a + i10 * b;       // collections.py:181-185
          out[np + k] = i01 * a + i11 * b;
        }
      }
    }
  }
}

}  // namespace

size_t tri_smem_bytes(const TriJob& j) {
  const int np = j.Q1 * j.Q2;
  const int t = j.m1 * j.Q2 > np ? j.m1 * j.Q2 : np;
  return sizeof(double) * (j.ntab + np + t + np) + sizeof(int) * (j.nm + j.m1 + 1);
}

cudaError_t tri_apply(const TriJob& j, int num_sms, cudaStream_t s) {
  if (j.E == 0) return cudaSuccess;
  const size_t smem = tri_smem_bytes(j);
  if (smem > 200 * 1024) return cudaErrorNotSupported;
  static int configured = 0;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    configured = 1;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tri_kernel, kThreads, smem);
  const int64_t g = (int64_t)num_sms * (occ > 0 ? occ : 1);
  const unsigned grid = (unsigned)(j.E < g ? j.E : g);
  tri_kernel<<<grid, kThreads, smem, s>>>(j);
  return cudaGetLastError();
}

}  // namespace sphp
