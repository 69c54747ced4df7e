// Shared device-side machinery for the spechp B200 kernels:
//   * the constant-memory table pool for the fast (GLL, Modified_A) keys,
//   * TMA bulk-copy (cp.async.bulk) + mbarrier helpers for sm_100a,
//   * the pencil contraction used by every sum-factorisation stage.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sphp {

// ---------------------------------------------------------------------------
// Fast-path key set: Modified_A modes M per direction with GLL Q = M+1
// (the reference default, stdregions.py:376-381) or Q = M+2 (the BASELINE
// configs).  Each key's tables live in __constant__ memory so the unrolled
// contractions take their coefficients as DFMA constant operands.
// ---------------------------------------------------------------------------
constexpr int FAST_M_MIN = 2;
constexpr int FAST_M_MAX = 10;

// even-odd (parity) sizes: H = ceil(Q/2) point pairs incl. the middle,
// HF = floor(Q/2); ME / MO = modes in the even set {s = c0+c1, bubbles 2,4,..}
// and the odd set {d = c1-c0, bubbles 3,5,..}
__host__ __device__ constexpr int eo_h(int Q) { return (Q + 1) / 2; }
__host__ __device__ constexpr int eo_hf(int Q) { return Q / 2; }
__host__ __device__ constexpr int eo_me(int M) { return 1 + (M - 1) / 2; }
__host__ __device__ constexpr int eo_mo(int M) { return M - eo_me(M); }
__host__ __device__ constexpr int eo_size(int M, int Q) {
  return 2 * (eo_me(M) + eo_mo(M)) * eo_h(Q) + 2 * eo_h(Q) * eo_hf(Q) + 2 * eo_h(Q) * eo_h(Q);
}
__host__ __device__ constexpr int tab_size(int M, int Q) { return 2 * M * Q + Q * Q + Q + eo_size(M, Q); }
__host__ __device__ constexpr bool fast_key(int M, int Q) {
  return M >= FAST_M_MIN && M <= FAST_M_MAX && (Q == M + 1 || Q == M + 2);
}
__host__ __device__ constexpr int tab_off(int M, int Q) {
  int off = 0;
  for (int m = FAST_M_MIN; m <= FAST_M_MAX; ++m)
    for (int q = m + 1; q <= m + 2; ++q) {
      if (m == M && q == Q) return off;
      off += tab_size(m, q);
    }
  return -1;
}
constexpr int TAB_TOTAL = tab_off(FAST_M_MAX, FAST_M_MAX + 2) + tab_size(FAST_M_MAX, FAST_M_MAX + 2);

// layout inside one key: B[M][Q], Bd[M][Q], D[Q][Q], w[Q], then the
// even-odd tables BE[ME][H], BO[MO][H], BDE[ME][H], BDO[MO][H],
// DE[H][HF], DO[H][H], DTE[H][HF], DTO[H][H]  (see eo.cuh)
template <int M, int Q>
struct Tab {
  static constexpr int B = tab_off(M, Q);
  static constexpr int BD = B + M * Q;
  static constexpr int D = BD + M * Q;
  static constexpr int W = D + Q * Q;
  static constexpr int H = eo_h(Q), HF = eo_hf(Q), ME = eo_me(M), MO = eo_mo(M);
  static constexpr int BE = W + Q;
  static constexpr int BO = BE + ME * H;
  static constexpr int BDE = BO + MO * H;
  static constexpr int BDO = BDE + ME * H;
  static constexpr int DE = BDO + MO * H;
  static constexpr int DO = DE + H * HF;
  static constexpr int DTE = DO + H * H;
  static constexpr int DTO = DTE + H * HF;
};

// host: the full pool (computed once, uploaded to every TU's bank)
const double* fast_table_pool();

// ---------------------------------------------------------------------------
// PTX helpers (sm_90+ bulk async copies; SASS UBLKCP / SYNCS)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0,
// both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// bulk prefetch of a global range into L2 (no shared memory, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// shared -> global bulk copy (bulk_group completion)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// per-thread 8-byte async gathers into shared memory (SASS LDGSTS)
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ int ld_volatile_s32(const int* p) {
  int v;
  asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)));
  return v;
}
// 16-byte async copy, L2 only (SASS LDGSTS.E.BYPASS.128)
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// Storage slot of quadrature point pt = (i*Q + j)*Q + k inside one METRIC
// component of a hex element record.  Q = 8 stores the points j-major,
// (j*Q + i)*Q + k: the Q = 8 Helmholtz reads the metric on j-pencils with
// lanes (i, k), which in point order would put 16 lanes on 8 bank pairs
// (ncu P=6: 59 M of 133 M excess wavefronts); j-major puts lanes i and i+1
// 8 banks apart.  Every producer (geometry kernels) and consumer (the
// Helmholtz kernels, the Jacobi diagonal) goes through this function.
// ---------------------------------------------------------------------------
#ifndef SPHP_KMAJOR_QMASK
#define SPHP_KMAJOR_QMASK (1 << 9)  // bit Q: hex METRIC components of Q stored k-major
#endif
// k-major METRIC points, (k*Q + i)*Q + j: the K-row Helmholtz reads its
// (i, j) rows one k at a time with lanes on consecutive (i, j), i.e. one
// coalesced 32-point run per k, which lets its local operator read the
// geometry straight from global memory (pipeline MODE 7) instead of staging
// 7 Q^3 doubles per element in shared memory.  Measured (cfg4, local):
// Q = 9 (P = 7) 2.409 -> 2.298 ms; Q = 5, 7 unchanged; Q = 6, 10 lose their
// 128-bit row reads (P = 4 0.613 -> 0.635, P = 8 3.26 -> 3.57 ms with the
// global reads, 3.30 staged); the class operator with global geometry
// (MODE 6) loses 7-20 % at every Q >= 5 (profiles/r02_kmajor.log)
// Orders whose fused hex Helmholtz runs the i-column plan (HexHelmCol,
// hex_ops.cuh): bit Q.  That plan reads the metric in natural point order.
// Measured (cfg4 64^3, local / class-assembled ms; profiles/r02_col*.log):
// Q = 4 (P = 2) 0.198 -> 0.158 / 0.217 -> 0.181 (against the skewed Q = 4 plan
// and its global-geometry class launch), Q = 5 (P = 3) 0.399 -> 0.312 /
// 0.467 -> 0.370, Q = 6 (P = 4) 0.612 -> 0.567 / 0.691 -> 0.665, Q = 7 (P = 5)
// 1.088 -> 1.022 / 1.294 -> 1.187.  One element per tile at Q >= 8 leaves the
// column stage too few threads: the row / pencil plans stay (P = 6..8: 1.54
// vs 1.50, 2.79 vs 2.25, 3.56 vs 3.27 ms).
#ifndef SPHP_COL_QMASK
#define SPHP_COL_QMASK ((1 << 4) | (1 << 5) | (1 << 6) | (1 << 7))
#endif
__host__ __device__ constexpr bool col_plan(int Q) { return Q < 32 && ((SPHP_COL_QMASK >> Q) & 1); }
__host__ __device__ constexpr bool metric_kmajor(int Q) {
  return Q < 32 && ((SPHP_KMAJOR_QMASK >> Q) & 1) && !col_plan(Q);
}
__host__ __device__ __forceinline__ int metric_slot(int dim, int Q, int pt) {
  if (dim != 3 || col_plan(Q)) return pt;
  if (metric_kmajor(Q)) {
    const int ij = pt / Q, k = pt - ij * Q;
    return k * Q * Q + ij;
  }
  if (Q != 8) return pt;
  const int i = pt >> 6, j = (pt >> 3) & 7, k = pt & 7;
  return (j << 6) | (i << 3) | k;
}

// ---------------------------------------------------------------------------
// Pencil contraction: out[o*OS] (+)= sum_l T(o,l) in[l*IS], T(o,l) read from
// constant memory at TOFF + o*TSO + l*TSI.  Summation order l = 0..NIN-1
// (fixed, so repeated applies are bitwise identical).
// ---------------------------------------------------------------------------
template <int NIN, int NOUT, int TOFF, int TSO, int TSI, int IS, int OS, bool ACC>
__device__ __forceinline__ void pencil(const double* tab, const double* __restrict__ in,
                                       double* __restrict__ out) {
  double x[NIN];
#pragma unroll
  for (int l = 0; l < NIN; ++l) x[l] = in[l * IS];
#pragma unroll
  for (int o = 0; o < NOUT; ++o) {
    double acc = ACC ? out[o * OS] : 0.0;
#pragma unroll
    for (int l = 0; l < NIN; ++l) acc = fma(tab[TOFF + o * TSO + l * TSI], x[l], acc);
    out[o * OS] = acc;
  }
}

__host__ __device__ constexpr int odd_up(int x) { return x | 1; }

}  // namespace sphp

// every kernel TU declares its own constant bank with this macro and
// registers an uploader that the host calls once per device
#define SPHP_DECLARE_TABLE_BANK(NAME)                                              \
  static __constant__ double c_tab[sphp::TAB_TOTAL];                               \
  namespace sphp {                                                                 \
  cudaError_t upload_tables_##NAME() {                                             \
    return cudaMemcpyToSymbol(c_tab, fast_table_pool(), sizeof(double) * TAB_TOTAL); \
  }                                                                                \
  }
