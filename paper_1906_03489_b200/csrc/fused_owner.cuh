// Assembled Helmholtz with the owner-computes sum fused into the operator
// launch (assembly algorithm FUSED: GlobalSystem.apply, assembly.py:177-182,
// on the periodic structured hex map; the same sums as owner_periodic_v3).
//
// Warp-specialised persistent kernel, NT + 32 threads per CTA:
//   * warps 0 .. NT/32-1 run the fused Helmholtz tiles exactly as the local
//     pipeline does (local block in by TMA, Op::compute, local block out),
//     tiles claimed in order from an atomic counter; after a tile's
//     write-back a per-tile done flag is released;
//   * the last warp is the owner warp: it claims owner segments (L
//     consecutive elements of one x-row, queue sorted by the last tile each
//     depends on), waits for those tiles' flags and sums every global dof
//     the segment's elements own (low vertex, the 3 edges and 3 faces
//     leaving it, the interior) from the local outputs of the <= 8 elements
//     touching it, in the fixed lexicographic (a, b, c) offset order of
//     owner_periodic_v3 — bitwise the split algorithm's y.
// The owner warp never joins the compute barriers (named barrier 1 over NT
// threads, cta_bar), so its L2 reads overlap the tiles' HBM streaming; the
// local outputs it reads were written moments earlier and come from L2.
// Tiles never wait and every tile an owner segment waits for was claimed by
// a running CTA, so there is no co-residency assumption.
#pragma once
#include "pipeline.cuh"

namespace sphp {

#ifndef SPHP_OWNER_LOADS
#define SPHP_OWNER_LOADS 16
#endif

struct FusedArgs {
  const int* queue;  // owner segment ids in dependency order
  int nqueue;
  int* sync;         // [0] tile counter, [1] owner counter, [2 + t] tile t done (zeroed per launch)
  double* y;
  int n, L, accumulate;
  int debug;  // tuning: bit 0 skips the owner sums
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// j-th subset of the 3-bit mask z in increasing order (bit deposit)
__host__ __device__ constexpr int subset_bits(int z, int j) {
  int o = 0, k = 0;
  for (int d = 0; d < 3; ++d)
    if ((z >> d) & 1) o |= ((j >> k++) & 1) << d;
  return o;
}

// Owner sums of one owned class C for a segment: K = 2^|Z| terms per dof
// (Z = axes where the owned mode index is 0: p -> bit 2, q -> 1, r -> 0),
// U = SPHP_OWNER_LOADS / K dofs per lane per batch (that many loads in
// flight per lane: the warp is latency bound on L2).
// Classes in owner_periodic_v3 order: vertex, x/y/z edges, x/y/z-normal
// faces, interior; dof r0 = el * SIZE + off of the class maps to y[base + r0].
template <int M, int C>
__device__ __forceinline__ void owner_class(const double* __restrict__ loc, double* __restrict__ y, int L,
                                            int n, int ex0, int segout, int rowb, int accumulate, int lane) {
  constexpr int b = M > 2 ? M - 2 : 1, nm = M * M * M;  // M >= 3 (P >= 2) at launch
  constexpr int Z = C == 0 ? 7 : C == 1 ? 3 : C == 2 ? 5 : C == 3 ? 6 : C == 4 ? 4 : C == 5 ? 2 : C == 6 ? 1 : 0;
  constexpr int K = Z == 7 ? 8 : (Z == 3 || Z == 5 || Z == 6) ? 4 : Z ? 2 : 1;
  constexpr int U = SPHP_OWNER_LOADS / K;
  constexpr int SIZE = C == 0 ? 1 : C < 4 ? b : C < 7 ? b * b : b * b * b;
  const int total = L * SIZE;
  const int base_out = __shfl_sync(0xffffffffu, segout, C);
  int rb[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) rb[q] = __shfl_sync(0xffffffffu, rowb, q);
  for (int t0 = lane; t0 < total; t0 += 32 * U) {
    double v[U][K];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r0 = t0 + 32 * u;
      const int el = r0 / SIZE, off = r0 - el * SIZE;
      int m0;
      if constexpr (C == 0) m0 = 0;
      else if constexpr (C == 1) m0 = (off + 2) * M * M;
      else if constexpr (C == 2) m0 = (off + 2) * M;
      else if constexpr (C == 3) m0 = off + 2;
      else if constexpr (C == 4) m0 = (off / b + 2) * M + off % b + 2;
      else if constexpr (C == 5) m0 = (off / b + 2) * M * M + off % b + 2;
      else if constexpr (C == 6) m0 = (off / b + 2) * M * M + (off % b + 2) * M;
      else m0 = ((off / (b * b) + 2) * M + (off / b) % b + 2) * M + off % b + 2;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const int o8 = subset_bits(Z, j);
        const int aa = o8 >> 2, bb = (o8 >> 1) & 1, cc = o8 & 1;
        int x = ex0 + el - aa;
        x += x < 0 ? n : 0;
        const int64_t e = (int64_t)rb[(bb << 1) | cc] + x;
        v[u][j] = r0 < total ? __ldcg(loc + e * nm + m0 + aa * M * M + bb * M + cc) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r0 = t0 + 32 * u;
      if (r0 >= total) continue;
      double acc = v[u][0];
#pragma unroll
      for (int j = 1; j < K; ++j) acc += v[u][j];
      double* dst = y + base_out + r0;
      *dst = accumulate ? *dst + acc : acc;
    }
  }
}

template <class Op>
constexpr int fused_min_blocks() {
  constexpr size_t sm = Scaffold<Op, 0>::SMEM_BYTES + 2048;
  constexpr int nb = (int)((228 * 1024) / sm);
  return nb < 1 ? 1 : (nb > 4 ? 4 : nb);
}

template <class Op>
__global__ void __launch_bounds__(Op::NT + 32, fused_min_blocks<Op>())
    fused_owner_kernel(const DevArgs a, const FusedArgs f) {
  using S = Scaffold<Op, 0>;
  constexpr int NE = Op::NE, NT = Op::NT, IN = Op::IN, OUT = Op::OUT, GEO = Op::GEO, M = Op::M;
  constexpr int GEO_S = S::GEO_S;
  static_assert(S::NST == 1, "the fused owner kernel runs one input stage");
  static_assert(IN == M * M * M && OUT == IN, "hex Helmholtz tiles only");
  extern __shared__ __align__(128) double smem[];
  double* in_s = smem;
  double* geo_s = in_s + S::IN_T;
  double* work = smem + S::STAGE + S::OUT_T;
  double* out_s = S::OUT_OFF >= 0 ? work + (S::OUT_OFF >= 0 ? S::OUT_OFF : 0) : smem + S::STAGE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(work + S::WORK_T);
  __shared__ int s_tile[2];
  const int tid = threadIdx.x;
  const int64_t count = a.E;
  const int ntiles = (int)((count + NE - 1) / NE);
  int* const tctr = f.sync;
  int* const octr = f.sync + 1;
  int* const done = f.sync + 2;

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    fence_mbar_init();
  }
  __syncthreads();

  if (tid >= NT) {
    // ======================= owner warp ===================================
    const int lane = tid - NT, n = f.n, L = f.L, segs = n / L;
    if (f.debug & 1) return;
    for (;;) {
      int id = 0;
      if (lane == 0) id = atomicAdd(octr, 1);
      id = __shfl_sync(0xffffffffu, id, 0);
      if (id >= f.nqueue) break;
      const int sg = __ldg(f.queue + id);
      const int seg = sg % segs, row = sg / segs;
      const int ey = row % n, ez = row / n, ex0 = seg * L;
      const int segout = lane < 8 ? class_gid(class_geom(owned_class(lane), n, M - 1), n, ex0, ey, ez) : 0;
      int sy = ey - ((lane >> 1) & 1), sz = ez - (lane & 1);
      sy += sy < 0 ? n : 0;
      sz += sz < 0 ? n : 0;
      const int rowb = n * (sy + n * sz);  // element id of x = 0 in neighbour row (lane & 3)
      // wait for the tiles holding elements ex0 - 1 .. ex0 + L - 1 of the
      // four rows (element n - 1 when ex0 == 0: periodic wrap)
      const int span = (L + NE - 1) / NE + 1;
      for (int i = lane; i < 4 * (span + 1); i += 32) {
        const int q = i / (span + 1), j = i - q * (span + 1);
        int qy = ey - ((q >> 1) & 1), qz = ez - (q & 1);
        qy += qy < 0 ? n : 0;
        qz += qz < 0 ? n : 0;
        const int rbase = n * (qy + n * qz);
        int tile;
        if (j == span) {
          tile = (rbase + (ex0 == 0 ? n - 1 : ex0 - 1)) / NE;
        } else {
          const int lo = (rbase + ex0) / NE, hi = (rbase + ex0 + L - 1) / NE;
          tile = lo + j;
          if (tile > hi) continue;
        }
        if (!(f.debug & 4))
          while (ld_acquire(done + tile) == 0) __nanosleep(128);
      }
      __syncwarp();
      if (f.debug & 2) continue;
      const double* loc = a.out;
      owner_class<M, 0>(loc, f.y, L, n, ex0, segout, rowb, f.accumulate, lane);
      owner_class<M, 1>(loc, f.y, L, n, ex0, segout, rowb, f.accumulate, lane);
      owner_class<M, 2>(loc, f.y, L, n, ex0, segout, rowb, f.accumulate, lane);
      owner_class<M, 3>(loc, f.y, L, n, ex0, segout, rowb, f.accumulate, lane);
      owner_class<M, 4>(loc, f.y, L, n, ex0, segout, rowb, f.accumulate, lane);
      owner_class<M, 5>(loc, f.y, L, n, ex0, segout, rowb, f.accumulate, lane);
      owner_class<M, 6>(loc, f.y, L, n, ex0, segout, rowb, f.accumulate, lane);
      owner_class<M, 7>(loc, f.y, L, n, ex0, segout, rowb, f.accumulate, lane);
    }
    return;
  }

  // ======================= compute warps ==================================
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
  // thread 0: TMA bulk copies of tile t's local block and geometry
  auto issue_tile = [&](int t) {
    if (t >= ntiles) return;
    const int64_t w0 = (int64_t)t * NE;
    const int r = (int)((count - w0) < NE ? (count - w0) : NE);
    int64_t a0, a1;
    int off;
    if (!in_window(t, a0, a1, off)) return;  // synchronous at consumption
    const uint32_t bytes_in = (uint32_t)(a1 - a0);
    const uint32_t bytes_g = (uint32_t)(sizeof(double) * r * GEO);
    mbar_expect_tx(&bar[0], bytes_in + bytes_g);
    bulk_g2s(in_s, reinterpret_cast<const char*>(a.in) + a0, bytes_in, &bar[0]);
    if (a.gstride == GEO && a.goff == 0 && GEO_S == GEO) {
      bulk_g2s(geo_s, a.geom + w0 * a.gstride, bytes_g, &bar[0]);
    } else {
      for (int e = 0; e < r; ++e)
        bulk_g2s(geo_s + e * GEO_S, a.geom + (w0 + e) * a.gstride + a.goff, (uint32_t)(sizeof(double) * GEO),
                 &bar[0]);
    }
  };
  // thread 0 keeps the id of the tile after next in flight (its atomic is
  // issued one tile ahead, so its latency never sits before a barrier)
  // The done flag of a tile is released by thread 0 one tile later, at the
  // next tile's release point: a release store waits for the CTA's earlier
  // global stores to complete, which right after the write-back costs a
  // microsecond per tile (measured 0.2 ms per apply at P = 4), mid-way
  // through the next tile's compute it is free.
  int ahead = 0, pending = -1;
  if (tid == 0) {
    const int t0 = atomicAdd(tctr, 1);
    ahead = atomicAdd(tctr, 1);
    s_tile[0] = t0;
    issue_tile(t0);
  }
  cta_bar<NT>();

  uint32_t phase = 0;
  for (int it = 0;; ++it) {
    const int t = s_tile[it & 1];
    if (t >= ntiles) break;
    const int64_t w0 = (int64_t)t * NE;
    const int r = (int)((count - w0) < NE ? (count - w0) : NE);
    const double* in_p = in_s;
    int64_t a0, a1;
    int off;
    if (in_window(t, a0, a1, off)) {
      mbar_wait(&bar[0], phase);
      phase ^= 1u;
      in_p = in_s + off;
    } else {
      for (int i = tid; i < r * IN; i += NT) in_s[i] = a.in[w0 * IN + i];
      for (int i = tid; i < r * GEO; i += NT) {
        const int e = i / GEO, c = i - e * GEO;
        geo_s[e * GEO_S + c] = a.geom[(w0 + e) * a.gstride + a.goff + c];
      }
    }
    for (int i = r * IN + tid; i < NE * IN; i += NT) in_s[(in_p - in_s) + i] = 0.0;
    for (int i = r * GEO_S + tid; i < NE * GEO_S; i += NT) geo_s[i] = 0.0;
    cta_bar<NT>();
    auto release = [&]() {
      if (tid == 0) {
        if (pending >= 0) st_release(done + pending, 1);
        pending = -1;
        const int nxt = ahead;
        ahead = atomicAdd(tctr, 1);
        s_tile[(it + 1) & 1] = nxt;
        fence_proxy_async();
        issue_tile(nxt);
      }
    };
    auto pre_out = [&]() {};
    Op::compute(in_p, geo_s, work, out_s, a.lam, release, pre_out, c_tab);
    cta_bar<NT>();
    for (int i = tid; i < r * OUT; i += NT) a.out[w0 * OUT + i] = out_s[i];
    pending = t;  // thread 0 releases it after the next barrier-separated stage
  }
  // the last tile: its stores happen-before thread 0's release
  cta_bar<NT>();
  if (tid == 0 && pending >= 0) st_release(done + pending, 1);
}

template <class Op>
cudaError_t launch_fused(const OpArgs& oa, int64_t gstride, cudaStream_t s) {
  using Sc = Scaffold<Op, 0>;
  auto kern = fused_owner_kernel<Op>;
  constexpr int NTHR = Op::NT + 32;
  static LaunchCache cache[16];
  int dev = 0;
  cudaGetDevice(&dev);
  LaunchCache& c = cache[dev & 15];
  if (c.dev != dev) {
    cudaError_t err =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sc::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int occ = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NTHR, Sc::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    c.occ = occ;
    c.smem = Sc::SMEM_BYTES;
    c.dev = dev;
  }
  if (oa.E <= 0) return cudaSuccess;
  const int n = oa.n;
  const int L = fused_segment_length(n);
  if (L == 0 || oa.sync == nullptr || (int64_t)n * n * n != oa.E) return cudaErrorNotSupported;
  const int64_t ntiles = (oa.E + Op::NE - 1) / Op::NE;
  int64_t grid = (int64_t)oa.num_sms * c.occ;
  static const int64_t max_grid = [] {
    const char* e = getenv("SPHP_MAX_GRID");
    return e ? (int64_t)atoll(e) : (int64_t)0;
  }();
  if (max_grid > 0 && grid > max_grid) grid = max_grid;
  if (grid > ntiles) grid = ntiles;
  FusedArgs f;
  f.queue = fused_queue(n, Op::NE, L, &f.nqueue);
  if (!f.queue) return cudaErrorMemoryAllocation;
  f.sync = oa.sync;
  f.y = oa.yg;
  f.n = n;
  f.L = L;
  f.accumulate = oa.accumulate;
  static const int dbg = [] {
    const char* e = getenv("SPHP_FUSED_DEBUG");
    return e ? atoi(e) : 0;
  }();
  f.debug = dbg;
  cudaError_t err = cudaMemsetAsync(oa.sync, 0, sizeof(int) * (size_t)(ntiles + 2), s);
  if (err != cudaSuccess) return err;
  DevArgs a{};
  a.E = oa.E;
  a.in = oa.in;
  a.out = oa.out;
  a.geom = oa.geom;
  a.gstride = gstride;
  a.goff = 0;
  a.lam = oa.lam;
  a.use_tma = ((reinterpret_cast<uintptr_t>(oa.in) & 15) == 0) &&
              (oa.geom == nullptr || (reinterpret_cast<uintptr_t>(oa.geom) & 15) == 0);
  kern<<<(unsigned)grid, NTHR, Sc::SMEM_BYTES, s>>>(a, f);
  return cudaGetLastError();
}

}  // namespace sphp
