// Periodic-grid scatter (global -> local block) and owner-computes sum
// (local block -> global) by entity class, for the split / owner assembly
// algorithms on the periodic structured hex map (periodic.cuh).
//
// A CTA handles L consecutive elements of one x-row at a time (persistent
// over such segments).  Consecutive elements own consecutive entities, so
// each of the 27 entity classes (8 vertices, 12 edges, 6 faces, the
// interior) maps to one contiguous range of the global vector, and both
// kernels move data class by class through a shared-memory block.  All the
// per-slot index arithmetic depends only on (P, L): it is precomputed once
// per CTA into one packed 32-bit word per slot, so the streaming loops cost
// a table load, a few bit operations, a global load and a shared store per
// value (the first versions were issue-bound on index math).  Each thread
// holds U register slots (U * 256 >= L * nm): the loads of segment i+1 are
// issued before segment i's block is written out / summed, so global reads
// stay in flight across the phases.
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "misc.h"
#include "periodic.cuh"

namespace sphp {

namespace {

constexpr int kThreads = 256;

// owned classes of an element: vertex 0, edges 8/12/16, faces 20/22/24, interior 26
__device__ __forceinline__ int owned_class(int c) {
  return c == 0 ? 0 : (c < 4 ? 8 + 4 * (c - 1) : (c < 7 ? 20 + 2 * (c - 4) : 26));
}
__device__ __forceinline__ int owned_size(int c, int b) {
  return c == 0 ? 1 : (c < 4 ? b : (c < 7 ? b * b : b * b * b));
}
// log2 of the number of elements contributing to a dof of owned class c
__device__ __forceinline__ int owned_log(int c) { return c == 0 ? 3 : (c < 4 ? 2 : (c < 7 ? 1 : 0)); }

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// L: largest of 32/16/8/4 dividing n with L * nm < 2^13 (packed slot
// indices) and block + tables within 48 KB (4+ CTAs per SM).  The owner sum
// prefers segments of at most ~3000 slots (fewer registers per thread, more
// resident CTAs); re-measured after the padded staging (tools/time_periodic.py,
// SPHP_PERIODIC_L): P=4 121 us at L=8 vs 116 us at L=16, P=6 314 us at L=4
// vs 294 us at L=8.
int segment_length(int n, int P, bool owner) {
  const int nm = (P + 1) * (P + 1) * (P + 1);
  static const int force = env_int("SPHP_PERIODIC_L", 0);  // tuning override
  if (force >= 4 && n % force == 0 && force * nm < 8192 && force <= 32) return force;
  auto fits = [&](int L) {
    return n % L == 0 && L * (nm + 2) < 8192 &&
           (size_t)L * nm * 12 + (size_t)L * P * P * P * 4 <= 48 * 1024;
  };
  if (owner)
    for (int L = 32; L >= 4; L /= 2)
      if (fits(L) && L * nm <= 3000) return L;
  for (int L = 32; L >= 4; L /= 2)
    if (fits(L)) return L;
  return 0;
}

template <typename K>
unsigned persistent_grid(K kernel, size_t smem, int64_t work) {
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem);
  static const int cap = env_int("SPHP_PERIODIC_CTAS", 0);  // tuning: CTAs per SM
  if (cap > 0 && cap < occ) occ = cap;
  const int64_t g = (int64_t)sms * (occ > 0 ? occ : 1);
  return (unsigned)(work < g ? work : g);
}

// segment schedule: the caller's counter (one int, owned by the stream's
// workspace) is zeroed on the launch stream and handed out by atomics, or
// the static round-robin schedule when it is null / SPHP_PERIODIC_DYNAMIC=0
int* schedule_counter(int* ctr, cudaStream_t s) {
  static const int dynamic = env_int("SPHP_PERIODIC_DYNAMIC", 1);
  if (!dynamic || !ctr) return nullptr;
  if (cudaMemsetAsync(ctr, 0, sizeof(int), s) != cudaSuccess) return nullptr;
  return ctr;
}

template <typename K>
void allow_smem(K kernel, int& configured) {
  if (!configured) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    configured = 1;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// scatter: loc[e][mode] = x[entity_base(e, class(mode)) + offset(mode)].
// Slots ordered (class, element, offset) -> coalesced reads per class range.
// Word: class (5 bits) | rel (13) << 5 | dest (13) << 18 | wrap << 31 with
// rel = el * size + offset relative to the segment's class range and dest =
// el * nm + mode in the element-major block.  (A TMA variant — one bulk copy
// per class range, permute in shared memory, one bulk store — measured
// 119 us against 90 us for this one at P = 4, n = 64: 27 small copies per
// segment keep too little in flight.)
// ---------------------------------------------------------------------------
template <int U>
__global__ void __launch_bounds__(kThreads, U <= 8 ? 4 : 3) periodic_scatter_v2_kernel(int n, int P, int L,
                                                                          const double* __restrict__ x,
                                                                          double* __restrict__ loc,
                                                                          int* __restrict__ ctr, int sg0,
                                                                          int sg1) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int cb[28];
  __shared__ int2 cseg[2][27];  // per class: (base, wrap correction)
  const int m = P + 1, nm = m * m * m, b = P - 1, total = L * nm;
  // element stride of the staged block: nm, or nm + 2 for even nm (an
  // element stride = 0 or 8 mod 16 put the consecutive-element slots of one
  // class on 1-2 bank pairs: 8-16-way conflicts at P = 3, 5, 7)
  const int nmp = (nm & 1) ? nm : nm + 2, total_p = L * nmp;
  double* blk = smem;                                                // L * nmp + 2 (scratch)
  uint32_t* word = reinterpret_cast<uint32_t*>(blk + total_p + 2);  // U * kThreads
  int* inv = reinterpret_cast<int*>(word + U * kThreads);          // nm: class slot -> local mode
  const int segs = n / L, nseg = sg1;  // segments [sg0, sg1) (x-rows of L elements)
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int k = 0; k < 27; ++k) {
      cb[k] = acc;
      acc += class_size(k, b);
    }
    cb[27] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nm; i += kThreads) {
    const int c = mode_code(m, i);
    inv[cb[c & 31] + (c >> 5)] = i;
  }
  __syncthreads();
  // padded to U * kThreads slots: the tail slots load x[segbase[0]] into
  // the scratch double after the block, so the streaming loop is branch-free
  for (int t = threadIdx.x; t < U * kThreads; t += kThreads) {
    if (t >= total) {
      word[t] = (uint32_t)total_p << 18;
      continue;
    }
    int k = 0;
    while (L * cb[k + 1] <= t) ++k;
    const int s = class_size(k, b);
    const int r = t - L * cb[k], el = r / s, o = r - el * s;
    const uint32_t dest = el * nmp + inv[cb[k] + o];
    const uint32_t wrap = (class_dx(k) && el == L - 1) ? 1u : 0u;
    word[t] = (uint32_t)k | ((uint32_t)r << 5) | (dest << 18) | (wrap << 31);
  }
  // gid(el, o) = segbase + el * size + o, minus n * size when the high-x
  // entity of the row's last element wraps to x = 0
  auto bases = [&](int sg, int buf) {
    if (threadIdx.x < 27 && sg < nseg) {
      const int seg = sg % segs, row = sg / segs, ex0 = seg * L;
      const int k = threadIdx.x;
      const ClassGeom cg = class_geom(k, n, P);
      cseg[buf][k] = make_int2(class_gid(cg, n, ex0, row % n, row / n),  // ex0 + dx < n
                              (ex0 + L == n) ? n * cg.s : 0);
    }
  };
  double v[U];
  int d[U];
  auto issue = [&](int sg, int buf) {
    if (sg >= nseg) return;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t w = word[u * kThreads + threadIdx.x];
      const int2 sb = cseg[buf][w & 31];
      const int g = sb.x + (int)((w >> 5) & 8191) - ((w >> 31) ? sb.y : 0);
      v[u] = __ldg(x + g);
      d[u] = (w >> 18) & 8191;
    }
  };
  // segment schedule: dynamic (atomic counter, keeps the CTAs' working set
  // of neighbouring rows tight in L2) or static round robin when ctr is null;
  // warp 0 grabs the id and computes the segment's bases
  __shared__ int ids[2];
  // lane 0 of warp 0 keeps one id in flight: the atomic for the segment
  // after next is issued when this one is consumed, so its latency never
  // sits in front of a barrier (ids are increasing per CTA, so every id
  // still in flight when the loop ends is past nseg)
  int ahead = 0;
  if (ctr && threadIdx.x == 0) ahead = atomicAdd(ctr, 1);
  auto grab = [&](int fallback, int buf) {
    if (threadIdx.x < 32) {
      int id = fallback;
      if (ctr) {
        id = __shfl_sync(0xffffffffu, ahead, 0);
        if (threadIdx.x == 0) ahead = atomicAdd(ctr, 1);
      }
      id += sg0;
      if (threadIdx.x == 0) ids[buf] = id;
      bases(id, buf);
    }
  };
  grab(blockIdx.x, 0);
  __syncthreads();  // tables + first bases
  int cur = ids[0];
  issue(cur, 0);
  int buf = 0;
  for (int k = 1; cur < nseg; ++k, buf ^= 1) {
#pragma unroll
    for (int u = 0; u < U; ++u) blk[d[u]] = v[u];
    grab(blockIdx.x + k * gridDim.x, buf ^ 1);
    fence_proxy_async();  // this thread's block writes -> the bulk copy
    __syncthreads();      // block complete, next bases visible
    const int nxt = ids[buf ^ 1];
    issue(nxt, buf ^ 1);  // next segment's loads overlap the write-out
    // one TMA bulk store of the block (L * nm is even and the block start
    // 16-byte aligned, L % 4 == 0); the threads only wait for its reads
    if (nmp == nm) {
      if (threadIdx.x == 0) {
        bulk_s2g(loc + (size_t)cur * total, blk, (uint32_t)(sizeof(double) * total));
        bulk_commit();
        bulk_wait_read0();
      }
    } else if (threadIdx.x < 32) {  // padded: one bulk copy per element
      for (int el = threadIdx.x; el < L; el += 32)
        bulk_s2g(loc + (size_t)cur * total + (size_t)el * nm, blk + el * nmp, (uint32_t)(sizeof(double) * nm));
      bulk_commit();
      bulk_wait_read0();
    }
    __syncthreads();  // block consumed
    cur = nxt;
  }
  if (threadIdx.x < 32) bulk_wait0();
}

// per-thread register batch: U * kThreads >= L * nm
template <typename F>
cudaError_t with_unroll(int slots, F&& f) {
  if (slots <= 4 * kThreads) return f(std::integral_constant<int, 4>());
  if (slots <= 8 * kThreads) return f(std::integral_constant<int, 8>());
  if (slots <= 12 * kThreads) return f(std::integral_constant<int, 12>());
  if (slots <= 16 * kThreads) return f(std::integral_constant<int, 16>());
  return cudaErrorNotSupported;
}

cudaError_t periodic_scatter_v2(int n, int P, const double* x, double* loc, cudaStream_t s, int row0,
                                int row1, int* ctr) {
  const int L = segment_length(n, P, false);
  if (L == 0 || P < 2) return cudaErrorNotSupported;
  if (reinterpret_cast<uintptr_t>(loc) & 15) return cudaErrorNotSupported;
  if (n == 0) return cudaSuccess;
  const int nm = (P + 1) * (P + 1) * (P + 1);
  return with_unroll(L * nm, [&](auto uc) {
    constexpr int U = decltype(uc)::value;
    const int nmp = (nm & 1) ? nm : nm + 2;
    const size_t smem = sizeof(double) * (L * nmp + 2) + sizeof(uint32_t) * U * kThreads + sizeof(int) * nm;
    static int configured = 0;
    allow_smem(periodic_scatter_v2_kernel<U>, configured);
    if (row1 < 0) row1 = n * n;  // rows ey + n ez
    const int segs = n / L;
    if (row1 <= row0) return cudaSuccess;
    const unsigned blocks =
        persistent_grid(periodic_scatter_v2_kernel<U>, smem, (int64_t)(row1 - row0) * segs);
    periodic_scatter_v2_kernel<U><<<blocks, kThreads, smem, s>>>(n, P, L, x, loc, schedule_counter(ctr, s),
                                                                 row0 * segs, row1 * segs);
    return cudaGetLastError();
  });
}

// ---------------------------------------------------------------------------
// Owner-computes sum.  Element e owns its low vertex, the 3 edges and 3 faces
// leaving it and its interior (P^3 dofs).  Neighbour e - (a,b,c) contributes
// to them its modes with index 1 in every direction where the offset is 1
// and index in {0, 2..P} elsewhere: (P+1)^3 values per owner, each used once.
// Phase 1 stages them (slots ordered offset, element, index: block-
// contiguous neighbour reads) into a layout where the terms of every owned
// dof are contiguous and in lexicographic (a, b, c) order; phase 2 sums each
// run and writes every owned class range contiguously.
//   phase-1 word: row (2) | (el - a + 1) * nm + mode (15) << 2 | dest (13) << 17
//                 | x-wrap << 31, row = the (b, c) bits of the offset
//   phase-2 word: class (3) | el * size + off (13) << 3 | start (13) << 16 | log2 count (2) << 29
// ---------------------------------------------------------------------------
template <int U>
__global__ void __launch_bounds__(kThreads, U <= 8 ? 4 : 3) owner_periodic_v3_kernel(int n, int P, int L,
                                                                     const double* __restrict__ loc,
                                                                     double* __restrict__ y,
                                                                     int accumulate,
                                                                     int* __restrict__ ctr, int sg0,
                                                                     int sg1) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int cstart[9], segout[2][8], wrapadd[2];
  __shared__ long long rowoff[2][4];  // per neighbour row: (row element + ex0 - 1) * nm
  const int m = P + 1, nm = m * m * m, b = P - 1, per = P * P * P;
  const int total1 = L * nm, total2 = L * per;
  // staged element stride: nm + 2 for even nm (bank spread, as the scatter)
  const int nmp = (nm & 1) ? nm : nm + 2, total1p = L * nmp;
  double* S = smem;                                              // L * nm + 2 (scratch)
  uint32_t* w1 = reinterpret_cast<uint32_t*>(S + total1p + 2);  // U * kThreads
  uint32_t* w2 = w1 + U * kThreads;                              // L * P^3
  const int segs = n / L, nseg = sg1;  // segments [sg0, sg1) (x-rows of L elements)
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int c = 0; c < 8; ++c) {
      cstart[c] = acc;  // start of the class's term runs in an element's block
      acc += owned_size(c, b) << owned_log(c);
    }
    cstart[8] = acc;  // == nm
  }
  __syncthreads();
  for (int t = threadIdx.x; t < U * kThreads; t += kThreads) {
    if (t >= total1) {  // padding: a valid load into the scratch double
      w1[t] = ((uint32_t)nm << 2) | ((uint32_t)total1p << 17);
      continue;
    }
    // offset o8 = (a, b, c) bits; its index set has P or 1 entries per axis
    int o8 = 0, first = 0, cnt = 0;
    for (;; ++o8) {
      cnt = (o8 & 4 ? 1 : P) * (o8 & 2 ? 1 : P) * (o8 & 1 ? 1 : P);
      if (t < first + L * cnt) break;
      first += L * cnt;
    }
    const int a = o8 >> 2, bb = (o8 >> 1) & 1, c = o8 & 1;
    const int sb = bb ? 1 : P, sc = c ? 1 : P;
    const int r0 = t - first, el = r0 / cnt, idx = r0 - el * cnt;
    const int ia = idx / (sb * sc), ib = (idx / sc) % sb, ic = idx % sc;
    // neighbour mode and the owner dof (p, q, r) it contributes to
    const int np = a ? 1 : (ia ? ia + 1 : 0);
    const int nq = bb ? 1 : (ib ? ib + 1 : 0);
    const int nr = c ? 1 : (ic ? ic + 1 : 0);
    const int p = a ? 0 : np, q = bb ? 0 : nq, r = c ? 0 : nr;
    // owned class / offset of (p, q, r) in mode_code order
    const int zmask = (p == 0 ? 4 : 0) | (q == 0 ? 2 : 0) | (r == 0 ? 1 : 0);
    int cc, off;
    switch (zmask) {
      case 7: cc = 0; off = 0; break;
      case 3: cc = 1; off = p - 2; break;
      case 5: cc = 2; off = q - 2; break;
      case 6: cc = 3; off = r - 2; break;
      case 4: cc = 4; off = (q - 2) * b + (r - 2); break;
      case 2: cc = 5; off = (p - 2) * b + (r - 2); break;
      case 1: cc = 6; off = (p - 2) * b + (q - 2); break;
      default: cc = 7; off = ((p - 2) * b + (q - 2)) * b + (r - 2); break;
    }
    // position of o8 in the dof's run: o8's bits on the zero axes, in
    // order of significance (so runs are in increasing o8 order)
    int pos = 0, nb = 0;
    for (int d = 0; d < 3; ++d)
      if (zmask >> d & 1) pos |= ((o8 >> d) & 1) << nb++;
    const uint32_t dest = el * nmp + cstart[cc] + (off << owned_log(cc)) + pos;
    const uint32_t mode = (np * m + nq) * m + nr;
    const uint32_t elx = el - a + 1, wrap = elx == 0 ? 1u : 0u;
    w1[t] = (uint32_t)(o8 & 3) | ((elx * nm + mode) << 2) | (dest << 17) | (wrap << 31);
  }
  for (int t = threadIdx.x; t < total2; t += kThreads) {
    int cc = 0, first = 0;
    while (t >= first + L * owned_size(cc, b)) first += L * owned_size(cc++, b);
    const int s = owned_size(cc, b), r0 = t - first, el = r0 / s, off = r0 - el * s;
    const uint32_t start = el * nmp + cstart[cc] + (off << owned_log(cc));
    w2[t] = (uint32_t)cc | ((uint32_t)r0 << 3) | (start << 16) | ((uint32_t)owned_log(cc) << 29);
  }
  // per segment: owned-class output bases and the 4 neighbour rows
  auto bases = [&](int sg, int buf) {
    if (threadIdx.x < 8 && sg < nseg) {
      const int seg = sg % segs, row = sg / segs;
      const int ey = row % n, ez = row / n, ex0 = seg * L;
      const int c = threadIdx.x;
      // owned classes sit at the element itself: gid = base + x * size + off
      segout[buf][c] = class_gid(class_geom(owned_class(c), n, P), n, ex0, ey, ez);
      // neighbour row for the (b, c) bits of o8 = c; the -1 pairs with the
      // +1 stored in the phase-1 word
      if (c < 4) {
        int sy = ey - ((c >> 1) & 1), sz = ez - (c & 1);
        sy += sy < 0 ? n : 0;
        sz += sz < 0 ? n : 0;
        rowoff[buf][c] = ((long long)n * (sy + n * sz) + ex0 - 1) * nm;
      }
      // element ex0 - 1 of the row's first segment wraps to x = n - 1
      if (c == 0) wrapadd[buf] = ex0 == 0 ? n * nm : 0;
    }
  };
  double v[U];
  int d[U];
  auto issue = [&](int sg, int buf) {
    if (sg >= nseg) return;
    const int wa = wrapadd[buf];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t w = w1[u * kThreads + threadIdx.x];
      const int rel = (int)((w >> 2) & 32767) + ((w >> 31) ? wa : 0);
      v[u] = __ldg(loc + rowoff[buf][w & 3] + rel);
      d[u] = (w >> 17) & 8191;
    }
  };
  // segment schedule: dynamic (atomic counter, keeps the CTAs' working set
  // of neighbouring rows tight in L2) or static round robin when ctr is null;
  // warp 0 grabs the id and computes the segment's bases
  __shared__ int ids[2];
  // lane 0 of warp 0 keeps one id in flight: the atomic for the segment
  // after next is issued when this one is consumed, so its latency never
  // sits in front of a barrier (ids are increasing per CTA, so every id
  // still in flight when the loop ends is past nseg)
  int ahead = 0;
  if (ctr && threadIdx.x == 0) ahead = atomicAdd(ctr, 1);
  auto grab = [&](int fallback, int buf) {
    if (threadIdx.x < 32) {
      int id = fallback;
      if (ctr) {
        id = __shfl_sync(0xffffffffu, ahead, 0);
        if (threadIdx.x == 0) ahead = atomicAdd(ctr, 1);
      }
      id += sg0;
      if (threadIdx.x == 0) ids[buf] = id;
      bases(id, buf);
    }
  };
  grab(blockIdx.x, 0);
  __syncthreads();  // tables + first bases
  int cur = ids[0];
  issue(cur, 0);
  int buf = 0;
  for (int k = 1; cur < nseg; ++k, buf ^= 1) {
#pragma unroll
    for (int u = 0; u < U; ++u) S[d[u]] = v[u];
    grab(blockIdx.x + k * gridDim.x, buf ^ 1);
    __syncthreads();  // staged block complete, next bases visible
    const int nxt = ids[buf ^ 1];
    issue(nxt, buf ^ 1);  // next segment's loads overlap the sums
    for (int t = threadIdx.x; t < total2; t += kThreads) {
      const uint32_t w = w2[t];
      const double* run = S + ((w >> 16) & 8191);
      const int cnt = 1 << (w >> 29);
      double acc = run[0];
      for (int j = 1; j < cnt; ++j) acc += run[j];
      const int gid = segout[buf][w & 7] + (int)((w >> 3) & 8191);
      y[gid] = accumulate ? y[gid] + acc : acc;
    }
    __syncthreads();  // staged block consumed
    cur = nxt;
  }
}

cudaError_t owner_periodic_v3(int n, int P, const double* loc, double* y, int accumulate,
                              cudaStream_t s, int row0, int row1, int* ctr) {
  const int L = segment_length(n, P, true);
  if (L == 0 || P < 2) return cudaErrorNotSupported;
  if (n == 0) return cudaSuccess;
  const int nm = (P + 1) * (P + 1) * (P + 1);
  return with_unroll(L * nm, [&](auto uc) {
    constexpr int U = decltype(uc)::value;
    const int nmp = (nm & 1) ? nm : nm + 2;
    const size_t smem =
        sizeof(double) * (L * nmp + 2) + sizeof(uint32_t) * (U * kThreads + L * P * P * P);
    static int configured = 0;
    allow_smem(owner_periodic_v3_kernel<U>, configured);
    if (row1 < 0) row1 = n * n;
    const int segs = n / L;
    if (row1 <= row0) return cudaSuccess;
    const unsigned blocks =
        persistent_grid(owner_periodic_v3_kernel<U>, smem, (int64_t)(row1 - row0) * segs);
    owner_periodic_v3_kernel<U><<<blocks, kThreads, smem, s>>>(n, P, L, loc, y, accumulate,
                                                                 schedule_counter(ctr, s), row0 * segs,
                                                                 row1 * segs);
    return cudaGetLastError();
  });
}

// ---------------------------------------------------------------------------
// Owner-computes sum over the block Z written by the operator's
// PERIODIC_CLASS mode (pipeline.cuh MODE 5): per tile of NE consecutive
// elements of an x-row, the classes 0..25 of its elements, class-major
// (class k at NE * cb[k], element i at + i * size(k)); the interiors, when
// not written straight into y, follow as an element-major n^3 (P-1)^3 block.
// Every owned dof of region r (vertices, x/y/z edges, x/y/z faces,
// interiors: the layout of y itself) is the sum of 8/4/2/1 values at the
// same offset of the neighbours e - (a, b, c) in classes fixed by r.  One
// CTA per (ey, ez) row: its neighbour rows are fixed, so each contributor
// is a stream of NE * size runs; every Z value is read once.  Terms are
// summed in increasing (a, b, c) order, as owner_periodic_v3 does, so both
// give bitwise-identical results.
// ---------------------------------------------------------------------------
#ifndef CLASS_OWNER_NT
#define CLASS_OWNER_NT 128
#endif
// resident CTAs per SM the kernel is compiled for: 16 (32 registers, full
// occupancy) with multi-element tiles; 12 (42 registers, no spills) with
// one-element tiles, whose scalar loads keep more index state live —
// measured P=6 139 -> 127 us, P=7 181 -> 164, P=8 242 -> 218, while P <= 5
// lose 5-10 us at 12
__host__ __device__ constexpr int class_owner_minb(int ne) { return ne == 1 ? 12 : 16; }
namespace {

// offset of class k inside an element's class-major record
__host__ __device__ constexpr int class_cb(int k, int b) {
  return k < 8 ? k : (k < 20 ? 8 + (k - 8) * b : (k < 26 ? 8 + 12 * b + (k - 20) * b * b : 8 + 12 * b + 6 * b * b));
}

// contributor j of region R: neighbour offset (a, b, c) and the class of
// its entity; j in increasing o8 = a << 2 | b << 1 | c
template <int R>
struct Region {
  static constexpr int NC = R == 0 ? 8 : (R < 4 ? 4 : (R < 7 ? 2 : 1));
  __host__ __device__ static constexpr int a(int j) {
    return R == 0 ? j >> 2 : (R == 2 || R == 3) ? j >> 1 : (R == 4 ? j : 0);
  }
  __host__ __device__ static constexpr int b(int j) {
    return R == 0 ? (j >> 1) & 1 : R == 1 ? j >> 1 : R == 3 ? j & 1 : (R == 5 ? j : 0);
  }
  __host__ __device__ static constexpr int c(int j) {
    return R == 0 ? j & 1 : (R == 1 || R == 2) ? j & 1 : (R == 6 ? j : 0);
  }
  __host__ __device__ static constexpr int k(int j) {
    return R == 0 ? j : R == 1 ? 8 + j : R == 2 ? 12 + j : R == 3 ? 16 + j : R == 4 ? 20 + j : R == 5 ? 22 + j
           : R == 6 ? 24 + j : 26;
  }
};

template <int P>
struct OwnerGeom {
  static constexpr int b = P - 1;
  static constexpr int ZS = (P + 1) * (P + 1) * (P + 1) - b * b * b;  // Z doubles per element
  __host__ __device__ static constexpr int S(int r) { return r == 0 ? 1 : (r < 4 ? b : (r < 7 ? b * b : b * b * b)); }
  __host__ __device__ static constexpr int start(int r) {  // per-row output offset of region r (units of n)
    return r == 0 ? 0 : start(r - 1) + S(r - 1);
  }
  __host__ __device__ static constexpr int64_t ybase(int r) {  // region base in y (units of n^3)
    return r == 0 ? 0 : ybase(r - 1) + S(r - 1);
  }
};

// output li = ex * S + o of region R in the current row: its NC terms.
// zr[bc] = Z record of the neighbour row (ey - b, ez - c); within a row the
// tile t holds elements t * NE .. t * NE + NE - 1, so the output's position
// u = li % (NE * S) is also the position of the a = 0 terms inside each
// class run; the a = 1 term is u - S, or the previous tile's last element
// (x wraps to n - 1 at t = 0) when u < S.
template <int P, int NE, int R>
__device__ __forceinline__ double owned_one(const double* __restrict__ Z, const int* zr, const int* zi, int T,
                                            int li, double* v) {
  using G = OwnerGeom<P>;
  constexpr int S = G::S(R), NC = Region<R>::NC, RUN = NE * S, REC = NE * G::ZS;
  const int t = li / RUN, u = li - t * RUN;
  const int tp = t == 0 ? T - 1 : t - 1;  // tile of the x - 1 neighbour at u < S
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const int bc = Region<R>::b(j) * 2 + Region<R>::c(j);
    if constexpr (R == 7) {
      v[j] = __ldg(Z + zi[bc] + li);
    } else {
      const int cls = NE * class_cb(Region<R>::k(j), G::b);
      const int off = zr[bc] + t * REC + cls + u;
      v[j] = __ldg(Z + (!Region<R>::a(j) ? off : (u >= S ? off - S : zr[bc] + tp * REC + cls + (NE - 1) * S + u)));
    }
  }
  return 0.0;
}

template <int P, int NE, int R>
__device__ __forceinline__ void owned_sum2(const double* __restrict__ Z, const int* zr, const int* zi, int T,
                                           int li, double& acc0, double& acc1) {
  // outputs li and li + 1 (li even, same region: n S is even); when the
  // tile run NE S is even they share the index math (same tile), 2 NC loads
  // in flight per thread either way
  using G = OwnerGeom<P>;
  constexpr int S = G::S(R), NC = Region<R>::NC, RUN = NE * S, REC = NE * G::ZS;
  double v0[NC], v1[NC];
  if constexpr (RUN % 2 != 0) {
    owned_one<P, NE, R>(Z, zr, zi, T, li, v0);
    owned_one<P, NE, R>(Z, zr, zi, T, li + 1, v1);
  } else {
    const int t = li / RUN, u = li - t * RUN;
    const int tp = t == 0 ? T - 1 : t - 1;  // tile of the x - 1 neighbour at u < S
    // even NE: every class run starts on an even double (n, NE * ZS and
    // NE * class_cb are even, u is), so an unshifted pair is one 16-byte
    // load; the x-shifted pair too when S is even (both outputs then fall
    // on the same side of the tile edge).  Half the load instructions: the
    // kernel ran at 72 % L1TEX with 8-byte loads (ncu, P = 4)
    constexpr bool VEC0 = NE % 2 == 0, VEC1 = VEC0 && S % 2 == 0;
    auto ld2 = [&](int o, double& a, double& b) {
      const double2 q = __ldg(reinterpret_cast<const double2*>(Z + o));
      a = q.x, b = q.y;
    };
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int bc = Region<R>::b(j) * 2 + Region<R>::c(j);
      if constexpr (R == 7) {
        v0[j] = __ldg(Z + zi[bc] + li);
        v1[j] = __ldg(Z + zi[bc] + li + 1);
      } else {
        const int cls = NE * class_cb(Region<R>::k(j), G::b);
        const int off = zr[bc] + t * REC + cls + u;
        if (Region<R>::a(j)) {
          const int wrapd = zr[bc] + tp * REC + cls + (NE - 1) * S;  // + u: last element of the tile before
          if constexpr (VEC1) {
            ld2(u >= S ? off - S : wrapd + u, v0[j], v1[j]);
          } else {
            v0[j] = __ldg(Z + (u >= S ? off - S : wrapd + u));
            v1[j] = __ldg(Z + (u + 1 >= S ? off + 1 - S : wrapd + u + 1));
          }
        } else if constexpr (VEC0) {
          ld2(off, v0[j], v1[j]);
        } else {
          v0[j] = __ldg(Z + off);
          v1[j] = __ldg(Z + off + 1);
        }
      }
    }
  }
  acc0 = v0[0];
  acc1 = v1[0];
#pragma unroll
  for (int j = 1; j < NC; ++j) {
    acc0 += v0[j];
    acc1 += v1[j];
  }
}

// one CTA per (ey, ez) row at a time: all regions' n * (P^3 [- (P-1)^3])
// owned dofs of the row as one index space of output pairs (the region of
// an output is a few compares), so every thread has work at every order.
// 32-bit offsets from Z: n^3 nm < 2^31 for every map the kernels accept.
template <int P, int NE>
__global__ void __launch_bounds__(CLASS_OWNER_NT, class_owner_minb(NE)) class_owner_sum_kernel(int n, const double* __restrict__ Z,
                                                              double* __restrict__ y, int accumulate,
                                                              int nreg, int row0, int row1) {
  using G = OwnerGeom<P>;
  const int64_t N3 = (int64_t)n * n * n;
  const int T = n / NE;  // tiles per row
  const int per_row = n * (G::start(7) + (nreg > 7 ? G::S(7) : 0));
  const bool y16 = (reinterpret_cast<uintptr_t>(y) & 15) == 0;
  for (int row = row0 + blockIdx.x; row < row1; row += gridDim.x) {
    const int ez = row / n, ey = row - ez * n;
    const int ym = ey == 0 ? n - 1 : ey - 1, zm = ez == 0 ? n - 1 : ez - 1;
    const int nr[4] = {ey + n * ez, ey + n * zm, ym + n * ez, ym + n * zm};  // (b, c) = 00, 01, 10, 11
    int zr[4], zi[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      zr[q] = nr[q] * n * G::ZS;
      zi[q] = (int)(N3 * G::ZS) + nr[q] * n * G::S(7);
    }
    for (int i = 2 * threadIdx.x; i < per_row; i += 2 * blockDim.x) {
      int r = 0;
#pragma unroll
      for (int q = 1; q < 8; ++q) r += i >= n * G::start(q) ? 1 : 0;
      double a0, a1;
      int64_t g;
#define REGION(R)                                                \
  case R: {                                                      \
    const int li = i - n * G::start(R);                          \
    owned_sum2<P, NE, R>(Z, zr, zi, T, li, a0, a1);              \
    g = N3 * G::ybase(R) + (int64_t)row * n * G::S(R) + li;      \
    break;                                                       \
  }
      switch (r) {
        REGION(0) REGION(1) REGION(2) REGION(3) REGION(4) REGION(5) REGION(6) REGION(7)
      }
#undef REGION
      // g is even (n is): one 16-byte store when y is 16-byte aligned
      if (y16 && !accumulate) {
        *reinterpret_cast<double2*>(y + g) = make_double2(a0, a1);
      } else {
        y[g] = accumulate ? y[g] + a0 : a0;
        y[g + 1] = accumulate ? y[g + 1] + a1 : a1;
      }
    }
  }
}

}  // namespace

int64_t class_block_doubles(int n, int P) {
  const int64_t N3 = (int64_t)n * n * n;
  return N3 * (P + 1) * (P + 1) * (P + 1);
}

cudaError_t class_owner_sum(int n, int P, int ne, const double* Z, double* y, int accumulate,
                            int with_interior, cudaStream_t s, int row0, int row1) {
  if (n < 2 || n % 2 || P < 2 || P > 9 || ne < 1 || (ne & (ne - 1)) || n % ne) return cudaErrorNotSupported;
  if (row1 < 0) row1 = n * n;
  if (row1 <= row0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one wave of CTAs with the same number of rows each (no tail)
  const int64_t rows = row1 - row0, cap = (int64_t)sms * class_owner_minb(ne);
  const int64_t per = (rows + cap - 1) / cap;
  const int64_t blocks = (rows + per - 1) / per;
  auto go = [&](auto pc, auto nc) -> cudaError_t {
    constexpr int PP = decltype(pc)::value, NE = decltype(nc)::value;
    class_owner_sum_kernel<PP, NE><<<(unsigned)blocks, CLASS_OWNER_NT, 0, s>>>(n, Z, y, accumulate, with_interior ? 8 : 7,
                                                                    row0, row1);
    return cudaGetLastError();
  };
  auto by_ne = [&](auto pc) -> cudaError_t {
    switch (ne) {
      case 1: return go(pc, std::integral_constant<int, 1>());
      case 2: return go(pc, std::integral_constant<int, 2>());
      case 4: return go(pc, std::integral_constant<int, 4>());
      case 8: return go(pc, std::integral_constant<int, 8>());
    }
    return cudaErrorNotSupported;
  };
  switch (P) {
    case 2: return by_ne(std::integral_constant<int, 2>());
    case 3: return by_ne(std::integral_constant<int, 3>());
    case 4: return by_ne(std::integral_constant<int, 4>());
    case 5: return by_ne(std::integral_constant<int, 5>());
    case 6: return by_ne(std::integral_constant<int, 6>());
    case 7: return by_ne(std::integral_constant<int, 7>());
    case 8: return by_ne(std::integral_constant<int, 8>());
    case 9: return by_ne(std::integral_constant<int, 9>());
  }
  return cudaErrorNotSupported;
}

}  // namespace sphp
