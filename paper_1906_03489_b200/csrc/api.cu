// C ABI of spechp_b200 (include/spechp_b200.h): handle management, argument
// checking with the reference's error wording, strategy dispatch and the
// assembly-map builders.  Every entry point cites the reference routine it
// replaces.
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/spechp_b200.h"
#include "dg.h"
#include "tri.h"
#include "common.cuh"
#include "kernels.h"
#include "misc.h"
#include "periodic.cuh"
#include "solver.h"
#include "tables.h"

// NVTX range around every apply-type entry point (tracing): shows
// up in nsys timelines and lets ncu filter launches (--nvtx --nvtx-include
// "sphp_helmholtz_assembled/").  Header-only NVTX v3: a no-op pointer check
// when no tool is attached.
namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

using namespace sphp;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(SPHP_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                         \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

int sm_count() {
  static int cache[64] = {0};
  int d = current_device();
  if (cache[d & 63] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess) n = 0;
    cache[d & 63] = n;
  }
  return cache[d & 63];
}

// per-device one-time upload of the constant-memory table pool
int ensure_tables_uploaded() {
  static std::mutex mu;
  static bool done[64] = {false};
  int d = current_device();
  std::lock_guard<std::mutex> lk(mu);
  if (!done[d & 63]) {
    cudaError_t e = upload_all_tables();
    if (e != cudaSuccess) return cuda_fail(e, "upload constant tables");
    done[d & 63] = true;
  }
  return SPHP_OK;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int dev = -1;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t ensure(size_t b) {
    if (p && bytes >= b) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, b ? b : 16);
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  // growth on a stream that is being captured would put cudaMalloc into the
  // graph: refused (reserve the workspace before capturing)
  cudaError_t ensure_on(size_t b, cudaStream_t s) {
    if (p && bytes >= b) return cudaSuccess;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (s) cudaStreamIsCapturing(s, &cap);
    if (cap != cudaStreamCaptureStatusNone) return cudaErrorStreamCaptureUnsupported;
    return ensure(b);
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

// Per-stream workspace of a handle: everything an apply writes besides its
// output.  Applies on distinct streams get distinct workspaces, so one
// handle may be applied concurrently on several streams (the handle itself
// is immutable after create); applies on one stream are ordered by it.
// Buffers are sized on first use on the stream (or by sphp_*_reserve,
// which a caller must do before capturing applies into a CUDA graph) and
// never shrink.
struct Workspace {
  DevBuf loc_x, loc_y;       // local blocks (split / owner / stdmat assembled), Z (class)
  DevBuf scratch;            // StdMat pointwise buffers
  DevBuf host_in, host_out;  // host-buffer applies: device staging
  DevBuf ctr;                // dynamic segment schedule counters (periodic kernels)
  // host-buffer pipeline: copy streams and per-slab events
  cudaStream_t pipe_h2d = nullptr, pipe_d2h = nullptr;
  std::vector<cudaEvent_t> pipe_ev;
  // sphp_gsys: one stream per batch and its events
  std::vector<cudaStream_t> bs;
  std::vector<cudaEvent_t> bev;
  ~Workspace() {
    for (cudaEvent_t e : pipe_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : bev) cudaEventDestroy(e);
    for (cudaStream_t q : bs) cudaStreamDestroy(q);
    if (pipe_h2d) cudaStreamDestroy(pipe_h2d);
    if (pipe_d2h) cudaStreamDestroy(pipe_d2h);
  }
  int* counter() { return ctr.ensure(2 * sizeof(int)) == cudaSuccess ? ctr.as<int>() : nullptr; }
};

class WorkspacePool {
 public:
  Workspace* get(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(mu_);
    for (auto& kv : v_)
      if (kv.first == s) return kv.second.get();
    v_.emplace_back(s, std::make_unique<Workspace>());
    return v_.back().second.get();
  }

 private:
  std::mutex mu_;
  std::vector<std::pair<cudaStream_t, std::unique_ptr<Workspace>>> v_;
};

}  // namespace

// ---------------------------------------------------------------------------
// fast-table pool (constant memory image)
// ---------------------------------------------------------------------------
namespace sphp {
const double* fast_table_pool() {
  static std::vector<double> pool;
  static std::once_flag once;
  std::call_once(once, [] {
    pool.assign(TAB_TOTAL, 0.0);
    for (int m = FAST_M_MIN; m <= FAST_M_MAX; ++m)
      for (int q = m + 1; q <= m + 2; ++q) {
        std::vector<double> z, w, B, Bd, D;
        make_rule(q, SPHP_POINTS_GAUSS_LOBATTO_LEGENDRE, z, w);
        basis_table(SPHP_BASIS_MODIFIED_A, m, z, B, Bd);
        diff_matrix(z, D);
        double* dst = pool.data() + tab_off(m, q);
        std::copy(B.begin(), B.end(), dst);
        std::copy(Bd.begin(), Bd.end(), dst + m * q);
        std::copy(D.begin(), D.end(), dst + 2 * m * q);
        std::copy(w.begin(), w.end(), dst + 2 * m * q + q * q);
        // even-odd tables (eo.cuh): GLL points are symmetric, Modified_A
        // rows 0/1 mirror each other and bubble k has parity (-1)^k
        const int H = eo_h(q), HF = eo_hf(q), ME = eo_me(m), MO = eo_mo(m);
        double* e = dst + 2 * m * q + q * q + q;
        double* BE = e;
        double* BO = BE + ME * H;
        double* BDE = BO + MO * H;
        double* BDO = BDE + ME * H;
        double* DE = BDO + MO * H;
        double* DO = DE + H * HF;
        double* DTE = DO + H * H;
        double* DTO = DTE + H * HF;
        for (int i = 0; i < H; ++i) {
          BE[0 * H + i] = 0.5 * (B[0 * q + i] + B[1 * q + i]);
          BO[0 * H + i] = 0.5 * (B[1 * q + i] - B[0 * q + i]);
          BDE[0 * H + i] = 0.0;
          BDO[0 * H + i] = 0.5 * (Bd[1 * q + i] - Bd[0 * q + i]);
          int ie = 1, io = 1;
          for (int k = 2; k < m; ++k) {
            if (k % 2 == 0) {
              BE[ie * H + i] = B[k * q + i];
              BDE[ie * H + i] = Bd[k * q + i];
              ++ie;
            } else {
              BO[io * H + i] = B[k * q + i];
              BDO[io * H + i] = Bd[k * q + i];
              ++io;
            }
          }
          for (int j = 0; j < HF; ++j) {
            DE[i * HF + j] = 0.5 * (D[i * q + j] - D[i * q + (q - 1 - j)]);
            DO[i * H + j] = 0.5 * (D[i * q + j] + D[i * q + (q - 1 - j)]);
            // transposed operator: (D^T)[i][j] = D[j][i]
            DTE[i * HF + j] = 0.5 * (D[j * q + i] - D[(q - 1 - j) * q + i]);
            DTO[i * H + j] = 0.5 * (D[j * q + i] + D[(q - 1 - j) * q + i]);
          }
          if (q % 2) {  // middle point
            DO[i * H + HF] = D[i * q + HF];
            DTO[i * H + HF] = D[HF * q + i];
          }
        }
      }
  });
  return pool.data();
}
cudaError_t upload_tables_hex_helm0();
cudaError_t upload_tables_hex_helm1();
cudaError_t upload_tables_hex_helm2();
cudaError_t upload_tables_hex_misc();
cudaError_t upload_tables_quad();
cudaError_t upload_all_tables() {
  cudaError_t e = upload_tables_hex_helm0();
  if (e == cudaSuccess) e = upload_tables_hex_helm1();
  if (e == cudaSuccess) e = upload_tables_hex_helm2();
  if (e == cudaSuccess) e = upload_tables_hex_misc();
  if (e == cudaSuccess) e = upload_tables_quad();
  return e;
}
}  // namespace sphp

// ---------------------------------------------------------------------------
// handles
// ---------------------------------------------------------------------------
struct sphp_tables {
  int shape = 0, dim = 0;
  int m[3] = {0, 0, 0}, q[3] = {0, 0, 0}, ptype[3] = {0, 0, 0}, btype[3] = {0, 0, 0};
  std::vector<double> z[3], w[3], B[3], Bd[3], D[3];
  int64_t nm = 0, np = 0;
  bool fast = false;  // sum-factorisation kernels available for this key
  // lazily built device copies
  std::mutex mu;
  DevBuf d_z, d_w, d_wstd, d_B, d_Bd;
  std::vector<double> wstd;  // tensor weights, point order
  // triangles: direction-2 table is Modified_B with nm rows; mode blocks,
  // collapse factors, and the packed device tables of tri.cu
  bool tri = false;
  std::vector<int> tri_p, tri_start;
  std::vector<double> tri_f, tri_g;
  DevBuf d_tri, d_tri_i;
  int tri_ntab = 0;
};

struct sphp_coll {
  sphp_tables* t = nullptr;
  int op = 0, strategy = 0, geom_kind = 0;
  int64_t E = 0, in_size = 0, out_size = 0;
  const double* geom = nullptr;
  int64_t gstride = 0, cs = 0;
  double lam = 0.0;
  // StdMat operators, built at create (and by set_lambda for Helmholtz)
  DevBuf mat_a;   // dense elemental operator
  DevBuf helm_H;  // Helmholtz element matrices
  WorkspacePool ws;
};

struct sphp_amap {
  int periodic = 0, n = 0, P = 0, nm = 0;
  int64_t E = 0, num_global = 0;
  int ncolours = 0;
  std::vector<int64_t> codes_host;  // explicit only
  std::vector<int64_t> colour_off;  // explicit only (ncolours+1)
  std::vector<int> elist_host;      // explicit only, element ids by colour
  int alg = SPHP_ASSEMBLY_OWNER;
  std::mutex mu;
  DevBuf d_codes, d_elist, d_rowp, d_ent;  // explicit: codes, colour lists, CSR
  DevBuf d_entity;                          // periodic: (E, 27) entity bases
  AmapDev dev() const {
    AmapDev a;
    a.periodic = periodic;
    a.n = n;
    a.P = P;
    a.nm = nm;
    a.E = E;
    a.num_global = num_global;
    a.codes = d_codes.as<int>();
    return a;
  }
};

namespace {

int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  while (e--) r *= b;
  return r;
}

int tables_device(sphp_tables* t) {
  std::lock_guard<std::mutex> lk(t->mu);
  if (t->d_z.p) return SPHP_OK;
  CK(t->d_z.ensure(sizeof(double) * t->q[0]));
  CK(t->d_w.ensure(sizeof(double) * t->q[0]));
  CK(cudaMemcpy(t->d_z.p, t->z[0].data(), sizeof(double) * t->q[0], cudaMemcpyHostToDevice));
  CK(cudaMemcpy(t->d_w.p, t->w[0].data(), sizeof(double) * t->q[0], cudaMemcpyHostToDevice));
  CK(t->d_wstd.ensure(sizeof(double) * t->np));
  CK(cudaMemcpy(t->d_wstd.p, t->wstd.data(), sizeof(double) * t->np, cudaMemcpyHostToDevice));
  CK(t->d_B.ensure(sizeof(double) * t->B[0].size()));
  CK(cudaMemcpy(t->d_B.p, t->B[0].data(), sizeof(double) * t->B[0].size(), cudaMemcpyHostToDevice));
  CK(t->d_Bd.ensure(sizeof(double) * t->Bd[0].size()));
  CK(cudaMemcpy(t->d_Bd.p, t->Bd[0].data(), sizeof(double) * t->Bd[0].size(), cudaMemcpyHostToDevice));
  return SPHP_OK;
}

// dense (Kronecker) operators on host --------------------------------------
// B[n][i] = prod_a B_a[idx_a(n)][idx_a(i)]   (stdregions.py:189-198)
std::vector<double> dense_bwd(const sphp_tables* t) {
  std::vector<double> M((size_t)t->nm * t->np);
  if (t->tri) {  // stdregions.py:199-208, collapsed-vertex mode (0,1) gains A1[1] B2[1]
    const int Q1 = t->q[0], Q2 = t->q[1];
    for (int64_t n = 0; n < t->nm; ++n) {
      const int p = t->tri_p[n];
      for (int i = 0; i < Q1; ++i)
        for (int j = 0; j < Q2; ++j) {
          double v = t->B[0][(size_t)p * Q1 + i] * t->B[1][(size_t)n * Q2 + j];
          if (n == 1) v += t->B[0][(size_t)1 * Q1 + i] * t->B[1][(size_t)n * Q2 + j];
          M[(size_t)n * t->np + (size_t)i * Q2 + j] = v;
        }
    }
    return M;
  }
  for (int64_t n = 0; n < t->nm; ++n)
    for (int64_t i = 0; i < t->np; ++i) {
      int64_t rn = n, ri = i;
      double v = 1.0;
      for (int a = t->dim - 1; a >= 0; --a) {
        int pn = (int)(rn % t->m[a]), pi = (int)(ri % t->q[a]);
        rn /= t->m[a];
        ri /= t->q[a];
        v *= t->B[a][(size_t)pn * t->q[a] + pi];
      }
      M[(size_t)n * t->np + i] = v;
    }
  return M;
}
// derivative along direction a acting on flattened point vectors:
// (D_a)[i][j] (stdregions.py:218-235)
double dense_deriv(const sphp_tables* t, int a, int64_t i, int64_t j) {
  if (t->tri) {  // collapsed chain rule (stdregions.py:221-235)
    const int Q2 = t->q[1], Q1 = t->q[0];
    const int i1 = (int)(i / Q2), i2 = (int)(i % Q2), j1 = (int)(j / Q2), j2 = (int)(j % Q2);
    const double k1 = (i2 == j2) ? t->D[0][(size_t)i1 * Q1 + j1] : 0.0;
    const double k2 = (i1 == j1) ? t->D[1][(size_t)i2 * Q2 + j2] : 0.0;
    return a == 0 ? t->tri_f[i2] * k1 : t->tri_g[i] * k1 + k2;
  }
  int64_t ri = i, rj = j;
  double v = 1.0;
  for (int b = t->dim - 1; b >= 0; --b) {
    int ii = (int)(ri % t->q[b]), jj = (int)(rj % t->q[b]);
    ri /= t->q[b];
    rj /= t->q[b];
    if (b == a)
      v *= t->D[b][(size_t)ii * t->q[b] + jj];
    else if (ii != jj)
      return 0.0;
  }
  return v;
}

int64_t geom_record(const sphp_tables* t, int kind) {
  const int d = t->dim;
  const int64_t cs = (t->np + 1) & ~1LL;
  switch (kind) {
    case SPHP_GEOM_NONE: return 0;
    case SPHP_GEOM_AFFINE: return d == 3 ? 10 : 6;
    case SPHP_GEOM_POINT: return (1 + d * d) * cs;
    case SPHP_GEOM_METRIC: return (d * (d + 1) / 2 + 1) * cs;
  }
  return -1;
}

OpArgs base_args(const sphp_coll* c) {
  OpArgs a;
  a.M = c->t->m[0];
  a.Q = c->t->q[0];
  a.E = c->E;
  a.in = nullptr;
  a.out = nullptr;
  a.geom = c->geom;
  a.geom_kind = c->geom_kind;
  a.gstride = c->gstride;
  a.lam = c->lam;
  a.num_sms = sm_count();
  a.mode = AsmMode::LOCAL;
  a.xg = nullptr;
  a.yg = nullptr;
  a.elist = nullptr;
  a.nlist = 0;
  a.codes = nullptr;
  a.ent_g = nullptr;
  a.n = 0;
  a.colour = 0;
  return a;
}

cudaError_t sumfac_launch(const sphp_coll* c, const OpArgs& a, cudaStream_t s) {
  if (c->t->tri) {
    TriJob j;
    j.op = c->op;
    j.m1 = c->t->m[0];
    j.nm = (int)c->t->nm;
    j.Q1 = c->t->q[0];
    j.Q2 = c->t->q[1];
    j.ntab = c->t->tri_ntab;
    j.tab = c->t->d_tri.as<double>();
    j.itab = c->t->d_tri_i.as<int>();
    j.geom_kind = a.geom_kind;
    j.geom = a.geom;
    j.gstride = a.gstride;
    j.cs = c->cs;
    j.E = a.E;
    j.in = a.in;
    j.out = a.out;
    return tri_apply(j, a.num_sms, s);
  }
  const bool hex = c->t->shape == SPHP_SHAPE_HEX;
  switch (c->op) {
    case SPHP_OP_BWD_TRANS: return hex ? hex_bwd(a, s) : quad_bwd(a, s);
    case SPHP_OP_IPRODUCT_WRT_BASE: return hex ? hex_iprod(a, s) : quad_iprod(a, s);
    case SPHP_OP_PHYS_DERIV: return hex ? hex_physderiv(a, s) : quad_physderiv(a, s);
    case SPHP_OP_IPRODUCT_WRT_DERIV_BASE: return hex ? hex_ipderiv(a, s) : quad_ipderiv(a, s);
    case SPHP_OP_HELMHOLTZ: return hex ? hex_helmholtz(a, s) : quad_helmholtz(a, s);
  }
  return cudaErrorInvalidValue;
}

PointJob point_job(const sphp_coll* c) {
  PointJob j;
  j.dim = c->t->dim;
  j.kind = c->geom_kind;
  j.E = c->E;
  j.np = c->t->np;
  j.cs = c->cs;
  j.stride = c->gstride;
  j.geom = c->geom;
  j.wstd = c->t->d_wstd.as<double>();
  return j;
}

// build the StdMat operators of a collection: at create (and, for the
// Helmholtz element matrices, which depend on lambda, in set_lambda), on a
// private stream, synchronously — applies never build or allocate them
int stdmat_prepare(sphp_coll* c) {
  sphp_tables* t = c->t;
  const int64_t nm = t->nm, np = t->np;
  const int d = t->dim;
  if (c->op == SPHP_OP_HELMHOLTZ) {
    if (!t->fast)
      return fail(SPHP_ERR_UNSUPPORTED, "stdmat Helmholtz needs a sum-factorisation key to build H_e");
    // dense element matrices: up to half the free device memory (B200: 180
    // GB HBM3e; e.g. the cfg5 P = 6 / P = 7 batches, 21 / 46 GB)
    const double bytes = 8.0 * c->E * nm * nm;
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    if (bytes > 0.5 * (double)free_b) {
      char buf[160];
      std::snprintf(buf, sizeof(buf),
                    "stdmat Helmholtz element matrices (%.1f GB) exceed half the free device memory (%.1f GB)",
                    bytes / 1e9, free_b / 1e9);
      return fail(SPHP_ERR_UNSUPPORTED, buf);
    }
    CK(c->helm_H.ensure((size_t)bytes));
    DevBuf ux, uy;
    CK(ux.ensure(sizeof(double) * c->E * nm));
    CK(uy.ensure(sizeof(double) * c->E * nm));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    // column n of every H_e = fused Helmholtz applied to unit vector e_n
    OpArgs a = base_args(c);
    cudaError_t e = cudaSuccess;
    for (int n = 0; n < nm && e == cudaSuccess; ++n) {
      e = unit_block(c->E, (int)nm, n, ux.as<double>(), s);
      a.in = ux.as<double>();
      a.out = uy.as<double>();
      if (e == cudaSuccess) e = sumfac_launch(c, a, s);
      if (e == cudaSuccess) e = store_column(c->E, (int)nm, n, uy.as<double>(), c->helm_H.as<double>(), s);
    }
    if (e == cudaSuccess) e = symmetrise(c->E, (int)nm, c->helm_H.as<double>(), s);  // geometry.py:184
    const cudaError_t e2 = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (e != cudaSuccess) return cuda_fail(e, "stdmat Helmholtz build");
    if (e2 != cudaSuccess) return cuda_fail(e2, "stdmat Helmholtz build");
    return SPHP_OK;
  }
  std::vector<double> Bm = dense_bwd(t);  // (nm, np)
  std::vector<double> A;
  switch (c->op) {
    case SPHP_OP_BWD_TRANS:
      A = Bm;  // out = in (E,nm) @ B (nm,np)   collections.py:205
      break;
    case SPHP_OP_IPRODUCT_WRT_BASE:
      A.assign((size_t)np * nm, 0.0);  // B^T (np, nm)   collections.py:218
      for (int64_t n = 0; n < nm; ++n)
        for (int64_t i = 0; i < np; ++i) A[(size_t)i * nm + n] = Bm[(size_t)n * np + i];
      break;
    case SPHP_OP_PHYS_DERIV:
      A.assign((size_t)np * d * np, 0.0);  // [D_0^T .. D_{d-1}^T] (np, d*np)   collections.py:228-229
      for (int a = 0; a < d; ++a)
        for (int64_t i = 0; i < np; ++i)
          for (int64_t j = 0; j < np; ++j) A[(size_t)j * d * np + a * np + i] = dense_deriv(t, a, i, j);
      break;
    case SPHP_OP_IPRODUCT_WRT_DERIV_BASE: {
      // stacked B_a^T = D_a B^T (d*np, nm)   geometry.py:163-168
      A.assign((size_t)d * np * nm, 0.0);
      for (int a = 0; a < d; ++a)
        for (int64_t i = 0; i < np; ++i)
          for (int64_t j = 0; j < np; ++j) {
            const double v = dense_deriv(t, a, i, j);
            if (v == 0.0) continue;
            for (int64_t n = 0; n < nm; ++n) A[((size_t)a * np + i) * nm + n] += v * Bm[(size_t)n * np + j];
          }
      break;
    }
  }
  CK(c->mat_a.ensure(sizeof(double) * A.size()));
  CK(cudaMemcpy(c->mat_a.p, A.data(), sizeof(double) * A.size(), cudaMemcpyHostToDevice));
  return SPHP_OK;
}

int ws_fail(cudaError_t e, const char* where) {
  if (e == cudaErrorStreamCaptureUnsupported)
    return fail(SPHP_ERR_BAD_ARG, std::string(where) +
                                      ": the workspace of this stream is not reserved (call the handle's "
                                      "reserve entry point before capturing applies into a CUDA graph)");
  return cuda_fail(e, where);
}
#define CKW(call)                                         \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return ws_fail(_e, #call);     \
  } while (0)

int stdmat_apply(sphp_coll* c, const double* in, double* out, cudaStream_t s) {
  Workspace* w = c->ws.get(s);
  sphp_tables* t = c->t;
  const int64_t nm = t->nm, np = t->np;
  const int d = t->dim;
  const double* A = c->mat_a.as<double>();
  switch (c->op) {
    case SPHP_OP_BWD_TRANS:
      CK(dgemm(c->E, (int)np, (int)nm, in, A, out, s));
      break;
    case SPHP_OP_IPRODUCT_WRT_BASE:
      CKW(w->scratch.ensure_on(sizeof(double) * c->E * np, s));
      CK(pointwise(0, point_job(c), in, w->scratch.as<double>(), s));
      CK(dgemm(c->E, (int)nm, (int)np, w->scratch.as<double>(), A, out, s));
      break;
    case SPHP_OP_PHYS_DERIV:
      CK(dgemm(c->E, (int)(d * np), (int)np, in, A, out, s));
      if (c->geom_kind != SPHP_GEOM_NONE) CK(pointwise(1, point_job(c), nullptr, out, s));
      break;
    case SPHP_OP_IPRODUCT_WRT_DERIV_BASE:
      CKW(w->scratch.ensure_on(sizeof(double) * c->E * d * np, s));
      CK(pointwise(2, point_job(c), in, w->scratch.as<double>(), s));
      CK(dgemm(c->E, (int)nm, (int)(d * np), w->scratch.as<double>(), A, out, s));
      break;
    case SPHP_OP_HELMHOLTZ:
      CK(elem_matvec(c->E, (int)nm, c->helm_H.as<double>(), in, out, s));
      break;
    default:
      return fail(SPHP_ERR_BAD_ARG, "unknown operator");
  }
  return SPHP_OK;
}

int64_t mac_count(const sphp_coll* c) {
  const sphp_tables* t = c->t;
  const int d = t->dim;
  const int64_t m = t->m[0], Q = t->q[0], nm = t->nm, np = t->np, E = c->E;
  const bool geo = c->geom_kind != SPHP_GEOM_NONE;
  const bool sm = c->strategy == SPHP_STRATEGY_CUDA_STDMAT;
  int64_t staged = (d == 2) ? m * m * Q + m * Q * Q : m * m * m * Q + m * m * Q * Q + m * Q * Q * Q;
  if (t->tri) {  // collections.py:250-273, triangle staged shapes
    const int64_t q1 = t->q[0], q2 = t->q[1];
    staged = (nm + 1) * q2 + m * q1 * q2;
    int64_t per = 0;
    switch (c->op) {
      case SPHP_OP_BWD_TRANS: per = sm ? nm * np : staged; break;
      case SPHP_OP_IPRODUCT_WRT_BASE: per = np + (sm ? nm * np : staged); break;
      default: per = (sm ? 2 * np * np : q1 * q1 * q2 + q1 * q2 * q2 + 2 * np) + (geo ? 4 * np : 0); break;
    }
    return E * per;
  }
  const int64_t dense = nm * np;
  int64_t per = 0;
  switch (c->op) {
    case SPHP_OP_BWD_TRANS: per = sm ? dense : staged; break;
    case SPHP_OP_IPRODUCT_WRT_BASE: per = np + (sm ? dense : staged); break;
    case SPHP_OP_PHYS_DERIV: per = (sm ? d * np * np : d * ipow(Q, d + 1)) + (geo ? d * d * np : 0); break;
    case SPHP_OP_IPRODUCT_WRT_DERIV_BASE:
      per = (sm ? d * np * nm : d * ipow(Q, d + 1) + staged) + (d * d + d) * np;
      break;
    case SPHP_OP_HELMHOLTZ:
      per = sm ? nm * nm : 2 * staged + 2 * d * ipow(Q, d + 1) + (d * d + d + 2) * np;
      break;
  }
  return E * per;
}

int64_t hbm_bytes(const sphp_coll* c) {
  const sphp_tables* t = c->t;
  const int d = t->dim;
  const int64_t nm = t->nm, np = t->np, E = c->E;
  int64_t io = 8 * E * (c->in_size + c->out_size);
  int64_t g = 0;
  const bool pt = c->geom_kind == SPHP_GEOM_POINT || c->geom_kind == SPHP_GEOM_METRIC;
  switch (c->op) {
    case SPHP_OP_IPRODUCT_WRT_BASE: g = c->geom_kind == SPHP_GEOM_NONE ? 0 : (pt ? np : 1); break;
    case SPHP_OP_PHYS_DERIV: g = c->geom_kind == SPHP_GEOM_NONE ? 0 : (pt ? d * d * np : d * d); break;
    case SPHP_OP_IPRODUCT_WRT_DERIV_BASE:
      g = c->geom_kind == SPHP_GEOM_NONE ? 0 : (pt ? (1 + d * d) * np : 1 + d * d);
      break;
    case SPHP_OP_HELMHOLTZ:
      if (c->strategy == SPHP_STRATEGY_CUDA_STDMAT)
        g = nm * nm;
      else
        g = c->geom_kind == SPHP_GEOM_METRIC ? (d * (d + 1) / 2 + 1) * np : 1 + d * d;
      break;
  }
  return io + 8 * E * g;
}

}  // namespace

// stdregions.make_tri / StdExpansion(Shape.TRI) (stdregions.py:83-240, 402-408):
// direction 1 Modified_A, direction 2 Modified_B (basis.py:117-157) with the
// collapse Jacobian (1 - eta2)/2 folded into the direction-2 weights
int tables_create_tri(const int* nmodes, const int* npoints, const int* points_type,
                      const int* basis_type, sphp_tables** out) {
  if (basis_type[1] != SPHP_BASIS_MODIFIED_B)
    return fail(SPHP_ERR_BAD_ARG, "triangle direction 2 must use the collapsed-direction basis");
  if (basis_type[0] != SPHP_BASIS_MODIFIED_A)
    return fail(SPHP_ERR_BAD_ARG, "triangle direction 1 must be modal");
  if (nmodes[1] < nmodes[0]) return fail(SPHP_ERR_BAD_ARG, "triangle needs P2 >= P1");
  auto* t = new sphp_tables();
  t->shape = SPHP_SHAPE_TRI;
  t->dim = 2;
  t->tri = true;
  try {
    for (int a = 0; a < 2; ++a) {
      t->m[a] = nmodes[a];
      t->q[a] = npoints[a];
      t->ptype[a] = points_type[a];
      t->btype[a] = basis_type[a];
      if (nmodes[a] < 2) throw std::invalid_argument("modified basis needs num_modes >= 2");
      if (npoints[a] < 1) throw std::invalid_argument("num_points must be a positive integer");
      make_rule(npoints[a], points_type[a], t->z[a], t->w[a]);
      diff_matrix(t->z[a], t->D[a]);
    }
    basis_table(SPHP_BASIS_MODIFIED_A, nmodes[0], t->z[0], t->B[0], t->Bd[0]);
    modified_b_table(nmodes[0] - 1, nmodes[1] - 1, t->z[1], t->B[1], t->Bd[1], t->tri_p, t->tri_start);
  } catch (const std::exception& ex) {
    delete t;
    return fail(SPHP_ERR_BAD_ARG, ex.what());
  }
  const int Q1 = t->q[0], Q2 = t->q[1];
  t->nm = (int64_t)t->tri_p.size();
  t->np = (int64_t)Q1 * Q2;
  t->fast = false;
  t->wstd.resize(t->np);
  t->tri_f.resize(Q2);
  t->tri_g.resize(t->np);
  for (int j = 0; j < Q2; ++j) t->tri_f[j] = 2.0 / (1.0 - t->z[1][j]);
  for (int i = 0; i < Q1; ++i)
    for (int j = 0; j < Q2; ++j) {
      t->wstd[(size_t)i * Q2 + j] = t->w[0][i] * (t->w[1][j] * 0.5 * (1.0 - t->z[1][j]));
      t->tri_g[(size_t)i * Q2 + j] = (1.0 + t->z[0][i]) / (1.0 - t->z[1][j]);
    }
  *out = t;
  return SPHP_OK;
}

// packed device tables for tri.cu (once per tables object)
int tri_tables_device(sphp_tables* t) {
  std::lock_guard<std::mutex> lk(t->mu);
  if (t->d_tri.p) return SPHP_OK;
  std::vector<double> tab;
  auto put = [&](const std::vector<double>& v) { tab.insert(tab.end(), v.begin(), v.end()); };
  put(t->B[0]);
  put(t->B[1]);
  put(t->D[0]);
  put(t->D[1]);
  put(t->tri_f);
  put(t->tri_g);
  put(t->wstd);
  std::vector<int> it(t->tri_p);
  it.insert(it.end(), t->tri_start.begin(), t->tri_start.end());
  CK(t->d_tri.ensure(sizeof(double) * tab.size()));
  CK(cudaMemcpy(t->d_tri.p, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice));
  CK(t->d_tri_i.ensure(sizeof(int) * it.size()));
  CK(cudaMemcpy(t->d_tri_i.p, it.data(), sizeof(int) * it.size(), cudaMemcpyHostToDevice));
  t->tri_ntab = (int)tab.size();
  return SPHP_OK;
}

// ===========================================================================
extern "C" {

int sphp_abi_version(void) { return SPHP_ABI_VERSION; }
const char* sphp_last_error(void) { return g_err.c_str(); }
int sphp_device_sm_count(void) { return sm_count(); }
int sphp_hex_helmholtz_plan(int M, int Q) {
  if (!sphp::fast_key(M, Q) || M > 9) return -1;
  if (sphp::col_plan(Q)) return 3;
  return Q % 4 == 0 ? 1 : 0;
}

// stdregions.StdExpansion (stdregions.py:70-240)
int sphp_tables_create(int shape, const int* nmodes, const int* npoints, const int* points_type,
                       const int* basis_type, sphp_tables** out) {
  if (!out || !nmodes || !npoints || !points_type || !basis_type)
    return fail(SPHP_ERR_BAD_ARG, "null argument");
  int dim;
  switch (shape) {
    case SPHP_SHAPE_SEG: dim = 1; break;
    case SPHP_SHAPE_QUAD: dim = 2; break;
    case SPHP_SHAPE_HEX: dim = 3; break;
    case SPHP_SHAPE_TRI: return tables_create_tri(nmodes, npoints, points_type, basis_type, out);
    default: return fail(SPHP_ERR_BAD_ARG, "unknown shape");
  }
  auto* t = new sphp_tables();
  t->shape = shape;
  t->dim = dim;
  try {
    for (int a = 0; a < dim; ++a) {
      t->m[a] = nmodes[a];
      t->q[a] = npoints[a];
      t->ptype[a] = points_type[a];
      t->btype[a] = basis_type[a];
      if (nmodes[a] < 1) throw std::invalid_argument("num_modes must be positive");
      if (npoints[a] < 1) throw std::invalid_argument("num_points must be a positive integer");
      if (basis_type[a] == SPHP_BASIS_MODIFIED_B)
        throw std::invalid_argument("collapsed-direction basis is only valid on triangles");
      make_rule(npoints[a], points_type[a], t->z[a], t->w[a]);
      basis_table(basis_type[a], nmodes[a], t->z[a], t->B[a], t->Bd[a]);
      diff_matrix(t->z[a], t->D[a]);
    }
  } catch (const std::exception& ex) {
    delete t;
    return fail(SPHP_ERR_BAD_ARG, ex.what());
  }
  t->nm = 1;
  t->np = 1;
  for (int a = 0; a < dim; ++a) {
    t->nm *= t->m[a];
    t->np *= t->q[a];
  }
  bool uniform = true;
  for (int a = 1; a < dim; ++a)
    uniform = uniform && t->m[a] == t->m[0] && t->q[a] == t->q[0] && t->ptype[a] == t->ptype[0] &&
              t->btype[a] == t->btype[0];
  t->fast = uniform && (shape == SPHP_SHAPE_QUAD || shape == SPHP_SHAPE_HEX) &&
            t->ptype[0] == SPHP_POINTS_GAUSS_LOBATTO_LEGENDRE && t->btype[0] == SPHP_BASIS_MODIFIED_A &&
            fast_key(t->m[0], t->q[0]) && (shape == SPHP_SHAPE_QUAD || t->m[0] <= 9);
  // tensor weights in point order (stdregions.py:113-121)
  t->wstd.assign(t->np, 1.0);
  for (int64_t i = 0; i < t->np; ++i) {
    int64_t r = i;
    double w = 1.0;
    int idx[3] = {0, 0, 0};
    for (int a = dim - 1; a >= 0; --a) {
      idx[a] = (int)(r % t->q[a]);
      r /= t->q[a];
    }
    for (int a = 0; a < dim; ++a) w *= t->w[a][idx[a]];
    t->wstd[i] = w;
  }
  *out = t;
  return SPHP_OK;
}

int sphp_tables_destroy(sphp_tables* t) {
  delete t;
  return SPHP_OK;
}

int sphp_tables_query(const sphp_tables* t, int dir, double* z, double* w, double* B, double* Bd,
                      double* D) {
  if (!t || dir < 0 || dir >= t->dim) return fail(SPHP_ERR_BAD_ARG, "bad direction");
  // triangle direction 2: the Modified_B table has one row per mode
  const size_t q = t->q[dir], m = (t->tri && dir == 1) ? (size_t)t->nm : (size_t)t->m[dir];
  if (z) std::memcpy(z, t->z[dir].data(), sizeof(double) * q);
  if (w) std::memcpy(w, t->w[dir].data(), sizeof(double) * q);
  if (B) std::memcpy(B, t->B[dir].data(), sizeof(double) * m * q);
  if (Bd) std::memcpy(Bd, t->Bd[dir].data(), sizeof(double) * m * q);
  if (D) std::memcpy(D, t->D[dir].data(), sizeof(double) * q * q);
  return SPHP_OK;
}

int sphp_tables_sizes(const sphp_tables* t, int64_t* nmodes, int64_t* npoints, int* dim) {
  if (!t) return fail(SPHP_ERR_BAD_ARG, "null tables");
  if (nmodes) *nmodes = t->nm;
  if (npoints) *npoints = t->np;
  if (dim) *dim = t->dim;
  return SPHP_OK;
}

int64_t sphp_geom_stride(const sphp_tables* t, int kind) {
  if (!t) return -1;
  return geom_record(t, kind);
}

// geometry.geom_factors (geometry.py:125-142) for analytic structured maps
int sphp_geom_analytic(const sphp_tables* tc, int kind, int mapping, int n, const double* lengths,
                       double amp, int64_t e0, int64_t E, const int64_t* ids, double* geom,
                       sphp_stream stream) {
  sphp_tables* t = const_cast<sphp_tables*>(tc);
  if (!t || !geom || n < 1 || E < 0) return fail(SPHP_ERR_BAD_ARG, "bad geometry arguments");
  if (t->dim < 2) return fail(SPHP_ERR_UNSUPPORTED, "analytic geometry needs quad or hex");
  for (int a = 1; a < t->dim; ++a)
    if (t->q[a] != t->q[0]) return fail(SPHP_ERR_UNSUPPORTED, "analytic geometry needs equal Q per direction");
  if (kind != SPHP_GEOM_AFFINE && kind != SPHP_GEOM_POINT && kind != SPHP_GEOM_METRIC)
    return fail(SPHP_ERR_BAD_ARG, "unknown geometry encoding");
  if (kind == SPHP_GEOM_AFFINE && mapping != SPHP_MAP_AFFINE)
    return fail(SPHP_ERR_BAD_ARG, "AFFINE encoding needs an affine map (constant Jacobian)");
  if ((mapping == SPHP_MAP_QUAD_SINE && t->dim != 2) || (mapping == SPHP_MAP_HEX_SINE && t->dim != 3))
    return fail(SPHP_ERR_BAD_ARG, "mapping does not match the element dimension");
  int rc = tables_device(t);
  if (rc) return rc;
  GeomJob j;
  j.dim = t->dim;
  j.Q = t->q[0];
  j.n = n;
  j.kind = kind;
  j.mapping = mapping;
  j.E = E;
  j.e0 = e0;
  j.npts = t->np;
  j.cs = (t->np + 1) & ~1LL;
  j.stride = geom_record(t, kind);
  j.ids = ids;
  j.z = t->d_z.as<double>();
  j.w = t->d_w.as<double>();
  for (int a = 0; a < 3; ++a) j.L[a] = lengths ? lengths[a < t->dim ? a : 0] : 1.0;
  j.amp = amp;
  j.out = geom;
  int* bad = nullptr;
  CK(cudaMalloc(&bad, sizeof(int)));
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), s);
  if (e == cudaSuccess) e = geom_analytic(j, bad, s);
  int hbad = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(bad);
  if (e != cudaSuccess) return cuda_fail(e, "sphp_geom_analytic");
  if (hbad)  // geometry.py:133-136 GeometryError wording
    return fail(SPHP_ERR_BAD_ARG, "non-positive Jacobian at quadrature point(s); invalid element");
  return SPHP_OK;
}

int sphp_geom_from_factors(const sphp_tables* tc, int kind, int64_t E, const double* wj,
                           const double* inv, double* geom, sphp_stream stream) {
  sphp_tables* t = const_cast<sphp_tables*>(tc);
  if (!t || !wj || !inv || !geom) return fail(SPHP_ERR_BAD_ARG, "null argument");
  if (kind != SPHP_GEOM_POINT && kind != SPHP_GEOM_METRIC)
    return fail(SPHP_ERR_BAD_ARG, "from_factors produces POINT or METRIC encodings");
  GeomJob j;
  std::memset(&j, 0, sizeof(j));
  j.dim = t->dim;
  j.Q = t->q[0];
  j.kind = kind;
  j.E = E;
  j.npts = t->np;
  j.cs = (t->np + 1) & ~1LL;
  j.stride = geom_record(t, kind);
  j.out = geom;
  int* bad = nullptr;
  CK(cudaMalloc(&bad, sizeof(int)));
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), s);
  if (e == cudaSuccess) e = geom_convert(j, wj, inv, bad, s);
  int hbad = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(bad);
  if (e != cudaSuccess) return cuda_fail(e, "sphp_geom_from_factors");
  if (hbad) return fail(SPHP_ERR_BAD_ARG, "non-positive world weight (w*|J|) in GeomFactors");
  return SPHP_OK;
}

// geometry.geom_factors (geometry.py:125-142) on the device, from the
// reference-direction derivatives of the coordinate map at the points
int sphp_geom_from_jacobian(const sphp_tables* tc, int kind, int64_t E, const double* dx,
                            const double* dy, double* geom, int64_t* first_bad, sphp_stream stream) {
  sphp_tables* t = const_cast<sphp_tables*>(tc);
  if (!t || !dx || !dy || !geom) return fail(SPHP_ERR_BAD_ARG, "null argument");
  if (t->dim != 2) return fail(SPHP_ERR_UNSUPPORTED, "coordinate-map geometry is 2D (quad, tri)");
  if (kind != SPHP_GEOM_POINT && kind != SPHP_GEOM_METRIC)
    return fail(SPHP_ERR_BAD_ARG, "geometry from a map produces POINT or METRIC encodings");
  if (first_bad) *first_bad = -1;
  if (E == 0) return SPHP_OK;
  if (int rc = tables_device(t)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t np = t->np;
  DevBuf scratch;
  CK(scratch.ensure(sizeof(double) * E * np * 5 + 2 * sizeof(unsigned long long)));
  double* wj = scratch.as<double>();
  double* inv = wj + E * np;
  auto* bad = reinterpret_cast<unsigned long long*>(inv + E * np * 4);
  const unsigned long long init[2] = {0ull, ~0ull};
  CK(cudaMemcpyAsync(bad, init, sizeof(init), cudaMemcpyHostToDevice, s));
  CK(jacobian_factors(E, np, dx, dy, t->d_wstd.as<double>(), wj, inv, bad, s));
  unsigned long long hb[2];
  CK(cudaMemcpyAsync(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hb[0]) {
    if (first_bad) *first_bad = (int64_t)hb[1];
    return fail(SPHP_ERR_BAD_ARG, "element " + std::to_string(hb[1]) + ": non-positive Jacobian at " +
                                      std::to_string(hb[0]) + " quadrature point(s); invalid element");
  }
  GeomJob j;
  std::memset(&j, 0, sizeof(j));
  j.dim = 2;
  j.kind = kind;
  j.E = E;
  j.npts = np;
  j.cs = (np + 1) & ~1LL;
  j.stride = geom_record(t, kind);
  j.out = geom;
  int* cbad = reinterpret_cast<int*>(bad);
  CK(cudaMemsetAsync(cbad, 0, sizeof(int), s));
  CK(geom_convert(j, wj, inv, cbad, s));
  CK(cudaStreamSynchronize(s));
  return SPHP_OK;
}

// collections.Collection.__init__ (collections.py:79-129)
int sphp_collection_create(const sphp_tables* tc, int op, int strategy, int64_t E, int geom_kind,
                           const double* geom, double lambda, sphp_coll** out) {
  sphp_tables* t = const_cast<sphp_tables*>(tc);
  if (!t || !out) return fail(SPHP_ERR_BAD_ARG, "null argument");
  if (E < 1) return fail(SPHP_ERR_BAD_ARG, "empty element group");  // collections.py:63-64
  if (op < SPHP_OP_BWD_TRANS || op > SPHP_OP_HELMHOLTZ) return fail(SPHP_ERR_BAD_ARG, "unknown operator");
  if (strategy != SPHP_STRATEGY_CUDA_SUMFAC && strategy != SPHP_STRATEGY_CUDA_STDMAT)
    return fail(SPHP_ERR_BAD_ARG, "strategy must be concrete");  // collections.py:80-81
  if (t->dim < 2) return fail(SPHP_ERR_UNSUPPORTED, "segment collections are not built on the GPU");
  if (geom_kind < SPHP_GEOM_NONE || geom_kind > SPHP_GEOM_METRIC)
    return fail(SPHP_ERR_BAD_ARG, "unknown geometry encoding");
  if (geom_kind != SPHP_GEOM_NONE && !geom) return fail(SPHP_ERR_BAD_ARG, "geometry pointer is null");
  if (op == SPHP_OP_HELMHOLTZ) {
    if (geom_kind != SPHP_GEOM_METRIC && geom_kind != SPHP_GEOM_AFFINE)
      return fail(SPHP_ERR_BAD_ARG, "Helmholtz needs METRIC or AFFINE geometry");
  } else if (geom_kind == SPHP_GEOM_METRIC) {
    return fail(SPHP_ERR_BAD_ARG, "METRIC geometry is specific to the Helmholtz operator");
  }
  if (op == SPHP_OP_BWD_TRANS && geom_kind != SPHP_GEOM_NONE) geom_kind = SPHP_GEOM_NONE;
  if (t->tri) {
    if (op != SPHP_OP_BWD_TRANS && op != SPHP_OP_IPRODUCT_WRT_BASE && op != SPHP_OP_PHYS_DERIV &&
        !(op == SPHP_OP_IPRODUCT_WRT_DERIV_BASE && strategy == SPHP_STRATEGY_CUDA_STDMAT))
      return fail(SPHP_ERR_UNSUPPORTED,
                  "triangle collections: BwdTrans, IProductWRTBase, PhysDeriv (sumfac or stdmat), "
                  "IProductWRTDerivBase (stdmat)");
    if (strategy == SPHP_STRATEGY_CUDA_SUMFAC) {
      int rc = tri_tables_device(t);
      if (rc) return rc;
    }
  } else if (strategy == SPHP_STRATEGY_CUDA_SUMFAC && !t->fast)
    return fail(SPHP_ERR_UNSUPPORTED,
                "sumfac kernels cover Modified_A/GLL with Q = P+2 or P+3 (hex P <= 8, quad P <= 9); "
                "use the stdmat strategy for this key");
  int rc = ensure_tables_uploaded();
  if (rc) return rc;
  rc = tables_device(t);
  if (rc) return rc;
  auto* c = new sphp_coll();
  c->t = t;
  c->op = op;
  c->strategy = strategy;
  c->E = E;
  c->geom_kind = geom_kind;
  c->geom = geom;
  c->gstride = geom_record(t, geom_kind);
  c->cs = (t->np + 1) & ~1LL;
  c->lam = lambda;
  const int d = t->dim;
  switch (op) {
    case SPHP_OP_BWD_TRANS: c->in_size = t->nm; c->out_size = t->np; break;
    case SPHP_OP_IPRODUCT_WRT_BASE: c->in_size = t->np; c->out_size = t->nm; break;
    case SPHP_OP_PHYS_DERIV: c->in_size = t->np; c->out_size = d * t->np; break;
    case SPHP_OP_IPRODUCT_WRT_DERIV_BASE: c->in_size = d * t->np; c->out_size = t->nm; break;
    case SPHP_OP_HELMHOLTZ: c->in_size = t->nm; c->out_size = t->nm; break;
  }
  if (strategy == SPHP_STRATEGY_CUDA_STDMAT) {
    rc = stdmat_prepare(c);
    if (rc) {
      delete c;
      return rc;
    }
  }
  *out = c;
  return SPHP_OK;
}

int sphp_collection_destroy(sphp_coll* c) {
  delete c;
  return SPHP_OK;
}

// the one mutation a handle allows (collections.py: lam is a constructor
// argument there); not concurrent with applies of the handle
int sphp_collection_set_lambda(sphp_coll* c, double lambda) {
  if (!c) return fail(SPHP_ERR_BAD_ARG, "null collection");
  const bool rebuild = c->strategy == SPHP_STRATEGY_CUDA_STDMAT && c->op == SPHP_OP_HELMHOLTZ && lambda != c->lam;
  c->lam = lambda;
  if (rebuild) return stdmat_prepare(c);  // dense H_e depends on lambda
  return SPHP_OK;
}

int sphp_collection_info(const sphp_coll* c, int64_t* in_size, int64_t* out_size, int64_t* macs,
                         int64_t* bytes) {
  if (!c) return fail(SPHP_ERR_BAD_ARG, "null collection");
  if (in_size) *in_size = c->in_size;
  if (out_size) *out_size = c->out_size;
  if (macs) *macs = mac_count(c);
  if (bytes) *bytes = hbm_bytes(c);
  return SPHP_OK;
}

// collections.Collection.apply (collections.py:189-246)
int sphp_apply(sphp_coll* c, int64_t E, int64_t n_in, const double* in, double* out, sphp_stream stream) {
  NvtxRange nvtx_range("sphp_apply");
  if (!c) return fail(SPHP_ERR_BAD_ARG, "null collection");
  if (E != c->E || n_in != c->in_size) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "block shape (%lld, %lld) does not match (%lld, %lld)", (long long)E,
                  (long long)n_in, (long long)c->E, (long long)c->in_size);
    return fail(SPHP_ERR_BAD_SHAPE, buf);
  }
  if (!in || !out) return fail(SPHP_ERR_BAD_ARG, "null buffer");
  cudaStream_t s = (cudaStream_t)stream;
  if (c->strategy == SPHP_STRATEGY_CUDA_STDMAT) return stdmat_apply(c, in, out, s);
  OpArgs a = base_args(c);
  a.in = in;
  a.out = out;
  cudaError_t e = sumfac_launch(c, a, s);
  if (e == cudaErrorNotSupported) return fail(SPHP_ERR_UNSUPPORTED, "no sum-factorisation kernel for this key");
  if (e != cudaSuccess) return cuda_fail(e, "sphp_apply");
  return SPHP_OK;
}

int sphp_apply_host(sphp_coll* c, int64_t E, int64_t n_in, const double* in, double* out,
                    sphp_stream stream) {
  NvtxRange nvtx_range("sphp_apply_host");
  if (!c) return fail(SPHP_ERR_BAD_ARG, "null collection");
  if (E != c->E || n_in != c->in_size) return sphp_apply(c, E, n_in, in, out, stream);
  cudaStream_t s = (cudaStream_t)stream;
  Workspace* w = c->ws.get(s);
  const size_t bi = sizeof(double) * c->E * c->in_size, bo = sizeof(double) * c->E * c->out_size;
  CKW(w->host_in.ensure_on(bi, s));
  CKW(w->host_out.ensure_on(bo, s));
  CK(cudaMemcpyAsync(w->host_in.p, in, bi, cudaMemcpyHostToDevice, s));
  int rc = sphp_apply(c, E, n_in, w->host_in.as<double>(), w->host_out.as<double>(), stream);
  if (rc) return rc;
  CK(cudaMemcpyAsync(out, w->host_out.p, bo, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return SPHP_OK;
}

static int amap_device(const sphp_amap* ac);

// Allocate the per-stream workspace a later apply on `stream` would size on
// first use (so that apply can be captured into a CUDA graph): device
// applies (StdMat scratch; with a map, the local blocks / class block and
// the schedule counters of the assembled apply) and, with
// SPHP_RESERVE_HOST, the host-buffer staging and copy pipeline.
int sphp_collection_reserve(sphp_coll* c, const sphp_amap* a, int flags, sphp_stream stream) {
  if (!c) return fail(SPHP_ERR_BAD_ARG, "null collection");
  cudaStream_t s = (cudaStream_t)stream;
  Workspace* w = c->ws.get(s);
  const int64_t E = c->E, nm = c->t->nm, np = c->t->np, d = c->t->dim;
  if (flags & SPHP_RESERVE_DEVICE) {
    if (c->strategy == SPHP_STRATEGY_CUDA_STDMAT) CKW(w->scratch.ensure_on(sizeof(double) * E * d * np, s));
    if (a) {
      CKW(w->loc_x.ensure_on(sizeof(double) * E * nm, s));
      CKW(w->loc_y.ensure_on(sizeof(double) * E * nm, s));
      CKW(w->ctr.ensure_on(2 * sizeof(int), s));
      if (int rc = amap_device(a)) return rc;
    }
  }
  if (flags & SPHP_RESERVE_HOST) {
    int64_t hb = std::max(E * c->in_size, E * c->out_size);
    if (a) hb = std::max<int64_t>(hb, a->num_global);
    CKW(w->host_in.ensure_on(sizeof(double) * hb, s));
    CKW(w->host_out.ensure_on(sizeof(double) * hb, s));
    if (a) {
      CKW(w->loc_x.ensure_on(sizeof(double) * E * nm, s));
      CKW(w->loc_y.ensure_on(sizeof(double) * E * nm, s));
      CKW(w->ctr.ensure_on(2 * sizeof(int), s));
      if (!w->pipe_h2d) {
        CK(cudaStreamCreateWithFlags(&w->pipe_h2d, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&w->pipe_d2h, cudaStreamNonBlocking));
      }
    }
  }
  return SPHP_OK;
}

// ---- assembly ---------------------------------------------------------------
static int amap_colour_and_upload(sphp_amap* a) {
  // greedy colouring in element order: elements sharing a global dof get
  // distinct colours (deterministic)
  std::vector<uint64_t> mask(a->num_global, 0);
  std::vector<int> col(a->E, 0);
  int ncol = 0;
  for (int64_t e = 0; e < a->E; ++e) {
    uint64_t used = 0;
    for (int k = 0; k < a->nm; ++k) {
      int64_t c = a->codes_host[e * a->nm + k];
      int64_t g = c >= 0 ? c : (c == -1 ? -1 : -c - 2);
      if (g >= 0) used |= mask[g];
    }
    int cc = 0;
    while (cc < 64 && (used >> cc) & 1) ++cc;
    if (cc == 64) return fail(SPHP_ERR_UNSUPPORTED, "element graph needs more than 64 colours");
    col[e] = cc;
    ncol = std::max(ncol, cc + 1);
    for (int k = 0; k < a->nm; ++k) {
      int64_t c = a->codes_host[e * a->nm + k];
      int64_t g = c >= 0 ? c : (c == -1 ? -1 : -c - 2);
      if (g >= 0) mask[g] |= (1ull << cc);
    }
  }
  a->ncolours = ncol;
  a->colour_off.assign(ncol + 1, 0);
  for (int64_t e = 0; e < a->E; ++e) a->colour_off[col[e] + 1]++;
  for (int c = 0; c < ncol; ++c) a->colour_off[c + 1] += a->colour_off[c];
  std::vector<int> elist(a->E);
  std::vector<int64_t> fill(a->colour_off.begin(), a->colour_off.end() - 1);
  for (int64_t e = 0; e < a->E; ++e) elist[fill[col[e]]++] = (int)e;
  a->elist_host = std::move(elist);
  return SPHP_OK;
}

// device tables of a map, built when the map is created (explicit maps:
// codes, colour lists, CSR) or switched to the owner algorithm (periodic
// maps: the (E, 27) entity table only the gathering owner path reads);
// applies find them built and never allocate.  (Without a visible device,
// e.g. host-only map construction, the build waits for the first device
// call.)
static bool device_present() {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
}
static int amap_device(const sphp_amap* ac) {
  sphp_amap* a = const_cast<sphp_amap*>(ac);
  if (a->periodic) {
    if (a->alg != SPHP_ASSEMBLY_OWNER) return SPHP_OK;
    std::lock_guard<std::mutex> lk(a->mu);
    if (a->d_entity.p) return SPHP_OK;
    DevBuf tmp;
    CK(tmp.ensure(sizeof(int) * a->E * 27));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaError_t e = periodic_entity_table(a->n, a->P, tmp.as<int>(), s);
    const cudaError_t e2 = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    CK(e);
    CK(e2);
    std::swap(a->d_entity.p, tmp.p);
    std::swap(a->d_entity.bytes, tmp.bytes);
    return SPHP_OK;
  }
  if (a->d_codes.p) return SPHP_OK;
  std::lock_guard<std::mutex> lk(a->mu);
  if (a->d_codes.p) return SPHP_OK;
  std::vector<int> codes32(a->codes_host.size());
  for (size_t i = 0; i < codes32.size(); ++i) codes32[i] = (int)a->codes_host[i];
  CK(a->d_elist.ensure(sizeof(int) * a->elist_host.size()));
  CK(cudaMemcpy(a->d_elist.p, a->elist_host.data(), sizeof(int) * a->elist_host.size(),
                cudaMemcpyHostToDevice));
  // owner-computes CSR: per global dof, its local entries in element order
  std::vector<int64_t> rowp(a->num_global + 1, 0);
  for (int64_t c : a->codes_host)
    if (c != -1) rowp[(c >= 0 ? c : -c - 2) + 1]++;
  for (int64_t g = 0; g < a->num_global; ++g) rowp[g + 1] += rowp[g];
  std::vector<int> ent(rowp[a->num_global]);
  std::vector<int64_t> fill(rowp.begin(), rowp.end() - 1);
  for (int64_t i = 0; i < (int64_t)a->codes_host.size(); ++i) {
    const int64_t c = a->codes_host[i];
    if (c == -1) continue;
    const int64_t g = c >= 0 ? c : -c - 2;
    ent[fill[g]++] = c >= 0 ? (int)i : -(int)i - 1;
  }
  CK(a->d_rowp.ensure(sizeof(int64_t) * rowp.size()));
  CK(cudaMemcpy(a->d_rowp.p, rowp.data(), sizeof(int64_t) * rowp.size(), cudaMemcpyHostToDevice));
  CK(a->d_ent.ensure(sizeof(int) * (ent.size() + 1)));
  if (!ent.empty())
    CK(cudaMemcpy(a->d_ent.p, ent.data(), sizeof(int) * ent.size(), cudaMemcpyHostToDevice));
  DevBuf tmp;
  CK(tmp.ensure(sizeof(int) * codes32.size()));
  CK(cudaMemcpy(tmp.p, codes32.data(), sizeof(int) * codes32.size(), cudaMemcpyHostToDevice));
  std::swap(a->d_codes.p, tmp.p);
  std::swap(a->d_codes.bytes, tmp.bytes);
  return SPHP_OK;
}

// local (E, nm) -> global with the map's algorithm; accumulate adds to g
static int amap_assemble_any(const sphp_amap* a, const double* loc, double* g, int accumulate,
                             cudaStream_t s, int mode_major = 0, int* ctr = nullptr) {
  if (a->alg == SPHP_ASSEMBLY_OWNER || a->alg == SPHP_ASSEMBLY_SPLIT || a->alg == SPHP_ASSEMBLY_CLASS) {
    if (a->periodic) {
      CK(owner_assemble_periodic(a->n, a->P, loc, g, accumulate, mode_major, s, ctr));
    } else {
      CK(owner_assemble_csr(a->num_global, a->d_rowp.as<int64_t>(), a->d_ent.as<int>(), loc, g,
                            accumulate, a->nm, a->E, mode_major, s));
    }
    return SPHP_OK;
  }
  CK(amap_assemble(a->dev(), loc, g, a->ncolours, a->d_elist.as<int>(), a->colour_off.data(),
                   accumulate, s));
  return SPHP_OK;
}

int sphp_amap_create_explicit(int64_t E, int nmodes, const int64_t* codes, int64_t num_global,
                              sphp_amap** out) {
  if (!out || !codes || E < 1 || nmodes < 1 || num_global < 0) return fail(SPHP_ERR_BAD_ARG, "bad map arguments");
  if (num_global > 2147483645LL) return fail(SPHP_ERR_UNSUPPORTED, "more than 2^31-3 global dofs");
  for (int64_t i = 0; i < E * nmodes; ++i) {
    int64_t c = codes[i];
    int64_t g = c >= 0 ? c : (c == -1 ? -1 : -c - 2);
    if (g >= num_global) return fail(SPHP_ERR_BAD_ARG, "map code outside [0, num_global)");
  }
  auto* a = new sphp_amap();
  a->nm = nmodes;
  a->E = E;
  a->num_global = num_global;
  a->codes_host.assign(codes, codes + E * nmodes);
  int rc = amap_colour_and_upload(a);
  if (!rc && device_present()) rc = amap_device(a);
  if (rc) {
    delete a;
    return rc;
  }
  *out = a;
  return SPHP_OK;
}

int sphp_amap_create_hex_periodic(int n, int P, sphp_amap** out) {
  if (!out || n < 1 || P < 1) return fail(SPHP_ERR_BAD_ARG, "bad periodic map arguments");
  if (n % 2) return fail(SPHP_ERR_UNSUPPORTED, "parity colouring of a periodic grid needs even n");
  auto* a = new sphp_amap();
  a->periodic = 1;
  a->n = n;
  a->P = P;
  a->nm = (P + 1) * (P + 1) * (P + 1);
  a->E = (int64_t)n * n * n;
  a->num_global = ipow((int64_t)n * P, 3);
  a->ncolours = 8;
  // default: class-range assembly (the operator gathers x by entity class,
  // one streaming owner sum; falls back to split when the mesh does not
  // divide into its tiles or x is misaligned): 4-19 % faster than split at
  // every order P = 2..8 (tools/time_phases.py, n = 64)
  a->alg = P < 2 ? SPHP_ASSEMBLY_OWNER : SPHP_ASSEMBLY_CLASS;
  if (a->num_global > 2147483645LL) {
    delete a;
    return fail(SPHP_ERR_UNSUPPORTED, "periodic map with more than 2^31-3 global dofs");
  }
  if (int rc = device_present() ? amap_device(a) : SPHP_OK) {
    delete a;
    return rc;
  }
  *out = a;
  return SPHP_OK;
}

// numbering of oracle/assembly.py hex_periodic + build_map, variable order
int sphp_hexmap_variable(int n, const int* orders, int64_t* num_global, int64_t* offsets, int64_t* codes) {
  if (n < 1 || !orders || !num_global) return fail(SPHP_ERR_BAD_ARG, "bad arguments");
  const int64_t N3 = (int64_t)n * n * n;
  auto vid = [n](int i, int j, int k) -> int64_t {
    i %= n;
    j %= n;
    k %= n;
    return i + (int64_t)n * (j + (int64_t)n * k);
  };
  for (int64_t e = 0; e < N3; ++e)
    if (orders[e] < 1) return fail(SPHP_ERR_BAD_ARG, "orders must be >= 1");
  std::vector<int> eord(3 * N3, 1 << 30), ford(3 * N3, 1 << 30);
  for (int ez = 0; ez < n; ++ez)
    for (int ey = 0; ey < n; ++ey)
      for (int ex = 0; ex < n; ++ex) {
        const int P = orders[ex + (int64_t)n * (ey + (int64_t)n * ez)];
        const int b[3] = {ex, ey, ez};
        for (int d = 0; d < 3; ++d) {
          for (int s = 0; s < 2; ++s)
            for (int t2 = 0; t2 < 2; ++t2) {
              int o[3];
              int oo[2] = {s, t2}, c = 0;
              for (int a = 0; a < 3; ++a) o[a] = (a == d) ? 0 : oo[c++];
              int64_t eid = d * N3 + vid(b[0] + o[0], b[1] + o[1], b[2] + o[2]);
              eord[eid] = std::min(eord[eid], P);
            }
          for (int side = 0; side < 2; ++side) {
            int o[3] = {0, 0, 0};
            o[d] = side;
            int64_t fid = d * N3 + vid(b[0] + o[0], b[1] + o[1], b[2] + o[2]);
            ford[fid] = std::min(ford[fid], P);
          }
        }
      }
  std::vector<int64_t> eoff(3 * N3 + 1, 0), foff(3 * N3 + 1, 0);
  for (int64_t i = 0; i < 3 * N3; ++i) {
    eoff[i + 1] = eoff[i] + std::max(0, eord[i] - 1);
    foff[i + 1] = foff[i] + (int64_t)std::max(0, ford[i] - 1) * std::max(0, ford[i] - 1);
  }
  const int64_t ebase = N3, fbase = N3 + eoff[3 * N3], ibase = fbase + foff[3 * N3];
  int64_t gid = ibase;
  int64_t off = 0;
  for (int ez = 0; ez < n; ++ez)
    for (int ey = 0; ey < n; ++ey)
      for (int ex = 0; ex < n; ++ex) {
        const int64_t e = ex + (int64_t)n * (ey + (int64_t)n * ez);
        const int P = orders[e], m = P + 1;
        const int b[3] = {ex, ey, ez};
        if (offsets) offsets[e] = off;
        for (int p = 0; p < m; ++p)
          for (int q = 0; q < m; ++q)
            for (int r = 0; r < m; ++r) {
              const int idx[3] = {p, q, r};
              const int nb = (p >= 2) + (q >= 2) + (r >= 2);
              int64_t g = -1;
              if (nb == 0) {
                g = vid(ex + p, ey + q, ez + r);
              } else if (nb == 1) {
                const int d = (p >= 2) ? 0 : ((q >= 2) ? 1 : 2);
                int c[3];
                for (int a = 0; a < 3; ++a) c[a] = b[a] + (a == d ? 0 : idx[a]);
                const int64_t eid = d * N3 + vid(c[0], c[1], c[2]);
                if (idx[d] <= eord[eid]) g = ebase + eoff[eid] + (idx[d] - 2);
              } else if (nb == 2) {
                const int d = (p < 2) ? 0 : ((q < 2) ? 1 : 2);
                int c[3];
                for (int a = 0; a < 3; ++a) c[a] = b[a] + (a == d ? idx[a] : 0);
                const int64_t fid = d * N3 + vid(c[0], c[1], c[2]);
                const int k1 = (d == 0) ? q : p, k2 = (d == 2) ? q : r;
                const int pf = ford[fid];
                if (k1 <= pf && k2 <= pf) g = fbase + foff[fid] + (int64_t)(k1 - 2) * (pf - 1) + (k2 - 2);
              } else {
                g = -2;  // interior: numbered below in local order
              }
              if (g == -2) g = gid++;
              if (codes) codes[off] = g;  // signs are all +1 on the structured grid
              ++off;
            }
      }
  if (offsets) offsets[N3] = off;
  *num_global = gid;
  return SPHP_OK;
}

// rows [e0, e1) of the periodic structured hex map (the analytic numbering
// of sphp_amap_create_hex_periodic, = sphp_hexmap_variable at uniform
// order): per-slab maps for the sharded operator without the n^3 table
int sphp_hexmap_periodic_codes(int n, int P, int64_t e0, int64_t e1, int64_t* codes) {
  if (n < 1 || P < 1 || e0 < 0 || e1 < e0 || e1 > (int64_t)n * n * n || !codes)
    return fail(SPHP_ERR_BAD_ARG, "bad arguments");
  if (ipow((int64_t)n * P, 3) > 2147483645LL) return fail(SPHP_ERR_UNSUPPORTED, "more than 2^31-3 global dofs");
  const int M = P + 1, nm = M * M * M;
  std::vector<int> mc(nm);
  for (int i = 0; i < nm; ++i) mc[i] = mode_code(M, i);
  for (int64_t e = e0; e < e1; ++e) {
    const int ex = (int)(e % n), ey = (int)((e / n) % n), ez = (int)(e / ((int64_t)n * n));
    int base[27];
    for (int k = 0; k < 27; ++k) base[k] = entity_base(n, P, ex, ey, ez, k);
    int64_t* row = codes + (e - e0) * nm;
    for (int i = 0; i < nm; ++i) row[i] = base[mc[i] & 31] + (mc[i] >> 5);
  }
  return SPHP_OK;
}

// the sharded operator's interface exchange: dst[i] = src[idx[i]] (pack),
// y[idx[i]] = lo[i] + hi[i] (combine the two copies in rank order)
int sphp_index_gather(int64_t n, const int64_t* idx, const double* src, double* dst, sphp_stream stream) {
  if (n < 0 || (n > 0 && (!idx || !src || !dst))) return fail(SPHP_ERR_BAD_ARG, "bad arguments");
  CK(index_gather(n, idx, src, dst, (cudaStream_t)stream));
  return SPHP_OK;
}
int sphp_index_sum2(int64_t n, const int64_t* idx, const double* lo, const double* hi, double* y,
                    sphp_stream stream) {
  if (n < 0 || (n > 0 && (!idx || !lo || !hi || !y))) return fail(SPHP_ERR_BAD_ARG, "bad arguments");
  CK(index_sum2(n, idx, lo, hi, y, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_amap_set_algorithm(sphp_amap* a, int alg) {
  if (!a) return fail(SPHP_ERR_BAD_ARG, "null map");
  if (alg != SPHP_ASSEMBLY_OWNER && alg != SPHP_ASSEMBLY_COLOUR && alg != SPHP_ASSEMBLY_SPLIT &&
      alg != SPHP_ASSEMBLY_CLASS)
    return fail(SPHP_ERR_BAD_ARG, "unknown assembly algorithm");
  if (alg == SPHP_ASSEMBLY_CLASS && !a->periodic)
    return fail(SPHP_ERR_UNSUPPORTED, "class-range assembly needs a periodic map");
  a->alg = alg;
  return device_present() ? amap_device(a) : SPHP_OK;  // the owner path's entity table (periodic maps)
}

int sphp_amap_algorithm(const sphp_amap* a, int* alg) {
  if (!a || !alg) return fail(SPHP_ERR_BAD_ARG, "null map / output");
  *alg = a->alg;
  return SPHP_OK;
}

int sphp_amap_destroy(sphp_amap* a) {
  delete a;
  return SPHP_OK;
}

int sphp_amap_info(const sphp_amap* a, int64_t* ne, int* nm, int64_t* ng, int* nc) {
  if (!a) return fail(SPHP_ERR_BAD_ARG, "null map");
  if (ne) *ne = a->E;
  if (nm) *nm = a->nm;
  if (ng) *ng = a->num_global;
  if (nc) *nc = a->ncolours;
  return SPHP_OK;
}

int sphp_amap_codes(const sphp_amap* a, int64_t* codes) {
  if (!a || !codes) return fail(SPHP_ERR_BAD_ARG, "null argument");
  if (!a->periodic) {
    std::memcpy(codes, a->codes_host.data(), sizeof(int64_t) * a->codes_host.size());
    return SPHP_OK;
  }
  std::vector<int> orders((size_t)a->E, a->P);
  int64_t ng;
  return sphp_hexmap_variable(a->n, orders.data(), &ng, nullptr, codes);
}

int sphp_scatter(const sphp_amap* a, const double* g, double* loc, sphp_stream stream) {
  NvtxRange nvtx_range("sphp_scatter");
  if (!a || !g || !loc) return fail(SPHP_ERR_BAD_ARG, "null argument");
  if (int rc = amap_device(a)) return rc;
  CK(amap_scatter(a->dev(), g, loc, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_assemble(const sphp_amap* a, const double* loc, double* g, sphp_stream stream) {
  NvtxRange nvtx_range("sphp_assemble");
  if (!a || !g || !loc) return fail(SPHP_ERR_BAD_ARG, "null argument");
  if (int rc = amap_device(a)) return rc;
  return amap_assemble_any(a, loc, g, 0, (cudaStream_t)stream);
}

// phase markers of sphp_helmholtz_assembled_phases: when set (this thread
// only), the assembled apply records one event on its stream after each of
// its launches
thread_local std::vector<cudaEvent_t>* g_phase_marks = nullptr;
thread_local size_t g_phase_next = 0;
static void phase_mark(cudaStream_t s) {
  if (g_phase_marks && g_phase_next < g_phase_marks->size()) cudaEventRecord((*g_phase_marks)[g_phase_next++], s);
}

static int split_reverse() {
  static const int v = [] {
    const char* e = getenv("SPHP_SPLIT_REVERSE");  // tuning override
    return e ? atoi(e) : 1;
  }();
  return v;
}

// assembly.GlobalSystem.apply (assembly.py:177-182), fused
int sphp_helmholtz_assembled(sphp_coll* c, const sphp_amap* a, const double* x, double* y, int accumulate,
                             sphp_stream stream) {
  NvtxRange nvtx_range("sphp_helmholtz_assembled");
  if (!c || !a || !x || !y) return fail(SPHP_ERR_BAD_ARG, "null argument");
  if (c->op != SPHP_OP_HELMHOLTZ) return fail(SPHP_ERR_BAD_ARG, "collection is not a Helmholtz operator");
  if (a->E != c->E || a->nm != c->t->nm)
    return fail(SPHP_ERR_BAD_SHAPE, "assembly map and collection disagree on (E, nmodes)");
  if (a->periodic && c->t->shape != SPHP_SHAPE_HEX)
    return fail(SPHP_ERR_BAD_ARG, "periodic analytic maps are hexahedral");
  if (int rc = amap_device(a)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  Workspace* w = c->ws.get(s);
  const size_t lb = sizeof(double) * c->E * c->t->nm;
  int* ctr = nullptr;
  if (a->periodic) {
    CKW(w->ctr.ensure_on(2 * sizeof(int), s));
    ctr = w->ctr.as<int>();
  }
  if (c->strategy == SPHP_STRATEGY_CUDA_STDMAT) {
    CKW(w->loc_x.ensure_on(lb, s));
    CKW(w->loc_y.ensure_on(lb, s));
    CK(amap_scatter(a->dev(), x, w->loc_x.as<double>(), s, ctr));
    CK(elem_matvec(c->E, (int)c->t->nm, c->helm_H.as<double>(), w->loc_x.as<double>(), w->loc_y.as<double>(), s));
    return amap_assemble_any(a, w->loc_y.as<double>(), y, accumulate, s, 0, ctr + 1);
  }
  OpArgs o = base_args(c);
  o.xg = x;
  o.yg = y;
  if (a->alg == SPHP_ASSEMBLY_CLASS && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    // the operator gathers x by entity-class ranges and writes a class-major
    // block (interiors straight into y), then one owner-computes sum over it
    // (two launches, the local block never exists)
    CKW(w->loc_y.ensure_on(sizeof(double) * class_block_doubles(a->n, a->P), s));
    o.mode = AsmMode::PERIODIC_CLASS;
    o.n = a->n;
    o.zbuf = w->loc_y.as<double>();
    o.direct_interior = accumulate ? 0 : 1;
    int ne = 0;
    o.ne_out = &ne;
    cudaError_t e = sumfac_launch(c, o, s);
    if (e == cudaSuccess) {
      phase_mark(s);
      CK(class_owner_sum(a->n, a->P, ne, o.zbuf, y, accumulate, !o.direct_interior, s));
      phase_mark(s);
      return SPHP_OK;
    }
    if (e != cudaErrorNotSupported) return cuda_fail(e, "sphp_helmholtz_assembled");
    // no class-mode tile for this key / mesh: the split algorithm below
  }
  // (x not 16-byte aligned: the class gather moves 16-byte chunks; split)
  if (a->alg == SPHP_ASSEMBLY_SPLIT || a->alg == SPHP_ASSEMBLY_CLASS) {
    // scatter -> fused local operator -> owner-computes sum (three launches;
    // the fused kernel then runs in its block-input form)
    CKW(w->loc_x.ensure_on(lb, s));
    CKW(w->loc_y.ensure_on(lb, s));
    CK(amap_scatter(a->dev(), x, w->loc_x.as<double>(), s, ctr));
    phase_mark(s);
    o.in = w->loc_x.as<double>();
    o.out = w->loc_y.as<double>();
    o.mode = AsmMode::LOCAL;
    // the operator walks the elements backwards: it starts on the block the
    // scatter wrote last and ends on the elements the owner sum reads first,
    // both still in L2
    o.reverse = split_reverse();
    cudaError_t e = sumfac_launch(c, o, s);
    if (e == cudaErrorNotSupported) return fail(SPHP_ERR_UNSUPPORTED, "no kernel for this key");
    if (e != cudaSuccess) return cuda_fail(e, "sphp_helmholtz_assembled");
    phase_mark(s);
    const int rc = amap_assemble_any(a, w->loc_y.as<double>(), y, accumulate, s, 0, ctr + 1);
    phase_mark(s);
    return rc;
  }
  if (a->alg == SPHP_ASSEMBLY_OWNER) {
    // gather -> fused elemental operator -> local block, then the
    // owner-computes sum (two launches, no colour passes)
    CKW(w->loc_y.ensure_on(lb, s));
    o.out = w->loc_y.as<double>();
    if (a->periodic) {
      o.mode = AsmMode::PERIODIC_GATHER;
      o.n = a->n;
      o.ent_g = a->d_entity.as<int>();
    } else {
      o.mode = AsmMode::EXPLICIT_GATHER;
      o.codes = a->d_codes.as<int>();
    }
    cudaError_t e = sumfac_launch(c, o, s);
    if (e == cudaErrorNotSupported) return fail(SPHP_ERR_UNSUPPORTED, "no assembled kernel for this key");
    if (e != cudaSuccess) return cuda_fail(e, "sphp_helmholtz_assembled");
    return amap_assemble_any(a, w->loc_y.as<double>(), y, accumulate, s, /*mode_major=*/0, ctr + 1);
  }
  if (!accumulate) CK(cudaMemsetAsync(y, 0, sizeof(double) * a->num_global, s));
  for (int col = 0; col < a->ncolours; ++col) {
    if (a->periodic) {
      o.mode = AsmMode::PERIODIC;
      o.n = a->n;
      o.colour = col;
      o.nlist = (int64_t)(a->n / 2) * (a->n / 2) * (a->n / 2);
    } else {
      o.mode = AsmMode::EXPLICIT;
      o.codes = a->d_codes.as<int>();
      o.elist = a->d_elist.as<int>() + a->colour_off[col];
      o.nlist = a->colour_off[col + 1] - a->colour_off[col];
    }
    cudaError_t e = sumfac_launch(c, o, s);
    if (e == cudaErrorNotSupported) return fail(SPHP_ERR_UNSUPPORTED, "no assembled kernel for this key");
    if (e != cudaSuccess) return cuda_fail(e, "sphp_helmholtz_assembled");
  }
  return SPHP_OK;
}

// One assembled apply (accumulate = 0) with an event after each of its
// launches; waits for it and returns the launches' durations in ms (split:
// scatter, operator, owner sum; class: operator, owner sum).  Measurement
// entry for bench.py: the dominant kernel's time on its own stream.
int sphp_helmholtz_assembled_phases(sphp_coll* c, const sphp_amap* a, const double* x, double* y,
                                    sphp_stream stream, int max_phases, float* ms, int* nphases) {
  NvtxRange nvtx_range("sphp_helmholtz_assembled_phases");
  if (!ms || !nphases || max_phases < 1) return fail(SPHP_ERR_BAD_ARG, "null output");
  static thread_local std::vector<cudaEvent_t> ev;
  while ((int)ev.size() < max_phases + 1) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ev.push_back(e);
  }
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<cudaEvent_t> marks(ev.begin() + 1, ev.begin() + 1 + max_phases);
  CK(cudaEventRecord(ev[0], s));
  g_phase_marks = &marks;
  g_phase_next = 0;
  const int rc = sphp_helmholtz_assembled(c, a, x, y, 0, stream);
  const size_t np = g_phase_next;
  g_phase_marks = nullptr;
  if (rc) return rc;
  CK(cudaStreamSynchronize(s));
  for (size_t i = 0; i < np; ++i) CK(cudaEventElapsedTime(&ms[i], i ? marks[i - 1] : ev[0], marks[i]));
  *nphases = (int)np;
  return SPHP_OK;
}

// Host-buffer apply on a periodic split map, pipelined over K z-slabs: the
// host->device copy of slab k+1 overlaps the scatter / fused operator /
// owner sum of slab k, and the device->host copy of finished slabs runs in
// the other PCIe direction at the same time.  Global dofs are numbered
// region by region (vertices, edges by direction, faces by direction,
// interiors), each region z-plane-major, so a slab is 8 contiguous ranges.
// Dependencies: scatter(k) reads x planes [z0, z1] (the next slab's first
// plane, cyclically); owner(k) reads the local block of planes z0-1 .. z1-1,
// so owner(0) runs after the last slab's operator.
int assembled_host_pipelined(sphp_coll* c, const sphp_amap* a, const double* x, double* y,
                             cudaStream_t s, const std::vector<int>& zb, bool use_class) {
  const int n = a->n, P = a->P, b = P - 1, K = (int)zb.size() - 1;
  const int64_t N3 = (int64_t)n * n * n, n2 = (int64_t)n * n, nm = c->t->nm;
  // region r: base and dofs per z-plane; regions 1-3 (edges) and 4-6
  // (faces) have equal sizes, so a slab's three pieces of each are one
  // strided (2D) copy
  int64_t base[8], per[8];
  const int64_t sz[8] = {1, b, b, b, (int64_t)b * b, (int64_t)b * b, (int64_t)b * b, (int64_t)b * b * b};
  int64_t acc = 0;
  for (int r = 0; r < 8; ++r) {
    base[r] = acc;
    per[r] = n2 * sz[r];
    acc += N3 * sz[r];
  }
  if (acc != a->num_global) return fail(SPHP_ERR_UNSUPPORTED, "unexpected periodic numbering");
  const size_t bytes = sizeof(double) * a->num_global;
  Workspace* w = c->ws.get(s);
  CKW(w->host_in.ensure_on(bytes, s));
  CKW(w->host_out.ensure_on(bytes, s));
  CKW(w->loc_x.ensure_on(sizeof(double) * c->E * nm, s));
  CKW(w->loc_y.ensure_on(sizeof(double) * c->E * nm, s));
  CKW(w->ctr.ensure_on(2 * sizeof(int), s));
  if (!w->pipe_h2d) {
    CK(cudaStreamCreateWithFlags(&w->pipe_h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&w->pipe_d2h, cudaStreamNonBlocking));
  }
  while ((int)w->pipe_ev.size() < 2 * K + 2) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    w->pipe_ev.push_back(e);
  }
  int* ctr = w->ctr.as<int>();
  cudaEvent_t* ev_in = w->pipe_ev.data();
  cudaEvent_t* ev_out = ev_in + K;
  cudaEvent_t ev_start = ev_in[2 * K], ev_done = ev_in[2 * K + 1];
  double* dx = w->host_in.as<double>();
  double* dy = w->host_out.as<double>();
  double* lx = w->loc_x.as<double>();
  double* ly = w->loc_y.as<double>();
  // copy planes [z0, z1) of every region between host and device
  auto slab_copy = [&](double* dst, const double* src, int z0, int z1, cudaMemcpyKind kind,
                       cudaStream_t st) -> cudaError_t {
    const int nz = z1 - z0;
    for (int r : {0, 1, 4, 7}) {
      const int64_t o = base[r] + (int64_t)z0 * per[r];
      const size_t w = sizeof(double) * nz * per[r];
      cudaError_t e;
      if (r == 1 || r == 4)  // three equal regions, N3 * size apart
        e = cudaMemcpy2DAsync(dst + o, sizeof(double) * N3 * sz[r], src + o, sizeof(double) * N3 * sz[r],
                              w, 3, kind, st);
      else
        e = cudaMemcpyAsync(dst + o, src + o, w, kind, st);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  };
  // copies start after everything already queued on the caller's stream
  CK(cudaEventRecord(ev_start, s));
  CK(cudaStreamWaitEvent(w->pipe_h2d, ev_start, 0));
  CK(cudaStreamWaitEvent(w->pipe_d2h, ev_start, 0));
  for (int k = 0; k < K; ++k) {
    CK(slab_copy(dx, x, zb[k], zb[k + 1], cudaMemcpyHostToDevice, w->pipe_h2d));
    CK(cudaEventRecord(ev_in[k], w->pipe_h2d));
  }
  OpArgs o = base_args(c);
  o.mode = AsmMode::LOCAL;
  // class-range algorithm: the operator reads x and writes Z + y interiors
  // slab by slab, the class owner sum takes the place of owner_periodic_v3
  int ne = 0;
  if (use_class) {
    o.mode = AsmMode::PERIODIC_CLASS;
    o.n = n;
    o.xg = dx;
    o.yg = dy;
    o.zbuf = ly;
    o.direct_interior = 1;
    o.ne_out = &ne;
  }
  // (writing a pinned y directly from the owner sum over PCIe instead of
  // copying it measured slower: 4.8 ms vs 4.0 ms per apply at P=4, n=64)
  auto owner = [&](int k) -> int {
    if (use_class)
      CK(class_owner_sum(n, P, ne, ly, dy, 0, 0, s, zb[k] * n, zb[k + 1] * n));
    else
      CK(owner_periodic_v3(n, P, ly, dy, 0, s, zb[k] * n, zb[k + 1] * n, ctr + 1));
    CK(cudaEventRecord(ev_out[k], s));
    return SPHP_OK;
  };
  for (int k = 0; k < K; ++k) {
    CK(cudaStreamWaitEvent(s, ev_in[k], 0));
    CK(cudaStreamWaitEvent(s, ev_in[(k + 1) % K], 0));
    const int64_t e0 = (int64_t)zb[k] * n2;
    o.E = (int64_t)(zb[k + 1] - zb[k]) * n2;
    if (use_class) {
      o.e0 = e0;  // absolute element indexing; x, Z, y and geometry are whole-mesh
    } else {
      CK(periodic_scatter_v2(n, P, dx, lx, s, zb[k] * n, zb[k + 1] * n, ctr));
      o.in = lx + e0 * nm;
      o.out = ly + e0 * nm;
      o.geom = c->geom + e0 * c->gstride;
    }
    cudaError_t e = sumfac_launch(c, o, s);
    if (e == cudaErrorNotSupported && use_class && k == 0) return SPHP_ERR_UNSUPPORTED;  // caller: split
    if (e == cudaErrorNotSupported) return fail(SPHP_ERR_UNSUPPORTED, "no kernel for this key");
    if (e != cudaSuccess) return cuda_fail(e, "sphp_helmholtz_assembled_host");
    if (k > 0) {
      if (int rc = owner(k)) return rc;
    }
  }
  if (int rc = owner(0)) return rc;
  for (int i = 1; i <= K; ++i) {
    const int k = i % K;
    CK(cudaStreamWaitEvent(w->pipe_d2h, ev_out[k], 0));
    CK(slab_copy(y, dy, zb[k], zb[k + 1], cudaMemcpyDeviceToHost, w->pipe_d2h));
  }
  CK(cudaEventRecord(ev_done, w->pipe_d2h));
  CK(cudaStreamWaitEvent(s, ev_done, 0));
  CK(cudaStreamSynchronize(s));
  return SPHP_OK;
}

// z-slab boundaries of the host pipeline: small slabs at both ends (the
// first compute waits for two slabs of x, the last slabs' results leave
// after the final compute) and `mid`-plane slabs in between; SPHP_HOST_SLABS
// = plane count of the middle slabs (0: no pipeline)
std::vector<int> host_slabs(int n) {
  static const int mid = [] {
    const char* v = getenv("SPHP_HOST_SLABS");
    return v && *v ? atoi(v) : 8;
  }();
  // tuning override: explicit slab plane counts "1,1,2,8,..." summing to n
  static const std::vector<int> list = [] {
    std::vector<int> l;
    const char* v = getenv("SPHP_HOST_SLAB_LIST");
    while (v && *v) {
      l.push_back(atoi(v));
      v = strchr(v, ',');
      if (v) ++v;
    }
    return l;
  }();
  if (!list.empty()) {
    std::vector<int> zb{0};
    for (int c : list) zb.push_back(zb.back() + c);
    if (zb.back() == n) return zb;
  }
  std::vector<int> zb{0};
  if (mid <= 0 || n < 8) return zb;
  const int head[] = {1, 1, 2}, tail[] = {2, 1, 1};
  int body = n - 8;
  for (int h : head) zb.push_back(zb.back() + h);
  while (body > 0) {
    const int step = body < mid ? body : mid;
    zb.push_back(zb.back() + step);
    body -= step;
  }
  for (int t : tail) zb.push_back(zb.back() + t);
  return zb;
}

// ---------------------------------------------------------------------------
// Global system over several per-order batches that share one numbering
// (GlobalSystem with per-order element groups, assembly.py:185-215; the
// variable-order configuration).  Per batch: scatter x into the batch's
// slice of one concatenated local block, the fused operator on that slice
// (block in / block out, the tuned local tile shapes); then ONE
// owner-computes pass over the global dofs whose CSR entries index the
// concatenated output block, in (batch, element, mode) order — instead of
// one gathering launch plus one full-length owner pass per batch.
// ---------------------------------------------------------------------------
struct sphp_gsys {
  std::vector<sphp_coll*> colls;
  std::vector<const sphp_amap*> maps;
  std::vector<int64_t> off;  // batch slice offsets (doubles, 16-byte aligned)
  int64_t num_global = 0, total = 0;
  DevBuf rowp, ent;  // the owner-computes CSR (immutable after create)
  // per caller stream: the concatenated local blocks, one stream per batch
  // (the batches' scatter + operator launches overlap: each batch alone
  // leaves the GPU half idle in its ramp and tail) and the events
  // [0] start, [1 + b] batch b done
  WorkspacePool ws;
};

// a gsys workspace for stream s: local blocks, batch streams, events
static int gsys_workspace(sphp_gsys* g, cudaStream_t s, Workspace** out) {
  Workspace* w = g->ws.get(s);
  CKW(w->loc_x.ensure_on(sizeof(double) * (g->total + 2), s));
  CKW(w->loc_y.ensure_on(sizeof(double) * (g->total + 2), s));
  const size_t nb = g->colls.size();
  if (w->bs.size() < nb || w->bev.size() < nb + 1) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (s) cudaStreamIsCapturing(s, &cap);
    if (cap != cudaStreamCaptureStatusNone) return ws_fail(cudaErrorStreamCaptureUnsupported, "sphp_gsys_apply");
  }
  while (w->bs.size() < nb) {
    cudaStream_t q;
    CK(cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking));
    w->bs.push_back(q);
  }
  while (w->bev.size() < nb + 1) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    w->bev.push_back(e);
  }
  *out = w;
  return SPHP_OK;
}

int sphp_gsys_create(sphp_coll* const* colls, const sphp_amap* const* maps, int nbatch, int64_t num_global,
                     sphp_gsys** out) {
  if (!out || !colls || !maps || nbatch < 1 || num_global < 0) return fail(SPHP_ERR_BAD_ARG, "bad arguments");
  if (num_global > 2147483645LL) return fail(SPHP_ERR_UNSUPPORTED, "more than 2^31-3 global dofs");
  auto g = std::make_unique<sphp_gsys>();
  g->num_global = num_global;
  int64_t acc = 0;
  for (int b = 0; b < nbatch; ++b) {
    sphp_coll* c = colls[b];
    const sphp_amap* a = maps[b];
    if (!c || !a) return fail(SPHP_ERR_BAD_ARG, "null batch");
    if (c->op != SPHP_OP_HELMHOLTZ) return fail(SPHP_ERR_BAD_ARG, "collection is not a Helmholtz operator");
    if (a->periodic) return fail(SPHP_ERR_UNSUPPORTED, "gsys batches take explicit maps");
    if (a->E != c->E || a->nm != c->t->nm)
      return fail(SPHP_ERR_BAD_SHAPE, "assembly map and collection disagree on (E, nmodes)");
    if (a->num_global != num_global) return fail(SPHP_ERR_BAD_ARG, "batches disagree on num_global");
    g->colls.push_back(c);
    g->maps.push_back(a);
    g->off.push_back(acc);
    acc += (c->E * c->t->nm + 1) & ~(int64_t)1;
  }
  g->total = acc;
  if (acc > 2147483647LL) return fail(SPHP_ERR_UNSUPPORTED, "more than 2^31-1 local entries");
  // CSR over the global dofs: entries in (batch, element, mode) order
  std::vector<int> rowp(num_global + 1, 0);
  for (int b = 0; b < nbatch; ++b)
    for (int64_t c : g->maps[b]->codes_host)
      if (c != -1) rowp[(c >= 0 ? c : -c - 2) + 1]++;
  for (int64_t i = 0; i < num_global; ++i) rowp[i + 1] += rowp[i];
  std::vector<int> ent(rowp[num_global]);
  std::vector<int> fill(rowp.begin(), rowp.end() - 1);
  for (int b = 0; b < nbatch; ++b) {
    const auto& codes = g->maps[b]->codes_host;
    for (int64_t i = 0; i < (int64_t)codes.size(); ++i) {
      const int64_t c = codes[i];
      if (c == -1) continue;
      const int64_t gid = c >= 0 ? c : -c - 2;
      const int64_t idx = g->off[b] + i;
      ent[fill[gid]++] = c >= 0 ? (int)idx : -(int)idx - 1;
    }
  }
  for (int b = 0; b < nbatch; ++b)
    if (int rc = amap_device(g->maps[b])) return rc;
  CK(g->rowp.ensure(sizeof(int) * rowp.size()));
  CK(cudaMemcpy(g->rowp.p, rowp.data(), sizeof(int) * rowp.size(), cudaMemcpyHostToDevice));
  CK(g->ent.ensure(sizeof(int) * (ent.size() + 1)));
  if (!ent.empty()) CK(cudaMemcpy(g->ent.p, ent.data(), sizeof(int) * ent.size(), cudaMemcpyHostToDevice));
  *out = g.release();
  return SPHP_OK;
}

int sphp_gsys_apply(sphp_gsys* g, const double* x, double* y, sphp_stream stream) {
  NvtxRange nvtx_range("sphp_gsys_apply");
  if (!g || !x || !y) return fail(SPHP_ERR_BAD_ARG, "null argument");
  cudaStream_t s0 = (cudaStream_t)stream;
  Workspace* w = nullptr;
  if (int rc = gsys_workspace(g, s0, &w)) return rc;
  CK(cudaEventRecord(w->bev[0], s0));
  for (size_t b = 0; b < g->colls.size(); ++b) {
    sphp_coll* c = g->colls[b];
    const sphp_amap* a = g->maps[b];
    double* lx = w->loc_x.as<double>() + g->off[b];
    double* ly = w->loc_y.as<double>() + g->off[b];
    cudaStream_t s = w->bs[b];
    CK(cudaStreamWaitEvent(s, w->bev[0], 0));
    CK(amap_scatter(a->dev(), x, lx, s));
    if (c->strategy == SPHP_STRATEGY_CUDA_STDMAT) {
      CK(elem_matvec(c->E, (int)c->t->nm, c->helm_H.as<double>(), lx, ly, s));
    } else {
      OpArgs o = base_args(c);
      o.in = lx;
      o.out = ly;
      o.mode = AsmMode::LOCAL;
      cudaError_t e = sumfac_launch(c, o, s);
      if (e == cudaErrorNotSupported) return fail(SPHP_ERR_UNSUPPORTED, "no kernel for this key");
      if (e != cudaSuccess) return cuda_fail(e, "sphp_gsys_apply");
    }
    CK(cudaEventRecord(w->bev[1 + b], s));
    CK(cudaStreamWaitEvent(s0, w->bev[1 + b], 0));
  }
  CK(owner_assemble_csr32(g->num_global, g->rowp.as<int>(), g->ent.as<int>(), w->loc_y.as<double>(), y, s0));
  return SPHP_OK;
}

int sphp_gsys_reserve(sphp_gsys* g, sphp_stream stream) {
  if (!g) return fail(SPHP_ERR_BAD_ARG, "null argument");
  Workspace* w = nullptr;
  return gsys_workspace(g, (cudaStream_t)stream, &w);
}

int sphp_gsys_destroy(sphp_gsys* g) {
  delete g;
  return SPHP_OK;
}

// e2e path with HOST vectors: x (num_global) -> device, fused assembled
// apply, y -> host; staging buffers owned by the collection; synchronises.
// Periodic split maps take the slab pipeline above.
int sphp_helmholtz_assembled_host(sphp_coll* c, const sphp_amap* a, const double* x, double* y,
                                  sphp_stream stream) {
  NvtxRange nvtx_range("sphp_helmholtz_assembled_host");
  if (!c || !a || !x || !y) return fail(SPHP_ERR_BAD_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (c->op == SPHP_OP_HELMHOLTZ && c->strategy == SPHP_STRATEGY_CUDA_SUMFAC && a->periodic &&
      (a->alg == SPHP_ASSEMBLY_SPLIT || a->alg == SPHP_ASSEMBLY_CLASS) && a->P >= 2 && a->n % 4 == 0 &&
      a->E == c->E && a->nm == c->t->nm && c->t->shape == SPHP_SHAPE_HEX) {
    const std::vector<int> zb = host_slabs(a->n);
    if (zb.size() > 2) {
      if (int rc = amap_device(a)) return rc;
      // class-range slabs need the mesh to divide into the operator's tiles
      // (n % 8 covers every order's tile)
      const bool use_class = a->alg == SPHP_ASSEMBLY_CLASS && a->n % 8 == 0;
      const int rc = assembled_host_pipelined(c, a, x, y, s, zb, use_class);
      // no class-mode tile for this key: the same pipeline on split
      if (rc == SPHP_ERR_UNSUPPORTED && use_class) return assembled_host_pipelined(c, a, x, y, s, zb, false);
      return rc;
    }
  }
  const size_t b = sizeof(double) * a->num_global;
  Workspace* w = c->ws.get(s);
  CKW(w->host_in.ensure_on(b, s));
  CKW(w->host_out.ensure_on(b, s));
  CK(cudaMemcpyAsync(w->host_in.p, x, b, cudaMemcpyHostToDevice, s));
  int rc = sphp_helmholtz_assembled(c, a, w->host_in.as<double>(), w->host_out.as<double>(), 0, stream);
  if (rc) return rc;
  CK(cudaMemcpyAsync(y, w->host_out.p, b, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return SPHP_OK;
}

// ---- solver support (assembly.py:185-266) ------------------------------------
int sphp_helmholtz_diagonal(sphp_coll* c, double* out, sphp_stream stream) {
  NvtxRange nvtx_range("sphp_helmholtz_diagonal");
  if (!c || !out) return fail(SPHP_ERR_BAD_ARG, "null argument");
  if (c->op != SPHP_OP_HELMHOLTZ) return fail(SPHP_ERR_BAD_ARG, "collection is not a Helmholtz operator");
  sphp_tables* t = c->t;
  for (int a = 1; a < t->dim; ++a)
    if (t->m[a] != t->m[0] || t->q[a] != t->q[0])
      return fail(SPHP_ERR_UNSUPPORTED, "diagonal needs equal modes/points per direction");
  int rc = tables_device(t);
  if (rc) return rc;
  DiagJob j;
  j.dim = t->dim;
  j.m = t->m[0];
  j.Q = t->q[0];
  j.kind = c->geom_kind;
  j.E = c->E;
  j.stride = c->gstride;
  j.cs = c->cs;
  j.lam = c->lam;
  j.B = t->d_B.as<double>();
  j.Bd = t->d_Bd.as<double>();
  j.w = t->d_w.as<double>();
  j.geom = c->geom;
  j.out = out;
  CK(helmholtz_diagonal(j, (cudaStream_t)stream));
  return SPHP_OK;
}

int64_t sphp_reduction_workspace(void) { return 2 + reduction_partials(); }

int sphp_vec_dot2(int64_t n, const double* a, const double* b, const double* c, const double* d,
                  double* ws, sphp_stream stream) {
  if (!a || !b || !ws || ((c == nullptr) != (d == nullptr))) return fail(SPHP_ERR_BAD_ARG, "bad dot arguments");
  CK(vec_dot2(n, a, b, c, d, ws + 2, ws, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_cg_init(int64_t n, const double* rhs, const double* dinv, double* x, double* r, double* z,
                 double* p, double* ws, sphp_stream stream) {
  if (!rhs || !dinv || !x || !r || !z || !p || !ws) return fail(SPHP_ERR_BAD_ARG, "null argument");
  CK(cg_init(n, rhs, dinv, x, r, z, p, ws + 2, ws, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_cg_update(int64_t n, double alpha, const double* p, const double* ap, double* x, double* r,
                   const double* dinv, double* z, double* ws, sphp_stream stream) {
  if (!p || !ap || !x || !r || !dinv || !z || !ws) return fail(SPHP_ERR_BAD_ARG, "null argument");
  CK(cg_update(n, alpha, p, ap, x, r, dinv, z, ws + 2, ws, (cudaStream_t)stream));
  return SPHP_OK;
}

int64_t sphp_cg_state_size(int max_iter) { return cg_state_size(max_iter); }

int sphp_cg_init_dev(int64_t n, const double* rhs, const double* dinv, double* x, double* r, double* z,
                     double* p, double* st, int max_iter, double tol, sphp_stream stream) {
  if (!rhs || !dinv || !x || !r || !z || !p || !st || max_iter < 0) return fail(SPHP_ERR_BAD_ARG, "null argument");
  CK(cg_init_dev(n, rhs, dinv, x, r, z, p, st, max_iter, tol, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_cg_step_dev(int64_t n, const double* p, const double* ap, double* x, double* r, const double* dinv,
                     double* z, double* st, int max_iter, sphp_stream stream) {
  NvtxRange nvtx_range("sphp_cg_step_dev");
  if (!p || !ap || !x || !r || !dinv || !z || !st) return fail(SPHP_ERR_BAD_ARG, "null argument");
  CK(cg_step_dev(n, p, ap, x, r, dinv, z, const_cast<double*>(p), st, max_iter, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_cg_direction(int64_t n, double beta, const double* z, double* p, sphp_stream stream) {
  if (!z || !p) return fail(SPHP_ERR_BAD_ARG, "null argument");
  CK(cg_direction(n, beta, z, p, (cudaStream_t)stream));
  return SPHP_OK;
}

// build_assembly_map (assembly.py:72-138) for meshio.structured_quad_mesh
// (meshio.py:377-413): vertex j*(nx+1)+i, horizontal segments j*nx+i, then
// vertical (ny+1)*nx + j*(nx+1) + i, element j*nx+i with loop
// (v(i,j), v(i+1,j), v(i+1,j+1), v(i,j+1)); every edge is traversed
// forward, so all signs are +1.  dirichlet_mask: 1 south, 2 east, 4 north,
// 8 west.  codes packed per element (m_e^2 each) at offsets[e].
int sphp_quadmap_structured(int nx, int ny, const int* orders, int dmask, int64_t* num_global,
                            int64_t* num_dirichlet, int64_t* offsets, int64_t* codes) {
  if (nx < 1 || ny < 1 || !orders || !num_global) return fail(SPHP_ERR_BAD_ARG, "bad arguments");
  const int64_t E = (int64_t)nx * ny;
  const int64_t NV = (int64_t)(nx + 1) * (ny + 1);
  const int64_t NS = (int64_t)(ny + 1) * nx + (int64_t)ny * (nx + 1);
  auto vid = [nx](int i, int j) -> int64_t { return (int64_t)j * (nx + 1) + i; };
  auto hseg = [nx](int i, int j) -> int64_t { return (int64_t)j * nx + i; };
  auto vseg = [nx, ny](int i, int j) -> int64_t { return (int64_t)(ny + 1) * nx + (int64_t)j * (nx + 1) + i; };
  for (int64_t e = 0; e < E; ++e)
    if (orders[e] < 1) return fail(SPHP_ERR_BAD_ARG, "orders must be >= 1");
  std::vector<int> eord(NS, 1 << 30);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int P = orders[(int64_t)j * nx + i];
      const int64_t segs[4] = {hseg(i, j), vseg(i + 1, j), hseg(i, j + 1), vseg(i, j)};
      for (int k = 0; k < 4; ++k) eord[segs[k]] = std::min(eord[segs[k]], P);
    }
  std::vector<char> dseg(NS, 0), dvert(NV, 0);
  auto mark_h = [&](int j) {
    for (int i = 0; i < nx; ++i) {
      dseg[hseg(i, j)] = 1;
      dvert[vid(i, j)] = dvert[vid(i + 1, j)] = 1;
    }
  };
  auto mark_v = [&](int i) {
    for (int j = 0; j < ny; ++j) {
      dseg[vseg(i, j)] = 1;
      dvert[vid(i, j)] = dvert[vid(i, j + 1)] = 1;
    }
  };
  if (dmask & 1) mark_h(0);
  if (dmask & 2) mark_v(nx);
  if (dmask & 4) mark_h(ny);
  if (dmask & 8) mark_v(0);
  std::vector<int64_t> vg(NV), eg(NS);  // vertex gid; first gid of each segment's bubbles
  int64_t gid = 0;
  for (int64_t v = 0; v < NV; ++v)
    if (dvert[v]) vg[v] = gid++;
  for (int64_t sdx = 0; sdx < NS; ++sdx)
    if (dseg[sdx]) {
      eg[sdx] = gid;
      gid += std::max(0, eord[sdx] - 1);
    }
  const int64_t nd = gid;
  for (int64_t v = 0; v < NV; ++v)
    if (!dvert[v]) vg[v] = gid++;
  for (int64_t sdx = 0; sdx < NS; ++sdx)
    if (!dseg[sdx]) {
      eg[sdx] = gid;
      gid += std::max(0, eord[sdx] - 1);
    }
  int64_t off = 0;
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int64_t e = (int64_t)j * nx + i;
      const int m = orders[e] + 1;
      if (offsets) offsets[e] = off;
      std::vector<int64_t> l2g((size_t)m * m, -2);
      auto flat = [m](int p, int q) { return p * m + q; };
      const int64_t loop[4] = {vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)};
      const int vmodes[4] = {0, m, m + 1, 1};
      for (int k = 0; k < 4; ++k) l2g[vmodes[k]] = vg[loop[k]];
      const int64_t segs[4] = {hseg(i, j), vseg(i + 1, j), hseg(i, j + 1), vseg(i, j)};
      for (int le = 0; le < 4; ++le)
        for (int k = 2; k < m; ++k) {
          const int mode = le == 0 ? flat(k, 0) : le == 1 ? flat(1, k) : le == 2 ? flat(k, 1) : flat(0, k);
          l2g[mode] = (k <= eord[segs[le]]) ? eg[segs[le]] + (k - 2) : -1;
        }
      for (int n = 0; n < m * m; ++n)
        if (l2g[n] == -2) l2g[n] = gid++;  // interiors, ascending local order
      if (codes)
        for (int n = 0; n < m * m; ++n) codes[off + n] = l2g[n];
      off += (int64_t)m * m;
    }
  if (offsets) offsets[E] = off;
  *num_global = gid;
  if (num_dirichlet) *num_dirichlet = nd;
  return SPHP_OK;
}


// ---------------------------------------------------------------------------
// DG primitives (dg.cu)
// ---------------------------------------------------------------------------
int sphp_batched_matvec(int64_t E, int m, int n, const double* A, const double* x, const double* s,
                        double alpha, int accumulate, double* y, sphp_stream stream) {
  if (E < 0 || m < 0 || n < 0) return fail(SPHP_ERR_BAD_ARG, "negative size");
  if (E * m > 0 && (!A || !x || !y)) return fail(SPHP_ERR_BAD_ARG, "null argument");
  CK(sphp::batched_matvec(E, m, n, A, x, s, alpha, accumulate, y, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_trace_extract(int64_t T, int nq, int np, const double* ex, const int64_t* idx,
                       const double* phys, double* out, sphp_stream stream) {
  if (T < 0 || nq < 0 || np < 0) return fail(SPHP_ERR_BAD_ARG, "negative size");
  if (T * nq > 0 && (!ex || !idx || !phys || !out)) return fail(SPHP_ERR_BAD_ARG, "null argument");
  CK(sphp::trace_extract(T, nq, np, ex, idx, phys, out, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_trace_lift(int nrhs, int64_t E, int nm, int nq, int64_t T, const int64_t* rowptr,
                    const int64_t* codes, const double* Lm, const double* Lp, const double* w,
                    const double* s, double* b, sphp_stream stream) {
  if (nrhs < 0 || E < 0 || nm < 0 || nq < 0 || T < 0) return fail(SPHP_ERR_BAD_ARG, "negative size");
  if ((int64_t)nrhs * E * nm > 0 && (!rowptr || !codes || !Lm || !s || !b))
    return fail(SPHP_ERR_BAD_ARG, "null argument");
  CK(sphp::trace_lift(nrhs, E, nm, nq, T, rowptr, codes, Lm, Lp, w, s, b, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_ape_trace_flux(int64_t npts, int riemann, int bc, const double* qm, const double* qp,
                        const double* gv, const double* nrm, const double* base, const double* w,
                        double* out, int64_t out_stride, sphp_stream stream) {
  if (riemann != SPHP_RIEMANN_UPWIND && riemann != SPHP_RIEMANN_LAXFRIEDRICHS)
    return fail(SPHP_ERR_BAD_ARG, "unknown Riemann flux kind");
  if (bc < SPHP_BC_INTERIOR || bc > SPHP_BC_DIRICHLET) return fail(SPHP_ERR_BAD_ARG, "unknown bc kind");
  if (npts > 0 && (!qm || !nrm || !base || !w || !out || (bc == SPHP_BC_INTERIOR && !qp) ||
                   (bc == SPHP_BC_DIRICHLET && !gv)))
    return fail(SPHP_ERR_BAD_ARG, "null argument");
  if (out_stride != 0 && out_stride < npts) return fail(SPHP_ERR_BAD_ARG, "out_stride < npts");
  CK(sphp::ape_trace_flux(npts, riemann, bc, qm, qp, gv, nrm, base, w, out,
                          out_stride ? out_stride : npts, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_ape_volume(int64_t E, int np, const double* q, const double* base, double* G, double* HX,
                    double* HY, sphp_stream stream) {
  if (E * np > 0 && (!q || !base || !G || !HX || !HY)) return fail(SPHP_ERR_BAD_ARG, "null argument");
  CK(sphp::ape_volume(E, np, q, base, G, HX, HY, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_advect_volume(int64_t E, int np, const double* ax, const double* ay, const double* u,
                       double* F, sphp_stream stream) {
  if (E * np > 0 && (!ax || !ay || !u || !F)) return fail(SPHP_ERR_BAD_ARG, "null argument");
  CK(sphp::advect_volume(E, np, ax, ay, u, F, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_advect_trace_flux(int64_t npts, int bc, const double* an, const double* um,
                           const double* up, const double* gv, double* out, sphp_stream stream) {
  if (bc < SPHP_BC_INTERIOR || bc > SPHP_BC_DIRICHLET || bc == SPHP_BC_RIGID_WALL)
    return fail(SPHP_ERR_BAD_ARG, "bc kind unsupported for advection");
  if (npts > 0 && (!an || !um || !out || (bc == SPHP_BC_INTERIOR && !up) ||
                   (bc == SPHP_BC_DIRICHLET && !gv)))
    return fail(SPHP_ERR_BAD_ARG, "null argument");
  CK(sphp::advect_trace_flux(npts, bc, an, um, up, gv, out, (cudaStream_t)stream));
  return SPHP_OK;
}

int sphp_scale_points(int64_t n, const double* c, const double* v, const double* src, double* out,
                      sphp_stream stream) {
  if (n > 0 && (!c || !v || !out)) return fail(SPHP_ERR_BAD_ARG, "null argument");
  CK(sphp::scale_points(n, c, v, src, out, (cudaStream_t)stream));
  return SPHP_OK;
}

}  // extern "C"
