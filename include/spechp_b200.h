/*
 * spechp_b200 — C ABI over the B200 (sm_100a) Collections kernels.
 *
 * Drop-in boundary for the spechp Collections hot path.  The reference is
 * pure Python/numpy (/root/reference/pkg/src/spechp), so there is no
 * reference FFI; every entry point below replaces the Python routine cited
 * beside it, and INTEGRATION.md shows the ctypes binding a spechp
 * maintainer would add to `collections.py` / `assembly.py`.
 *
 * Conventions (all mirror the reference):
 *   - FP64 throughout; blocks are C-contiguous, element-major:
 *       (E, nmodes) / (E, npoints) / (E, dim, npoints)       collections.py:189-200
 *   - quad coefficient n = p*m2 + q, point (i,j) -> i*Q2 + j  stdregions.py:1-14
 *     hex  coefficient n = (p*m2+q)*m3 + r, point ((i*Q2)+j)*Q3 + k (generalised)
 *   - 1D Modified_A storage boundary-first                    basis.py:111-114
 *   - all data pointers passed to apply/scatter/assemble are DEVICE pointers
 *     unless the function name ends in _host; `stream` is a cudaStream_t
 *     (NULL = legacy default stream).
 *   - return value: SPHP_OK (0) or a negative SPHP_ERR_*; the message is in
 *     sphp_last_error() (thread-local), with the reference's wording where
 *     the reference raises (CollectionError text, collections.py:197-200).
 *   - handles are immutable after create (except set_lambda, which must not
 *     run concurrently with applies of the handle; collections.py:76-90):
 *     device tables, StdMat operators and map tables are built by create.
 *     Everything an apply writes besides its output lives in a per-stream
 *     workspace of the handle, so applies of one handle on distinct streams
 *     may run concurrently (from any host threads); applies on one stream
 *     are ordered by it.  A stream's workspace is sized at its first apply
 *     (cudaMalloc) or by sphp_collection_reserve / sphp_gsys_reserve; an
 *     apply captured into a CUDA graph must find it reserved (otherwise it
 *     fails with SPHP_ERR_BAD_ARG instead of allocating inside the capture).
 *   - repeated applies are bitwise equal (test_collections.py:193-201) — no
 *     floating-point atomics anywhere.
 */
#ifndef SPECHP_B200_H
#define SPECHP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPHP_ABI_VERSION 1

/* ---- error codes ------------------------------------------------------ */
#define SPHP_OK 0
#define SPHP_ERR_BAD_SHAPE (-1)   /* block shape mismatch (CollectionError) */
#define SPHP_ERR_BAD_ARG (-2)     /* invalid argument / key               */
#define SPHP_ERR_UNSUPPORTED (-3) /* valid request this build cannot run  */
#define SPHP_ERR_CUDA (-4)        /* CUDA runtime failure                 */
#define SPHP_ERR_ALLOC (-5)       /* device or host allocation failure    */

/* ---- enums (values match the reference Enum order) -------------------- */
/* stdregions.py:41-44 Shape (+ HEX, the 3D generalisation)               */
#define SPHP_SHAPE_SEG 0
#define SPHP_SHAPE_QUAD 1
#define SPHP_SHAPE_TRI 2 /* Modified_A x Modified_B, collapsed (tri.cu) */
#define SPHP_SHAPE_HEX 3
/* quadrature.py:19-25 PointsType                                          */
#define SPHP_POINTS_GAUSS_LEGENDRE 0
#define SPHP_POINTS_GAUSS_LOBATTO_LEGENDRE 1
#define SPHP_POINTS_GAUSS_RADAU_M_LEGENDRE 2
/* basis.py:26-29 BasisType                                                */
#define SPHP_BASIS_MODIFIED_A 0
#define SPHP_BASIS_MODIFIED_B 1
#define SPHP_BASIS_LAGRANGE_GLL 2
/* collections.py:26-29 OperatorKind (+ the two the north star adds)       */
#define SPHP_OP_BWD_TRANS 0
#define SPHP_OP_IPRODUCT_WRT_BASE 1
#define SPHP_OP_PHYS_DERIV 2
#define SPHP_OP_IPRODUCT_WRT_DERIV_BASE 3 /* geometry.py:163-168 batched */
#define SPHP_OP_HELMHOLTZ 4               /* geometry.py:171-184 fused   */
/* collections.py:32-36 Strategy: the GPU strategies                       */
#define SPHP_STRATEGY_CUDA_SUMFAC 0 /* staged 1D contractions, fused     */
#define SPHP_STRATEGY_CUDA_STDMAT 1 /* dense elemental operator, DGEMM   */
/* geometry encodings (collections.py:110-129 precomputation, on device)   */
#define SPHP_GEOM_NONE 0   /* standard elements: weights only              */
#define SPHP_GEOM_AFFINE 1 /* per element: [det, inv (d x d row-major a,k)] */
#define SPHP_GEOM_POINT 2  /* per element, per point SoA: [wJ, inv_ak...]   */
#define SPHP_GEOM_METRIC 3 /* per element, per point SoA: symmetric
                              G_ab = wJ sum_k inv[a,k] inv[b,k] then wJ:
                              quad [G00,G01,G11,wJ]; hex
                              [G00,G01,G02,G11,G12,G22,wJ]                 */
/* analytic structured-grid maps (BASELINE.json configs)                   */
#define SPHP_MAP_AFFINE 0    /* x' = x                                   */
#define SPHP_MAP_QUAD_SINE 1 /* cfg2: x'=x+a sin2πy, y'=y+a sin2πx        */
#define SPHP_MAP_HEX_SINE 2  /* cfg4: x'=x+a sin2πy sin2πz                */

typedef struct sphp_tables sphp_tables;
typedef struct sphp_coll sphp_coll;
typedef struct sphp_amap sphp_amap;
typedef void* sphp_stream; /* cudaStream_t */

/* ---- library ------------------------------------------------------------ */
int sphp_abi_version(void);
const char* sphp_last_error(void);
/* number of SMs of the current device, 0 if none (used by the autotuner)   */
int sphp_device_sm_count(void);
/* stage plan of the fused hex Helmholtz for nmodes = M, npoints = Q per
 * direction: 0 K-row, 1 J-pencil, 3 i-column;
 * -1: no fast kernel for the key.  Every launch mode of a key (block in /
 * block out, class, gathering) runs the same plan, so all assembly
 * algorithms of a map return bitwise the same vector.                        */
int sphp_hex_helmholtz_plan(int M, int Q);

/* ---- reference elements: StdExpansion tables ----------------------------
 * replaces stdregions.StdExpansion(shape, basis_keys) (stdregions.py:70-240)
 * with quadrature.make_rule (quadrature.py:188-214), diff_matrix (:246-260)
 * and basis tables (basis.py:78-114).  Arrays have one entry per direction. */
int sphp_tables_create(int shape, const int* nmodes, const int* npoints,
                       const int* points_type, const int* basis_type,
                       sphp_tables** out);
int sphp_tables_destroy(sphp_tables* t);
/* copy direction `dir`'s tables to host: z,w (Q); B,Bd (m*Q, B[p*Q+i]);
 * D (Q*Q, D[i*Q+j]).  Any pointer may be NULL.  Triangles: direction 1 is
 * the Modified_B table with one row per triangle mode (nmodes rows).
 * Triangle collections: BwdTrans / IProductWRTBase / PhysDeriv (sumfac and
 * stdmat), IProductWRTDerivBase (stdmat); geometry NONE, AFFINE or POINT.   */
int sphp_tables_query(const sphp_tables* t, int dir, double* z, double* w,
                      double* B, double* Bd, double* D);
/* sizes: num_modes, num_points, dim                                        */
int sphp_tables_sizes(const sphp_tables* t, int64_t* nmodes, int64_t* npoints,
                      int* dim);

/* ---- geometry (geometry.py:115-142 semantics, evaluated on device) ------
 * Fill per-element geometry for structured-grid elements of an n^dim grid on
 * [0,L]^dim with an analytic map.  elem_ids: device int64 ids (NULL -> ids
 * e0 .. e0+E-1).  Element id = ex + n*(ey + n*ez).  Layout is that of
 * sphp_geom_stride().  Raises BAD_ARG if a Jacobian is non-positive.       */
int64_t sphp_geom_stride(const sphp_tables* t, int geom_kind);
int sphp_geom_analytic(const sphp_tables* t, int geom_kind, int mapping,
                       int n, const double* lengths, double amp, int64_t e0,
                       int64_t E, const int64_t* elem_ids, double* geom,
                       sphp_stream stream);
/* convert reference GeomFactors arrays (device, reference layout:
 * wj (E,np), inv (E,np,d,d)) into geom_kind layout                         */
int sphp_geom_from_factors(const sphp_tables* t, int geom_kind, int64_t E,
                           const double* wj, const double* inv, double* geom,
                           sphp_stream stream);

/* geometry.geom_factors (geometry.py:125-142) on the device for 2D
 * elements: dx, dy (E, 2, np) = reference-direction derivatives (d/dxi1,
 * d/dxi2) of the x and y coordinate maps at the expansion's points (e.g.
 * PhysDeriv of the interpolated map); writes POINT or METRIC records.
 * Non-positive Jacobians fail naming the first element (*first_bad).      */
int sphp_geom_from_jacobian(const sphp_tables* t, int kind, int64_t E, const double* dx,
                            const double* dy, double* geom, int64_t* first_bad,
                            sphp_stream stream);
/* ---- collections: replaces collections.Collection (collections.py:76-246)
 * geom: device pointer in `geom_kind` layout, borrowed (must outlive the
 * handle); NULL with SPHP_GEOM_NONE.  lambda only used by HELMHOLTZ.        */
int sphp_collection_create(const sphp_tables* t, int op, int strategy,
                           int64_t E, int geom_kind, const double* geom,
                           double lambda, sphp_coll** out);
int sphp_collection_destroy(sphp_coll* c);
int sphp_collection_set_lambda(sphp_coll* c, double lambda);
/* input_size / output_size per element, MAC count of one apply
 * (collections.py:250-273 generalised), algorithmic HBM bytes of one apply */
int sphp_collection_info(const sphp_coll* c, int64_t* input_size,
                         int64_t* output_size, int64_t* mac_count,
                         int64_t* hbm_bytes);
/* Collection.apply (collections.py:189-246) on device buffers:
 * in (E, input_size), out (E, output_size).  E must equal the handle's E
 * (CollectionError "block shape (a, b) does not match (E, n)").            */
int sphp_apply(sphp_coll* c, int64_t E, int64_t n_in, const double* in,
               double* out, sphp_stream stream);
/* same with HOST buffers: copies in -> device, apply, device -> out, all on
 * `stream`, then synchronises it.  Uses a workspace owned by the handle.   */
int sphp_apply_host(sphp_coll* c, int64_t E, int64_t n_in, const double* in,
                    double* out, sphp_stream stream);

/* ---- assembly: replaces assembly.AssemblyMap / assemble / scatter
 * (assembly.py:44-160) and GlobalSystem.apply (:168-182).
 * Codes: gid >= 0 (sign +1), -1 pinned (sign 0), -(gid+2) (sign -1).      */
int sphp_amap_create_explicit(int64_t E, int nmodes, const int64_t* codes_host,
                              int64_t num_global, sphp_amap** out);
/* periodic n^3 hex grid, uniform order P: numbering of assembly.py:89-133
 * generalised (vertices, edges, faces, interiors); indices computed on the
 * fly on device (no map traffic).                                          */
int sphp_amap_create_hex_periodic(int n, int P, sphp_amap** out);
/* periodic n^3 hex grid with per-element orders (host array, n^3 entries):
 * fills num_global; if codes != NULL also writes per-element codes packed
 * back to back (element e at offsets[e], offsets has n^3+1 entries).       */
int sphp_hexmap_variable(int n, const int* orders, int64_t* num_global,
                         int64_t* offsets, int64_t* codes);
/* rows [e0, e1) (element id ex + n (ey + n ez)) of the uniform-order
 * periodic map's codes, (e1 - e0, (P+1)^3) int64: a rank's slab of the
 * sharded operator without building the whole n^3 table                  */
int sphp_hexmap_periodic_codes(int n, int P, int64_t e0, int64_t e1, int64_t* codes);
/* the sharded operator's interface exchange (distributed.py): pack
 * dst[i] = src[idx[i]]; combine y[idx[i]] = lo[i] + hi[i] (the lower
 * rank's partial sum first, so both sides hold identical bits)            */
int sphp_index_gather(int64_t n, const int64_t* idx, const double* src, double* dst,
                      sphp_stream stream);
int sphp_index_sum2(int64_t n, const int64_t* idx, const double* lo, const double* hi,
                    double* y, sphp_stream stream);
int sphp_amap_destroy(sphp_amap* a);
/* assembly algorithm of sphp_assemble / sphp_helmholtz_assembled, both
 * deterministic (bitwise reproducible) and atomic-free.  Default: SPLIT for
 * periodic maps with P >= 2 and n % 4 == 0 (class-range scatter and owner
 * kernels, the fastest measured), OWNER otherwise.
 *   OWNER  gather -> elemental operator -> local block, then one
 *          owner-computes pass that sums each global dof in a fixed order;
 *   COLOUR colour classes (parity colours on periodic grids, greedy
 *          colouring of explicit maps) fused gather/scatter-add, one launch
 *          per colour in a fixed colour order;
 *   SPLIT  scatter kernel -> fused operator on the local block -> owner
 *          sum (three launches).                                          */
#define SPHP_ASSEMBLY_OWNER 0
#define SPHP_ASSEMBLY_COLOUR 1
#define SPHP_ASSEMBLY_SPLIT 2
#define SPHP_ASSEMBLY_CLASS 3  /* periodic maps: class-range gather in the operator + class owner sum */
int sphp_amap_set_algorithm(sphp_amap* a, int alg);
int sphp_amap_algorithm(const sphp_amap* a, int* alg);
int sphp_amap_info(const sphp_amap* a, int64_t* num_elements, int* nmodes,
                   int64_t* num_global, int* num_colours);
/* materialise the map codes (E*nmodes int64, host) — for bit-exact tests   */
int sphp_amap_codes(const sphp_amap* a, int64_t* codes_host);
/* assembly.scatter: global (num_global) -> local (E, nmodes), pinned -> 0  */
int sphp_scatter(const sphp_amap* a, const double* global, double* local,
                 sphp_stream stream);
/* assembly.assemble: local (E, nmodes) -> global (num_global), overwritten;
 * deterministic colour-ordered signed sum (no atomics)                     */
int sphp_assemble(const sphp_amap* a, const double* local, double* global,
                  sphp_stream stream);
/* GlobalSystem.apply for a HELMHOLTZ collection: y = A^T H A x, fused
 * gather -> elemental Helmholtz -> colour-ordered scatter-add.  When
 * accumulate != 0, y is added to instead of overwritten (variable-order
 * meshes: one call per order batch, same y).                              */
int sphp_helmholtz_assembled(sphp_coll* c, const sphp_amap* a, const double* x,
                             double* y, int accumulate, sphp_stream stream);
/* same with HOST vectors (num_global each): copies in, applies, copies out
 * on `stream` and synchronises it (the end-to-end path)                    */
int sphp_helmholtz_assembled_host(sphp_coll* c, const sphp_amap* a,
                                  const double* x, double* y,
                                  sphp_stream stream);
/* pre-size the per-stream workspace of `c` for applies on `stream`:
 * SPHP_RESERVE_DEVICE — sphp_apply and, with map `a` (may be NULL),
 * sphp_helmholtz_assembled; SPHP_RESERVE_HOST — the *_host paths.          */
#define SPHP_RESERVE_DEVICE 1
#define SPHP_RESERVE_HOST 2
int sphp_collection_reserve(sphp_coll* c, const sphp_amap* a, int flags,
                            sphp_stream stream);
/* measurement: one apply (accumulate = 0) with a CUDA event after each of
 * its launches on `stream`; synchronises and writes the launches'
 * durations (ms) to ms[0 .. *nphases)  (class: operator, owner sum;
 * split: scatter, operator, owner sum)                                      */
int sphp_helmholtz_assembled_phases(sphp_coll* c, const sphp_amap* a,
                                    const double* x, double* y,
                                    sphp_stream stream, int max_phases,
                                    float* ms, int* nphases);

/* GlobalSystem over several per-order Helmholtz batches on explicit maps
 * sharing one numbering (assembly.py:185-215 with per-order element groups,
 * the variable-order configuration): per batch a scatter and the fused
 * operator on one concatenated local block, then ONE owner-computes pass
 * (fixed (batch, element, mode) order: deterministic).  The handle keeps
 * the collections and maps by pointer: they must outlive it.             */
typedef struct sphp_gsys sphp_gsys;
int sphp_gsys_create(sphp_coll* const* colls, const sphp_amap* const* maps,
                     int nbatch, int64_t num_global, sphp_gsys** out);
int sphp_gsys_apply(sphp_gsys* g, const double* x, double* y, sphp_stream stream);
int sphp_gsys_reserve(sphp_gsys* g, sphp_stream stream);  /* workspace of `stream` */
int sphp_gsys_destroy(sphp_gsys* g);

/* ---- solver support: GlobalSystem.diag / solve_pcg (assembly.py:185-266) -- */
/* diagonal of every elemental Helmholtz matrix (E, nmodes) — assemble it
 * with sphp_assemble for the Jacobi preconditioner                          */
int sphp_helmholtz_diagonal(sphp_coll* c, double* out, sphp_stream stream);
/* deterministic vector reductions for CG.  ws: device workspace of
 * sphp_reduction_workspace() doubles; results land in ws[0], ws[1].        */
int64_t sphp_reduction_workspace(void);
/* ws[0] = a.b, ws[1] = c.d (c, d may both be NULL)                          */
int sphp_vec_dot2(int64_t n, const double* a, const double* b, const double* c,
                  const double* d, double* ws, sphp_stream stream);
/* x = 0, r = rhs, z = p = dinv*r; ws = [r.z, r.r]                           */
int sphp_cg_init(int64_t n, const double* rhs, const double* dinv, double* x,
                 double* r, double* z, double* p, double* ws, sphp_stream stream);
/* x += alpha p, r -= alpha Ap, z = dinv*r; ws = [r.z, r.r]                  */
int sphp_cg_update(int64_t n, double alpha, const double* p, const double* ap,
                   double* x, double* r, const double* dinv, double* z,
                   double* ws, sphp_stream stream);
/* p = z + beta p                                                            */
int sphp_cg_direction(int64_t n, double beta, const double* z, double* p,
                      sphp_stream stream);
/* the same iteration with the scalars on the device (no host round trip;
 * a chunk of iterations can be captured into a CUDA graph): `st` holds
 * sphp_cg_state_size(max_iter) doubles — st[0] rz, st[1] rr, st[5] |rhs|,
 * st[7] converged flag, st[8] iterations, st[9 + k] residual of iteration
 * k; init sets x = 0, r = rhs, z = p = dinv r; each step takes ap = A p and
 * does alpha = rz / p.Ap, the update, the residual test against `tol`
 * and the new direction; steps after convergence leave x unchanged.     */
int64_t sphp_cg_state_size(int max_iter);
int sphp_cg_init_dev(int64_t n, const double* rhs, const double* dinv, double* x,
                     double* r, double* z, double* p, double* st, int max_iter,
                     double tol, sphp_stream stream);
int sphp_cg_step_dev(int64_t n, const double* p, const double* ap, double* x, double* r,
                     const double* dinv, double* z, double* st, int max_iter,
                     sphp_stream stream);
/* build_assembly_map (assembly.py:72-138) for meshio.structured_quad_mesh
 * (meshio.py:377-413) with per-element orders; dirichlet_mask bits:
 * 1 south, 2 east, 4 north, 8 west.  Codes packed per element (m_e^2 each,
 * element e at offsets[e], offsets has nx*ny+1 entries); NULL arrays only
 * return the counts.                                                         */
int sphp_quadmap_structured(int nx, int ny, const int* orders, int dirichlet_mask,
                            int64_t* num_global, int64_t* num_dirichlet,
                            int64_t* offsets, int64_t* codes);

/* ---- DG primitives: the batched pieces of the
 * reference's DGSystem (solvers.py:189-392), AdvectionOperator.rhs
 * (solvers.py:425-457) and ape_rhs (solvers.py:546-642) that are not
 * Collections operators.  Device pointers, row-major, FP64; deterministic. */
/* y[e] = alpha * A[e] (s[e] x[e]) (+ y[e] if accumulate); A (E, m, n),
 * x (E, n), y (E, m); s per-element scale or NULL.  DGSystem.mass_solve
 * (solvers.py:353-354) with A = minv.                                       */
int sphp_batched_matvec(int64_t E, int m, int n, const double* A, const double* x,
                        const double* s, double alpha, int accumulate, double* y,
                        sphp_stream stream);
/* out[t, q] = sum_n ex[t, q, n] phys[idx[t], n]: DGSystem.trace_minus /
 * trace_plus (solvers.py:366-372)                                           */
int sphp_trace_extract(int64_t T, int nq, int np, const double* ex, const int64_t* idx,
                       const double* phys, double* out, sphp_stream stream);
/* deterministic trace lift (np.add.at of solvers.py:374-389, 571-586): for
 * every rhs r and element e, over the CSR list rowptr[e]..rowptr[e+1] of
 * codes c = (t << 2) | (plus << 1) | neg, in list order,
 *   b[r, e, n] (-)= sum_q L[t, n, q] w[t, q] s[r, t, q],  L = plus ? Lp : Lm;
 * w may be NULL (weights already in s).  Lm, Lp (T, nm, nq), s (nrhs, T, nq),
 * b (nrhs, E, nm) updated in place.                                         */
int sphp_trace_lift(int nrhs, int64_t E, int nm, int nq, int64_t T, const int64_t* rowptr,
                    const int64_t* codes, const double* Lm, const double* Lp, const double* w,
                    const double* s, double* b, sphp_stream stream);
#define SPHP_RIEMANN_UPWIND 0
#define SPHP_RIEMANN_LAXFRIEDRICHS 1
#define SPHP_BC_INTERIOR 0   /* q_plus given                              */
#define SPHP_BC_RIGID_WALL 1 /* ghost = mirrored normal velocity           */
#define SPHP_BC_FARFIELD 2   /* ghost = 0                                  */
#define SPHP_BC_DIRICHLET 3  /* ghost p = 2 g - p (APE), u = 2 g - u (adv.) */
/* APE trace flux (riemann_flux, solvers.py:142-181, ghost states of
 * _ghost_state, solvers.py:498-517): qm, qp planes (3, npts) = (p, ux, uy),
 * qp NULL unless SPHP_BC_INTERIOR; gv (npts) for DIRICHLET; nrm (npts, 2);
 * base planes (4, npts) = (ux, uy, rho, c2); w = warc (npts).  out: 3 planes
 * (w F_p / c2, w F_ux, w F_uy) of npts values, plane r at out + r *
 * out_stride (out_stride 0 = npts).                                         */
int sphp_ape_trace_flux(int64_t npts, int riemann, int bc, const double* qm, const double* qp,
                        const double* gv, const double* nrm, const double* base, const double* w,
                        double* out, int64_t out_stride, sphp_stream stream);
/* APE volume fluxes (solvers.py:563-569), negated: q planes (3, E*np),
 * base planes (4, E*np); G = -(gx, gy), HX = -(h, 0), HY = -(0, h), each
 * (E, 2, np) as IProductWRTDerivBase takes it.                              */
int sphp_ape_volume(int64_t E, int np, const double* q, const double* base, double* G,
                    double* HX, double* HY, sphp_stream stream);
/* advection: F = (ax u, ay u) as (E, 2, np) (solvers.py:428-430), and the
 * upwind trace flux an (an >= 0 ? um : up) with boundary ghosts
 * (solvers.py:433-455; bc INTERIOR needs up, DIRICHLET gv)                  */
int sphp_advect_volume(int64_t E, int np, const double* ax, const double* ay, const double* u,
                       double* F, sphp_stream stream);
int sphp_advect_trace_flux(int64_t npts, int bc, const double* an, const double* um,
                           const double* up, const double* gv, double* out, sphp_stream stream);
/* out = c v (+ src): the pointwise-c2 branch of ape_rhs (solvers.py:621-624) */
int sphp_scale_points(int64_t n, const double* c, const double* v, const double* src,
                      double* out, sphp_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* SPECHP_B200_H */
