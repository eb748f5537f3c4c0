/*
 * nesa_b200.h -- C ABI of the B200-native NESA matrix-vector product.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (taskfmm, /root/reference/pkg/src/taskfmm) has no FFI; its operator API is
 * Python:
 *
 *   mvp_serial(tree, ops, q, near=True, far=True)           fastmvp.py:142-172
 *   mvp(tree, ops, q, runtime, vec=None, near, far)          fastmvp.py:124-139
 *   StageVectors / make_stage_vectors / reset                fastmvp.py:24-59
 *   Task(kind, accesses, _gemv_body(A, x, y))                fastmvp.py:62-65,
 *                                                             runtime.py:73-86
 *
 * The Python host package (paper_1801_03589_b200.fastmvp.mvp) keeps those
 * signatures and calls this library through ctypes:
 *
 *   nesa_plan_create   <- the one-time part of mvp(): flattening Tree +
 *                         OperatorSet (quadtree.py:71-93, operators.py:158-253)
 *                         and allocating StageVectors (fastmvp.py:48-59);
 *                         the plan owns every device buffer.
 *   nesa_matvec        <- one call of mvp_serial / mvp: gather q[perm]
 *                         (fastmvp.py:148), near field (152-156), radiation,
 *                         source transfer, translation, potential transfer,
 *                         reception (157-171), scatter phi[inverse_perm]
 *                         (172).  Zeroing of the work vectors (StageVectors.
 *                         reset, fastmvp.py:42-45) is internal.
 *   nesa_plan_destroy  <- end of the Runtime / StageVectors lifetime.
 *   nesa_last_error    <- the exception text the reference raises at
 *                         Runtime.barrier (runtime.py:163-168).
 *
 * Conventions: 0 = NESA_OK, any other return is a nesa_status; the detail
 * is in nesa_last_error() (thread-local).  All pointers in
 * nesa_plan_desc are HOST pointers and are copied during create.  Vector
 * pointers passed to nesa_matvec are DEVICE pointers owned by the caller.
 * A plan is immutable after create except for its workspace, so one plan
 * serves one stream at a time (the reference's single-submitter rule,
 * SPEC.md:461).
 */
#ifndef NESA_B200_H
#define NESA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NESA_ABI_VERSION 3

typedef enum {
  NESA_OK = 0,
  NESA_ERR_INVALID = 1,   /* bad descriptor / argument  (reference: ValueError) */
  NESA_ERR_CUDA = 2,      /* CUDA runtime or launch failure                       */
  NESA_ERR_OOM = 3,       /* device allocation failed                             */
  NESA_ERR_UNSUPPORTED = 4
} nesa_status;

typedef enum { NESA_F64 = 0, NESA_F32 = 1 } nesa_dtype;

/* nesa_matvec flags (reference: mvp_serial's near= / far= keywords). */
#define NESA_NEAR 1u
#define NESA_FAR 2u
#define NESA_PROFILE 16u /* record per-stage CUDA events (nesa_profile_*) */
#define NESA_PROFILE_NEAR 32u /* with NESA_PROFILE: only the near-field stage (its events
                                 sit on the near branch, off the critical path) */

typedef struct nesa_plan nesa_plan;

/*
 * Flattened Tree + operator tables.  Group ids follow the reference
 * (quadtree.py:177-199): leaves 0..n_leaves-1, then level L-1 ... l0, each
 * level a contiguous id range in Morton order.
 */
typedef struct nesa_plan_desc {
  int32_t abi_version;   /* NESA_ABI_VERSION */
  int32_t op_dtype;      /* nesa_dtype: storage + arithmetic precision */
  int32_t Q;             /* equivalent sources per group (NesaParams.Q) */
  int32_t n_check;       /* oversampling * Q                              */
  int64_t N;             /* points                                        */
  int64_t n_leaves;
  int64_t n_groups;
  int32_t l0, L;         /* coarsest / leaf level                          */

  /* tree (Tree.perm, Group.start/stop/parent, quadrant, level ranges) */
  const int64_t* perm;          /* [N] tree position -> original index     */
  const int64_t* group_start;   /* [G] point range in tree order           */
  const int64_t* group_stop;    /* [G]                                     */
  const int64_t* parent;        /* [G] parent id, -1 at level l0           */
  const int32_t* quad;          /* [G] 2*(ix&1)+(iy&1); octant with NESA_PLAN_OCTREE */
  const int64_t* level_first;   /* [L-l0+1] first id of level l0+i         */
  const int64_t* level_count;   /* [L-l0+1]                                */
  const int64_t* nbr_ptr;       /* [n_leaves+1] Group.neighbors CSR        */
  const int64_t* nbr_idx;
  const int64_t* int_ptr;       /* [G+1] Group.interaction CSR             */
  const int64_t* int_idx;
  const int64_t* int_dtab;      /* [nnz] index of the entry's D matrix     */

  /* shared operator tables, float64 row-major (y = M x) */
  const double* C;              /* [(L-l0) * 4 * Q * Q] child level l -> row l-l0-1
                                   (8 matrices per level with NESA_PLAN_OCTREE)    */
  const double* B;              /* same layout                                      */
  const double* D;              /* [n_dtab * Q * Q]                                 */
  int64_t n_dtab;

  /* Per-leaf / per-pair blocks computed on the host (OperatorSet), float64,
   * or NULL to assemble them on the device from the geometry below:
   *   near_blob: per leaf a, the n_a x W_a slab [K_a,b1 | ... | K_a,bk]
   *              (neighbor order), column-major, leaves concatenated;
   *   V_blob:    per leaf, Q x n column-major;  U_blob: n x Q column-major. */
  const double* near_blob;
  const double* V_blob;
  const double* U_blob;

  /* device-assembly inputs (operators.py:107-155 restated on the GPU) */
  const double* points_tree;    /* [N*2] Tree.points                       */
  const double* leaf_center;    /* [n_leaves*2] Group.center               */
  const double* leaf_r_check;   /* [n_leaves] rho_out_check * half_side    */
  const double* leaf_r_inaux;   /* [n_leaves] rho_in_aux * half_side       */
  const double* out_fit_leaf;   /* [Q * n_check] outgoing fit at level L   */
  const double* check_cos;      /* [n_check] cos(2 pi i / n_check)         */
  const double* check_sin;
  const double* aux_cos;        /* [Q] cos(2 pi i / Q)                     */
  const double* aux_sin;

  /* Multi-GPU sub-plan: leaves [leaf_begin, leaf_end) are this rank's
   * targets (leaf_end <= leaf_begin means all leaves).  The plan then
   * computes near/V/U for those leaves and C/D/B for their ancestors;
   * source amplitudes of remote interaction partners arrive through the
   * halo exchange between nesa_matvec_stage 1 and 2. */
  int64_t leaf_begin, leaf_end;

  uint32_t options;             /* NESA_PLAN_* bits                                 */

  /* NESA_PLAN_HELMHOLTZ_NEAR (Track B): the near blocks are assembled on the
   * device from the tree-order 3D points (one per complex unknown) and the
   * wavenumber, G = exp(-j k r) / (4 pi r), zero on the diagonal
   * (paper_1801_03589_b200.helmholtz.helmholtz_matrix). */
  const double* points3;        /* [N/2 * 3] with the real embedding's doubled N    */
  double wavenumber;
} nesa_plan_desc;

/* nesa_plan_desc.options */
#define NESA_PLAN_FAR_ONLY 1u   /* no near operator: far-field products only (extra
                                   plans that share the columns of a many-RHS product) */
#define NESA_PLAN_OCTREE 2u     /* Track B: an octree (quad[] holds the child octant
                                   4(ix&1) + 2(iy&1) + (iz&1), C / B tables have 8 matrices
                                   per level), operators from the host (near / V / U blobs
                                   required).  Complex operators are passed in their real
                                   embedding: every complex entry a+ib becomes the 2x2 block
                                   [[a, -b], [b, a]], so N, Q and the group point ranges are
                                   doubled and a complex vector is a real one of 2N entries
                                   (paper_1801_03589_b200.plan3). */
#define NESA_PLAN_COMPLEX_NEAR 4u /* with NESA_PLAN_OCTREE: near_blob holds each leaf's complex
                                   slab row-split (2 n_a x W_a real, column-major: row 2r = Re,
                                   row 2r+1 = Im of complex row r; W_a complex columns), read
                                   once per product with complex vectors -- 8 bytes per complex
                                   float32 entry instead of the embedding's 16.  Products run
                                   one complex right-hand side per pass. */
#define NESA_PLAN_STORED_VU 8u   /* store the per-leaf V and U blocks (assembled on the device) even
                                   for float32 plans from geometry: products of more than 4 real
                                   columns then run the far field as batched GEMMs over 128-column
                                   passes (C5: many right-hand sides), float32 adds the near field
                                   as one tensor-core GEMM per pass (nesa_matvec_near_wide) */
#define NESA_PLAN_HELMHOLTZ_NEAR 16u /* with NESA_PLAN_OCTREE | NESA_PLAN_COMPLEX_NEAR: near_blob may be
                                   NULL; the row-split complex near blocks are evaluated on the
                                   device from points3 / wavenumber (float64, stored in op_dtype) */

int nesa_plan_create(const nesa_plan_desc* desc, int device, nesa_plan** out);

/*
 * phi = K~ q for nrhs right-hand sides.  q_dev / phi_dev hold N x nrhs
 * values in ORIGINAL point order, point-major (numpy (N,) or (N, nrhs)
 * C-order); complex vectors are interleaved (re, im) pairs.  The element
 * type follows op_dtype: NESA_F64 -> float64 / complex128, NESA_F32 ->
 * float32 / complex64.  stream = cudaStream_t or NULL (legacy default).
 * Stream-ordered, no host synchronisation.
 */
int nesa_matvec(nesa_plan* plan, const void* q_dev, void* phi_dev,
                int32_t nrhs, int32_t is_complex, uint32_t flags, void* stream);

/* Multi-GPU pieces of one product (used by the Python dist layer):
 * stage 1 = gather + radiation + source transfer (up to the exchange),
 * stage 2 = near field (concurrent) + translation + potential transfer +
 *           reception + scatter.
 * s_dev() exposes the (G, Q, nrhs_real) source-amplitude workspace for the
 * halo exchange between the two stages. */
int nesa_matvec_stage(nesa_plan* plan, int32_t stage, const void* q_dev,
                      void* phi_dev, int32_t nrhs, int32_t is_complex,
                      uint32_t flags, void* stream);
void* nesa_plan_s_dev(nesa_plan* plan, int32_t nrhs_real);

/*
 * Multi-GPU plan (the reference has no distributed layer,
 * SPEC.md:9): `desc` describes this rank's sub-plan (leaf_begin / leaf_end
 * set), `nccl_comm` is the caller's ncclComm_t (not owned) and `xd` the halo
 * exchange tables (paper_1801_03589_b200.dist.build_exchange).  nesa_matvec
 * on such a plan is the whole distributed product as ONE graph launch:
 * gather, near field (local leaves, concurrent), radiation and upward pass,
 * pack -> ncclAllGather -> combine of the partial source amplitudes,
 * translation and downward pass, reception of the rank's points (its rows of
 * phi; the other rows are left untouched).  NCCL is loaded at run time
 * (libnccl.so.2).
 */
typedef struct nesa_exchange_desc {
  int64_t n_export;             /* groups whose partial s this rank sends       */
  const int64_t* export_ids;    /* [n_export]                                   */
  int64_t max_export;           /* send rows per rank (>= every rank's n_export) */
  int64_t n_import;             /* groups whose s this rank completes           */
  const int64_t* import_ids;    /* [n_import]                                   */
  int32_t max_contrib;          /* contributors per imported group             */
  const int64_t* contrib;       /* [n_import][max_contrib]: row < nranks*max_export
                                   = gathered row, else own s row (row - that); -1 none */
} nesa_exchange_desc;

int nesa_plan_create_dist(const nesa_plan_desc* desc, int device, void* nccl_comm, int32_t rank,
                          int32_t nranks, const nesa_exchange_desc* xd, nesa_plan** out);
/* NCCL bootstrap helpers: a 128-byte ncclUniqueId (rank 0; share it with the
 * other ranks out of band) and a communicator per rank (ncclCommInitRank). */
int nesa_nccl_unique_id(void* out, int32_t bytes);
int nesa_nccl_comm_init(const void* unique_id, int32_t nranks, int32_t rank, int32_t device,
                        void** comm_out);
int nesa_nccl_comm_destroy(void* comm);

/* Columns [col0, col0 + ncols_real) of an (N, ld_real) row-major real block
 * (a complex right-hand side is 2 adjacent real columns) -- the same product
 * as nesa_matvec on that column range, in blocks of <= 4 columns.  Lets a
 * caller spread many right-hand sides over several plans on several streams
 * (reference: mvp_serial on a multi-column q, fastmvp.py:142-172). */
int nesa_matvec_cols(nesa_plan* plan, const void* q_dev, void* phi_dev, int32_t ld_real,
                     int32_t col0, int32_t ncols_real, uint32_t flags, void* stream);

/* phi[:, col0 : col0 + ncols_real] += near field of q for real columns of
 * (N, ld_real) row-major blocks in original order: float32 plans with tensor
 * cores, 128 columns per tcgen05 GEMM pass with the operator streamed once
 * (C5: many right-hand sides).  nesa_matvec / nesa_matvec_cols with more
 * than 4 real columns on such a plan run the far field in blocks and this
 * for the near field; callers splitting the far field over several plans
 * (nesa_matvec_cols with NESA_FAR only) add the near field with this call.
 * The first call packs the operator into the tensor-core layout. */
int nesa_matvec_near_wide(nesa_plan* plan, const void* q_dev, void* phi_dev, int32_t ld_real,
                          int32_t col0, int32_t ncols_real, void* stream);

int nesa_plan_destroy(nesa_plan* plan);

const char* nesa_last_error(void);

/* One Arnoldi step of the GMRES solver around the product (SURVEY.md §8f row
 * 2; the reference has no solver): orthogonalise w against the basis
 * V[0..kk) (V[j] = basis + j * stride elements; complex vectors of n
 * elements, float32 or float64) by classical Gram-Schmidt applied twice in
 * three passes over the basis, write v_out = w'' / |w''| and the Hessenberg
 * column hcol[0..kk] (float64 (re, im) pairs: h1 + h2, then |w''|).  work:
 * nesa_gs_work_bytes() bytes of device memory, zero-filled once before the
 * first step (it holds self-resetting arrival counters).  Stream-ordered, no
 * host synchronisation, bitwise reproducible; 1 <= kk <= 128.
 * nesa_gs_step_shifted first adds shift * V[kk-1] to w (the (shift I + K~)
 * operator of the solver, fused into the first pass). */
int64_t nesa_gs_work_bytes(void);
int nesa_gs_step(const void* basis, int64_t stride, int32_t kk, void* w, void* v_out, int64_t n,
                 int32_t is_f64, void* work, void* hcol, void* stream);
int nesa_gs_step_shifted(const void* basis, int64_t stride, int32_t kk, void* w, void* v_out, int64_t n,
                         int32_t is_f64, double shift, void* work, void* hcol, void* stream);
const char* nesa_gs_last_error(void);
int nesa_abi_version(void);

/* Plan statistics: see NESA_STAT_* */
#define NESA_STAT_NEAR_ENTRIES 0   /* stored near entries (sum n_a * W_a)   */
#define NESA_STAT_V_ENTRIES 1
#define NESA_STAT_U_ENTRIES 2
#define NESA_STAT_D_REFS 3
#define NESA_STAT_N_DTAB 4
#define NESA_STAT_DEVICE_BYTES 5
#define NESA_STAT_NEAR_CTAS 6
#define NESA_STAT_KERNELS_PER_MATVEC 7
#define NESA_STAT_V_MOMENTS 8        /* outgoing moments per leaf (0: stored V)   */
#define NESA_STAT_U_TERMS 9          /* incoming expansion terms (0: stored U)    */
#define NESA_STAT_GRAPH_CAPTURES 10  /* stream captures so far (one per schedule)  */
#define NESA_STAT_GRAPHS_CACHED 11   /* instantiated graphs held by the plan       */
#define NESA_STAT_NEAR_WIDE 12       /* 1: nesa_matvec_near_wide available          */
#define NESA_STAT_FAR_WIDE 13        /* 1: many-column products run the far field as GEMMs */
int64_t nesa_plan_stat(nesa_plan* plan, int32_t which);

/* Profiling: with NESA_PROFILE in flags each nesa_matvec records CUDA
 * events around its stages on the streams the kernels run on. */
#define NESA_STAGE_TOTAL 0
#define NESA_STAGE_NEAR 1
#define NESA_STAGE_FAR 2     /* radiation .. potential transfer */
#define NESA_STAGE_RECEPTION 3
#define NESA_N_STAGES 4
int nesa_profile_reset(nesa_plan* plan);
/* Synchronises; fills up to max durations (ms) of `stage`, returns count. */
int nesa_profile_read(nesa_plan* plan, int32_t stage, float* ms, int32_t max);
/* Diagnostics: with NESA_TRACE=1 in the environment at plan creation, a
 * profiled product records an event after every kernel.  Fills up to max
 * times (ms from the product's start) of the last profiled product and
 * returns the count; nesa_trace_name(i) names the kernel of entry i. */
int nesa_trace_read(nesa_plan* plan, float* ms, int32_t max);
const char* nesa_trace_name(nesa_plan* plan, int32_t i);
/* Diagnostics: per-CTA kernel timeline without graph nodes.  enable(cap)
 * makes every instrumented CTA append {tag, grid, start_ns, end_ns}
 * (process-wide; cap 0 turns it off); read copies up to max records
 * (4 x uint64 each), resets the log and returns the count. */
int nesa_ktrace_enable(nesa_plan* plan, int64_t capacity);
int64_t nesa_ktrace_read(nesa_plan* plan, unsigned long long* out, int64_t max_records);

/* Exact O(N^2) potential sum (reference: dense.dense_matvec, dense.py:14-33)
 * on the device, float64: phi_i = sum_{j != i} -0.5 log|x_i - x_j|^2 q_j.
 * points_dev: (n, 2) row-major; q_dev / phi_dev: (n, ncols) row-major,
 * ncols real columns (a complex vector = 2).  Synchronises the stream.
 * Coincident distinct points -> NESA_ERR_INVALID "coincident points"
 * (the reference's ValueError).  The approximation-error oracle at sizes
 * the CPU cannot reach. */
int nesa_dense_matvec(const double* points_dev, const double* q_dev, double* phi_dev, int64_t n,
                      int32_t ncols, void* stream);

/* Multi-GPU halo exchange of partial source amplitudes (
 * the reference has no distributed layer).  Device pointers; s is the
 * (G, qr) amplitude block of nesa_plan_s_dev.  pack: send[r] =
 * s[export_ids[r]] for r < n_export, zero rows up to send_rows.  combine:
 * for each imported group i, s[import_ids[i]] = sum over k of row
 * contrib[i][k] (k ascending, -1 = none) of [recv rows | s rows], a row
 * c < n_recv_rows reading recv[c], c >= n_recv_rows reading s[c - n_recv_rows]
 * (only the group's own row).  Stream-ordered, no synchronisation. */
int nesa_exchange_pack(const void* s_dev, const int64_t* export_ids_dev, int64_t n_export,
                       int64_t send_rows, int32_t qr, int32_t is_f64, void* send_dev, void* stream);
int nesa_exchange_combine(void* s_dev, const void* recv_dev, const int64_t* import_ids_dev,
                          const int64_t* contrib_dev, int64_t n_import, int32_t max_contrib,
                          int64_t n_recv_rows, int32_t qr, int32_t is_f64, void* stream);

/* Native bit-exact quadtree build (reference: build_tree + _fill_lists,
 * quadtree.py:123-245).  points: (n, 2) row-major HOST doubles.  Returns 0,
 * 1 for invalid input (the reference's ValueError; text in
 * nesa_tree_error) or 2; *out is set in every case and must be freed.
 * nesa_tree_size(what): 0 groups, 1 leaves, 2 neighbor entries,
 * 3 interaction entries, 4 l0, 5 L, 6 points.  nesa_tree_copy(field, dst)
 * copies one array into caller memory: 0 level (int32), 1 ix, 2 iy,
 * 3 start, 4 stop, 5 parent, 6 child_first, 7 n_children (int64, per group),
 * 8 box (double, groups x 4), 9 level_first, 10 level_count (int64, index
 * level - l0), 11 nbr_ptr, 12 nbr_idx, 13 int_ptr, 14 int_idx, 15 perm
 * (int64), 16 origin x, origin y, side (3 doubles). */
typedef struct nesa_tree nesa_tree;
int nesa_tree_build(const double* points, int64_t n, double P, int32_t l0_groups_longest,
                    nesa_tree** out);
const char* nesa_tree_error(nesa_tree* tree);
int64_t nesa_tree_size(nesa_tree* tree, int32_t what);
int nesa_tree_copy(nesa_tree* tree, int32_t field, void* dst);
void nesa_tree_free(nesa_tree* tree);

#ifdef __cplusplus
}
#endif
#endif /* NESA_B200_H */
