/*
 * screenbem_b200 — C ABI of the B200 (sm_100a) hot path of the screenbem
 * reference (arXiv 2310.09204): dense Galerkin assembly of the Laplace
 * hypersingular operator on multiscreens, Schwarz-preconditioned CG.
 *
 * The reference is a header-only C++ library (proj/include/screenbem) with no
 * FFI; each entry point below replaces the reference function cited next to
 * it, with plain pointers and sizes.  The C++ wrappers in
 * include/screenbem/ headers restore the reference's C++ names and exceptions.
 *
 * Conventions
 *   - Every function returns SBG_OK (0) or an error code; sbg_last_error()
 *     gives the message (thread-local).  SBG_EVALIDATION mirrors the
 *     reference's ValidationError (CLI exit 2), SBG_ENUMERICAL its
 *     NumericalError (CLI exit 3) (inc/common.hpp:16-26).
 *   - The caller owns host buffers; opaque handles own host or device memory
 *     and are released with the matching *_destroy.
 *   - One CUDA stream per context; calls on one context must not overlap.
 *   - Dense matrices are exchanged row-major n x n (W is symmetric).
 *   - The GPU path has no CPU fallback: without a usable sm_100a device every
 *     device entry point fails with SBG_ECUDA.
 */
#ifndef SCREENBEM_B200_H
#define SCREENBEM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBG_OK 0
#define SBG_EVALIDATION 2 /* ValidationError (inc/common.hpp:17-20) */
#define SBG_ENUMERICAL 3  /* NumericalError  (inc/common.hpp:23-26) */
#define SBG_ECUDA 4       /* device / runtime failure */
#define SBG_EINTERNAL 5

typedef struct sbg_ctx sbg_ctx;
typedef struct sbg_mesh sbg_mesh;           /* SurfaceMesh      (inc/mesh.hpp:19-83) */
typedef struct sbg_level sbg_level;         /* MeshLevelPair    (inc/mesh.hpp:86-92) */
typedef struct sbg_inflated sbg_inflated;   /* InflatedMesh     (inc/inflate.hpp:48-76) */
typedef struct sbg_matrix sbg_matrix;       /* GalerkinMatrix   (inc/assemble.hpp:12), device-resident */
typedef struct sbg_partition sbg_partition; /* DofPartition     (inc/schwarz.hpp:14-17) */
typedef struct sbg_prolong sbg_prolong;     /* Prolongation     (inc/jump.hpp:87-89) */
typedef struct sbg_prec sbg_prec;           /* SchwarzPreconditioner (inc/schwarz.hpp:55-73), device-resident */
typedef struct sbg_aplan sbg_aplan;         /* assembly plan: mesh-derived device data of assemble_W */

/* QuadratureConfig (inc/quadrature.hpp:12-16).  The far / near tensor rules live in the
 * device's constant memory, written on each assembly's stream: assemblies with different
 * far_order must not run concurrently on one device (different threads / streams). */
typedef struct {
    int far_order;         /* 4 */
    int singular_order;    /* 8 */
    double near_threshold; /* 2.0 */
    int exact_far;         /* 0: fast far field; 1: depth-0 far pairs bitwise like the CPU
                              restatement (IEEE sqrt/division, no FMA, sequential order) */
} sbg_quad_cfg;

/* PcgReport (inc/pcg.hpp:9-16) */
typedef struct {
    int iterations;
    int converged;
    double kappa_estimate;
    int history_len; /* iterations + 1 residual norms */
} sbg_pcg_report;

/* SpectrumResult (inc/schwarz.hpp:150-154) + Lanczos bookkeeping */
typedef struct {
    double lambda_min, lambda_max, kappa;
    int iterations; /* CG / PCG steps of the Lanczos process */
    int converged;  /* the CG residual reached tol */
} sbg_spectrum;

/* assembly work counters (roofline bookkeeping) */
typedef struct {
    long long far_pairs, near_pairs, identical, edge, vertex, near_leaves, tiles, tiles_skipped;
    long long h2d_bytes; /* host-to-device bytes of the plan build (mesh data, curl lists, tiles) */
} sbg_assembly_stats;

const char* sbg_last_error(void);
const char* sbg_version(void);

/* ---- device context ---------------------------------------------------- */
int sbg_ctx_create(int device, sbg_ctx** out);
void sbg_ctx_destroy(sbg_ctx* ctx);
int sbg_ctx_synchronize(sbg_ctx* ctx);
/* matrix-vector form of sbg_matvec / sbg_pcg / the Lanczos path on this context (no
 * reference counterpart: the reference's W * p is Eigen's dense product, pcg.hpp:70):
 *   0 (default) symmetric — W is symmetric by construction (assemble.hpp:136-137), so for
 *     n >= 2048 only its upper triangle is read, half the bytes;
 *   1 full-matrix — every entry read; the row kernel shared with sbg_pcg_rows, whose
 *     results then equal sbg_pcg's bitwise. */
int sbg_ctx_set_matvec_form(sbg_ctx* ctx, int form);
int sbg_ctx_get_matvec_form(sbg_ctx* ctx, int* form);
int sbg_device_name(int device, char* buf, int cap, int* sm_count);
/* named CUDA-event timers on the context stream */
int sbg_timers_enable(sbg_ctx* ctx, int on);
int sbg_timers_reset(sbg_ctx* ctx);
int sbg_timer_get(sbg_ctx* ctx, const char* name, double* total_ms, long long* count);
/* user intervals on the same timer set (CUDA events on the context stream) */
int sbg_timer_begin(sbg_ctx* ctx, const char* name);
int sbg_timer_end(sbg_ctx* ctx);
/* kernels launched by this library so far (all contexts) */
long long sbg_launch_count(void);

/* ---- meshes (host) ------------------------------------------------------ */
int sbg_mesh_create(int nv, const double* verts, int nf, const int32_t* facets, sbg_mesh** out);
void sbg_mesh_destroy(sbg_mesh* m);
int sbg_mesh_sizes(const sbg_mesh* m, int* nv, int* nf);
int sbg_mesh_export(const sbg_mesh* m, double* verts, int32_t* facets);
int sbg_validate_mesh(const sbg_mesh* m);                     /* inc/mesh.hpp:238-272 */
int sbg_make_builtin(const char* spec, sbg_mesh** out);        /* inc/mesh.hpp:516-537 ("bowtie[:k]") */
int sbg_refine_uniform_times(const sbg_mesh* m, int k, sbg_level** out); /* inc/mesh.hpp:388-405 */
int sbg_level_create(const sbg_mesh* coarse, const sbg_mesh* fine, const int32_t* parent, sbg_level** out);
int sbg_make_config(int cfg, int ratio, sbg_level** out);      /* BASELINE.json configs 1-5 (ratio 0 = default H/h) */
int sbg_make_panels(int kind, int m, int r, sbg_level** out);  /* 0 flat, 1 T-junction, 2 triple cross */
/* Neumann field g of a BASELINE config: constant, or for cfg 2 / 4 the unit vector of three
 * std::normal_distribution<double> draws from std::mt19937(seed 1 / 7) (tests/test_pcg.cpp:14-15) */
int sbg_config_g(int cfg, double* g3);
int sbg_level_mesh(const sbg_level* l, int fine, sbg_mesh** out); /* copy of the coarse (0) / fine (1) mesh */
int sbg_level_parent(const sbg_level* l, int32_t* parent);
int sbg_level_sizes(const sbg_level* l, double* H, double* h);
void sbg_level_destroy(sbg_level* l);

/* ---- inflation / DOF numbering (host) ------------------------------------ */
int sbg_inflate(const sbg_mesh* m, int validate, sbg_inflated** out); /* inc/inflate.hpp:98-288 */
void sbg_inflated_destroy(sbg_inflated* im);
int sbg_inflated_sizes(const sbg_inflated* im, int* n_dofs, int* n_gvertices, int* nv, int* nf);
/* q[nv], gv_first[nv], dof_first[nv], ofacet_branch[2nf*3], jump_dofs[2n], normals[2nf*3] (nullable) */
int sbg_inflated_export(const sbg_inflated* im, int32_t* q, int32_t* gv_first, int32_t* dof_first,
                        int32_t* ofacet_branch, int32_t* jump_dofs, double* normals);

/* ---- Galerkin matrix (device) -------------------------------------------- */
/* assemble_W (inc/assemble.hpp:72-139); `workers` is accepted and ignored */
int sbg_assemble_w(sbg_ctx* ctx, const sbg_inflated* im, const sbg_quad_cfg* cfg, int workers, sbg_matrix** out,
                   sbg_assembly_stats* stats);
/* assemble_W with the host copy the reference returns (inc/assemble.hpp:72-139 returns W by
 * value): also fills host_w (n x n row-major doubles).  A page-locked host_w (sbg_host_alloc,
 * cudaHostRegister) gets the device-to-host copy overlapped with the near field (the far
 * part of W streams out while the near pairs are integrated, then only the band of entries
 * they touched is copied again); any other buffer is filled after the assembly. */
int sbg_assemble_w_host(sbg_ctx* ctx, const sbg_inflated* im, const sbg_quad_cfg* cfg, int workers, double* host_w,
                        sbg_matrix** out, sbg_assembly_stats* stats);
/* the same split in two: host preparation of one mesh (facet blocks, curl lists,
 * singular lists, rules, uploaded once) and the device-only assembly, which
 * (re)fills *W (allocated on first use) */
int sbg_assembly_plan_create(sbg_ctx* ctx, const sbg_inflated* im, const sbg_quad_cfg* cfg, sbg_aplan** out);
int sbg_assembly_run(sbg_aplan* plan, sbg_matrix** W, sbg_assembly_stats* stats);
/* one shard (rank of world) of sbg_assembly_run for multi-GPU assembly of one W:
 * far tiles k with k % world == rank, the near pairs whose pair hash maps to
 * rank, and a contiguous 1/world of each singular class; stats count the shard's
 * own work (far_pairs = -1); the world shards' W sum entrywise to the full W (the
 * caller reduces them, e.g. an NCCL all-reduce over sbg_matrix_device_view).
 * The reference's per-worker partial W + sum (inc/assemble.hpp:91-133), across processes. */
int sbg_assembly_run_shard(sbg_aplan* plan, sbg_matrix** W, int rank, int world, sbg_assembly_stats* stats);
void sbg_assembly_plan_destroy(sbg_aplan* plan);
int sbg_matrix_create(sbg_ctx* ctx, int n, const double* host_rowmajor, sbg_matrix** out);
int sbg_matrix_n(const sbg_matrix* W);
/* device storage of W: row-major n x ld doubles (ld >= n, padding zero), count = n * ld */
int sbg_matrix_device_view(const sbg_matrix* W, void** data, int* ld, long long* count);
/* the upper triangle of the symmetric W as one contiguous device vector of n (n + 1) / 2
 * doubles (row i at i n - i (i - 1) / 2, columns i..n-1), and back (writing both triangles):
 * a multi-GPU reduction of the shards' W moves half the bytes.  Enqueued on W's context
 * stream, no synchronisation. */
int sbg_matrix_pack_upper(const sbg_matrix* W, double* d_packed);
int sbg_matrix_unpack_upper(sbg_matrix* W, const double* d_packed);
int sbg_matrix_download(const sbg_matrix* W, double* host_rowmajor);
int sbg_matrix_download_rows(const sbg_matrix* W, const int32_t* rows, int nrows, double* host);
int sbg_matrix_symmetry_defect(const sbg_matrix* W, double* max_abs);
int sbg_matvec(sbg_ctx* ctx, const sbg_matrix* W, const double* x_host, double* y_host);
void sbg_matrix_destroy(sbg_matrix* W);
/* dump_matrix_binary / load_matrix_binary (inc/assemble.hpp:191-226): "SBEMW\0" header */
int sbg_matrix_dump_binary(const sbg_matrix* W, const char* path);
int sbg_matrix_load_binary(sbg_ctx* ctx, const char* path, sbg_matrix** out);

/* pair_integral (inc/quadrature.hpp:268-334) on the device for explicit pairs */
int sbg_pair_integrals(sbg_ctx* ctx, const sbg_mesh* m, const sbg_quad_cfg* cfg, const int32_t* f, const int32_t* g,
                       long long npairs, double* out);

/* assemble_rhs (inc/assemble.hpp:143-184): g constant (g_is_field = 0, 3 doubles) or
 * sampled at the nf*16 points of sbg_rhs_points (g_is_field = 1, 3 per point) */
int sbg_rhs_points(const sbg_inflated* im, const sbg_quad_cfg* cfg, double* pts);
int sbg_assemble_rhs(sbg_ctx* ctx, const sbg_inflated* im, const sbg_quad_cfg* cfg, const double* g, int g_is_field,
                     double* L);

/* ---- double-layer potential (inc/potential.hpp, 3-D) ----------------------- */
/* U(x) = sum_t int n_t.(y-x) / (4 pi |x-y|^3) [phi](y) of jump vector v (num_jump_dofs values)
 * at np points (np x 3, host, row-major) into out (np), potential.hpp:104-138: the rule
 * triangle_rule(far_order + 2), split4 subdivision of a facet while the point is closer than
 * its diameter (depth < 24).  cfg->exact_far: every facet in the reference's operation order,
 * bitwise the CPU restatement; else the far facets take the constant-normal form.  A point
 * within 0.5e-6 h of the screen: code 2 (ValidationError, potential.hpp:119-120). */
int sbg_eval_dl(sbg_ctx* ctx, const sbg_inflated* im, const double* v, const double* points, long long np,
                const sbg_quad_cfg* cfg, double* out);
/* potential.hpp:15-25: the nx x ny grid of cell centres of [lo,hi]^2 in the z = 0 plane, points
 * within mask_eps of the mesh dropped (mesh.hpp:121-133 distance_to); out: capacity 3 nx ny
 * doubles, *count = points kept */
int sbg_make_cartesian_grid(sbg_ctx* ctx, const sbg_mesh* mesh, double lo, double hi, int nx, int ny,
                            double mask_eps, double* out, int* count);

/* ---- partition / prolongation (host) ------------------------------------ */
int sbg_partition_dofs(const sbg_level* pair, const sbg_inflated* fine, sbg_partition** out); /* schwarz.hpp:19-51 */
int sbg_partition_create(int nfaces, const int32_t* face_ids, const int32_t* face_ptr, const int32_t* face_dofs,
                         int nwb, const int32_t* wb, sbg_partition** out);
int sbg_partition_sizes(const sbg_partition* p, int* nfaces, int* nface_dofs, int* nwb);
int sbg_partition_export(const sbg_partition* p, int32_t* face_ids, int32_t* face_ptr, int32_t* face_dofs,
                         int32_t* wb);
void sbg_partition_destroy(sbg_partition* p);
int sbg_build_prolongation(const sbg_level* pair, const sbg_inflated* coarse, const sbg_inflated* fine,
                           sbg_prolong** out); /* inc/jump.hpp:118-185 */
int sbg_prolong_create(int rows, int cols, const int32_t* col_ptr, const int32_t* row_idx, const double* val,
                       sbg_prolong** out);
int sbg_prolong_sizes(const sbg_prolong* p, int* rows, int* cols, int* nnz);
int sbg_prolong_export(const sbg_prolong* p, int32_t* col_ptr, int32_t* row_idx, double* val);
void sbg_prolong_destroy(sbg_prolong* p);

/* ---- Schwarz preconditioner (device) -------------------------------------- */
int sbg_build_preconditioner(sbg_ctx* ctx, const sbg_matrix* W, const sbg_partition* part, const sbg_prolong* R,
                             sbg_prec** out); /* inc/schwarz.hpp:100-118 */
/* mode 1 (default): block inverses L^-T L^-1 formed once, apply = one batched GEMV (when the
 * largest block exceeds 2048 DOFs, X = L^-1 is kept instead and the apply is X^T (X r), two
 * triangular GEMVs over the same bytes); mode 2: that factored form always;
 * mode 0: blocked forward/backward triangular solves with L (llt.solve, schwarz.hpp:130) */
int sbg_build_preconditioner_mode(sbg_ctx* ctx, const sbg_matrix* W, const sbg_partition* part, const sbg_prolong* R,
                                  int mode, sbg_prec** out);
int sbg_apply_preconditioner(sbg_ctx* ctx, sbg_prec* p, const double* r_host, int n, double* z_host); /* :121-140 */
int sbg_prec_num_subspaces(const sbg_prec* p);
int sbg_prec_block_diag(sbg_ctx* ctx, sbg_prec* p, int which, double* diag, int* n_out); /* which: face, -1 WB, -2 coarse */
int sbg_coarse_matrix(sbg_ctx* ctx, const sbg_matrix* W, const sbg_prolong* R, double* H);
double sbg_prec_factor_bytes(const sbg_prec* p);
void sbg_prec_destroy(sbg_prec* p);

/* ---- condition numbers (inc/schwarz.hpp:142-190) --------------------------- */
/* materialize_preconditioner (:142-148): the dense n x n M with columns apply(e_j),
 * built on the device from the block inverses and the coarse term */
int sbg_materialize_preconditioner(sbg_ctx* ctx, sbg_prec* p, sbg_matrix** out);
/* a dense SPD matrix M (device) used as the preconditioner, for condition_number(W, M) */
int sbg_prec_from_dense(sbg_ctx* ctx, const sbg_matrix* M, sbg_prec** out);
/* condition_number(W) (:168-172) when p is NULL, condition_number(W, prec) (:174-190)
 * otherwise: extreme eigenvalues by Lanczos on M W in the W inner product (seeded
 * start, full reorthogonalisation) until both extreme Ritz residuals are
 * <= tol |theta|; maxit <= 0: min(n, 1500) steps.  Replaces the dense eigensolve. */
int sbg_condition_number(sbg_ctx* ctx, const sbg_matrix* W, sbg_prec* p, double tol, int maxit, sbg_spectrum* out);

/* ---- PCG (device) --------------------------------------------------------- */
/* pcg (inc/pcg.hpp:33-116); prec nullable.  history/alphas/betas have hist_cap
 * entries (maxit+1 suffices; nullable).  rhs and x are host buffers. */
int sbg_pcg(sbg_ctx* ctx, const sbg_matrix* W, sbg_prec* prec, const double* rhs, int n, double tol, int maxit,
            double* x, double* history, double* alphas, double* betas, int hist_cap, sbg_pcg_report* rep);

/* pcg with the reference's optional exact solution (inc/pcg.hpp:33-35, 48-53, 59, 82):
 * energy[k] = sqrt(max(0, e_k^T W e_k)), e_k = x_k - exact, for k = 0..iterations
 * (history_len entries, as the residual history); one extra matvec per iteration. */
int sbg_pcg_exact(sbg_ctx* ctx, const sbg_matrix* W, sbg_prec* prec, const double* rhs, int n, double tol, int maxit,
                  const double* exact, double* x, double* history, double* energy, double* alphas, double* betas,
                  int hist_cap, sbg_pcg_report* rep);

/* Row-panel PCG for one GPU per rank (the multi-worker counterpart of
 * pcg, inc/pcg.hpp:33-116): W is replicated, this rank computes rows
 * [row_lo, row_hi) of y = W p each iteration, and `exchange` — called on the host
 * thread once per enqueued iteration, after those rows are enqueued on `stream` — must
 * enqueue on that stream the all-gather that fills the other ranks' rows of d_y
 * (e.g. NCCL over NVLink; d_p is the current search direction, for single-process
 * emulation).  Return non-zero to abort.  All other steps (dot products, updates,
 * preconditioner apply) are replicated.  Iterations are enqueued in batches; at each
 * batch boundary the host reads this rank's convergence state.  With `agree` (see
 * sbg_pcg_rows_agree) the stop decision is collective: `agree(user, local_stop,
 * &global_stop)` must return in global_stop the minimum of local_stop over the ranks
 * (e.g. an all-reduce MIN), so every rank enqueues the same exchanges even if its W or
 * rhs differ from the others' in the last bits (fp64 atomics in assembly).  Without it
 * (sbg_pcg_rows) each rank decides alone, which is safe only when W and rhs are bitwise
 * identical on every rank.  rhs/x are device buffers when on_device. */
typedef int (*sbg_exchange_fn)(void* user, const double* d_p, double* d_y, int n, void* stream);
typedef int (*sbg_agree_fn)(void* user, int local_stop, int* global_stop);
int sbg_pcg_rows(sbg_ctx* ctx, const sbg_matrix* W, sbg_prec* prec, const double* rhs, int n, int on_device,
                 double tol, int maxit, int row_lo, int row_hi, sbg_exchange_fn exchange, void* user, double* x,
                 double* history, double* alphas, double* betas, int hist_cap, sbg_pcg_report* rep);
int sbg_pcg_rows_agree(sbg_ctx* ctx, const sbg_matrix* W, sbg_prec* prec, const double* rhs, int n, int on_device,
                       double tol, int maxit, int row_lo, int row_hi, sbg_exchange_fn exchange, sbg_agree_fn agree,
                       void* user, double* x, double* history, double* alphas, double* betas, int hist_cap,
                       sbg_pcg_report* rep);
/* d_y[lo:hi] = W[lo:hi, :] d_x, enqueued on the context stream (no synchronisation).
 * d_x: n doubles, any alignment (copied into a zero-padded context scratch vector). */
int sbg_matvec_rows_device(sbg_ctx* ctx, const sbg_matrix* W, const double* d_x, double* d_y, int row_lo, int row_hi);
/* the context's CUDA stream (cudaStream_t), for enqueuing collectives in order with it */
int sbg_ctx_stream(sbg_ctx* ctx, void** stream);

/* ---- device-resident benchmarking helpers (inputs already in HBM) --------- */
int sbg_device_alloc(sbg_ctx* ctx, long long bytes, void** dptr);
int sbg_device_free(void* dptr);
/* page-locked host memory: sbg_matrix_download into it is one pitched DMA (no staging copy) */
int sbg_host_alloc(long long bytes, void** hptr);
int sbg_host_free(void* hptr);
int sbg_memcpy_h2d(sbg_ctx* ctx, void* dst, const void* src, long long bytes);
int sbg_memcpy_d2h(sbg_ctx* ctx, void* dst, const void* src, long long bytes);
int sbg_pcg_device(sbg_ctx* ctx, const sbg_matrix* W, sbg_prec* prec, const double* d_rhs, double tol, int maxit,
                   double* d_x, sbg_pcg_report* rep);
/* y = W x repeated `reps` times on device vectors; per-launch time via timers ("gemv_f64").
 * d_x: n doubles, any alignment (copied into a zero-padded context scratch vector). */
int sbg_matvec_device(sbg_ctx* ctx, const sbg_matrix* W, const double* d_x, double* d_y, int reps);
/* algorithmic DRAM bytes of one matvec on this context's form (roofline bookkeeping): the
 * entries read (8 n^2 full; the upper triangle and its diagonal blocks symmetric), x, y and
 * the symmetric form's partial sums */
int sbg_matvec_bytes(sbg_ctx* ctx, const sbg_matrix* W, double* bytes);
int sbg_apply_preconditioner_device(sbg_ctx* ctx, sbg_prec* p, const double* d_r, double* d_z, int reps);
/* write a buffer larger than L2 (L2 flush between timed iterations) */
int sbg_l2_flush(sbg_ctx* ctx);
int sbg_pool_stats(sbg_ctx* ctx, long long* reserved, long long* used); /* device memory pool, bytes */
/* measured DFMA throughput of this device (TFLOP/s), the FP64 roofline denominator */
int sbg_fp64_peak(sbg_ctx* ctx, double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* SCREENBEM_B200_H */
