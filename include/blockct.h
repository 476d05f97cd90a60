/*
 * blockct.h -- C ABI of the B200-native block row/column gradient solver
 * (CSGD/GCSGD, arXiv 1709.00953).  libblockct_cuda.so implements it with
 * hand-written sm_100a kernels; there is no CPU fallback.
 *
 * The reference package `blockct` (pure Python + numba) exposes this path at
 * four nested levels.  Each entry point below names the
 * reference interface it replaces:
 *
 *   bct_create / bct_create_parallel_beam
 *       <- BlockSystem.build/_assemble, projector.py:541-626 (cached store:
 *          per-panel CSR over hit rows, rbp, l2g) + the parallel-beam harness
 *          of SURVEY §8c.  The device additionally builds a per-panel CSC
 *          ("transposed panel") with per-(column,row-block) segment pointers
 *          so A_I^T r needs no atomics.
 *   bct_create_scan
 *       <- BlockSystem.build(geometry, partition, table) for any ScanGeometry
 *          (fan / cone beam), projector.py:541-626 with _trace_ray_kernel
 *          (projector.py:51-198) run on the device.
 *   bct_run_epoch
 *       <- EpochExecutor.run_epoch, executor.py:225-253, with the numba
 *          kernel _run_tasks (executor.py:42-102), commit_task/_commit_kernel
 *          (projector.py:723-740, 247-255), the refresh (executor.py:215-223,
 *          projector.py:742-754) and, with BCT_COMMIT, _commit_epoch
 *          (solvers.py:180-185).  Plan layout = the `loops` argument.
 *   bct_sample_epoch
 *       <- BlockScheduler.epoch_plan, sampling.py:140-152 (selection from
 *          host-drawn numpy variates; the device computes keys, stable
 *          top-k, chunking and beta = _group_beta, solvers.py:173-177).
 *   bct_set_* / bct_get_*   <- SolverState fields (solvers.py:50-82)
 *   bct_fill_z_from_image   <- BlockSystem.fill_z_from_image (projector.py:756-765)
 *   bct_projection_sum      <- BlockSystem.projection_sum (projector.py:767-777)
 *   bct_forward             <- BlockSystem.forward (projector.py:692-702)
 *   bct_audit               <- audit_state (solvers.py:154-166)
 *
 * Conventions: every function returns 0 on success and a negative code on
 * failure; bct_last_error() describes the last failure of a context (or of
 * context creation when ctx is NULL).  All array arguments are HOST pointers
 * unless the name says `dev`.  Vectors are in the reference's global order
 * (voxel ids, measurement ids); the library permutes to its panel-major
 * device layout.  One context = one device = one CUDA stream; contexts are
 * not thread-safe.
 */
#ifndef BLOCKCT_H
#define BLOCKCT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bct_ctx bct_ctx;

enum { BCT_OK = 0, BCT_EINVAL = -1, BCT_ECUDA = -2, BCT_ENOMEM = -3, BCT_ESCHEDULE = -4 };
enum { BCT_F64 = 0, BCT_F32 = 1 };                          /* value storage */
enum { BCT_SERIAL_FAITHFUL = 0, BCT_PARALLEL = 1 };         /* executor.py:37 */
/* whole-system baselines (solvers.py:283-379): sweep kind and scaling rule */
enum { BCT_ROW_ACTION = 0, BCT_COLUMN_ACTION = 1 };
enum { BCT_M_IDENTITY = 0, BCT_M_SUM_INVERSE = 1, BCT_M_NORM_INVERSE = 2 };   /* M_RULES */
enum { BCT_COMMIT = 1, BCT_METRICS = 2, BCT_SHARDED = 4,   /* bct_run_epoch flags */
       BCT_GUARD = 8, BCT_GUARD_REF = 16 };                 /* divergence guard    */
enum { BCT_IMPORTANCE = 0, BCT_RANDOM = 1, BCT_MIXED = 2 }; /* sampling.py:25 */

/* One column panel A_:j in the reference's cached layout (projector.py:474-488). */
typedef struct {
    int64_t n_rows;           /* hit rows of the panel                      */
    int64_t nnz;
    const double *data;       /* [nnz] intersection lengths                 */
    const int32_t *cols;      /* [nnz] local column ids, ascending per row  */
    const int64_t *indptr;    /* [n_rows+1]                                 */
    const int64_t *rbp;       /* [m+1] row-block ranges over local rows     */
    const int64_t *l2g;       /* [n_rows] global measurement ids            */
} bct_panel;

/* Partition, probability table and placement (geometry.py:442-478, 611-629). */
typedef struct {
    int32_t m;                      /* row (measurement) blocks, <= 256     */
    int32_t n_panels;               /* column (voxel) blocks, global count  */
    int64_t n_meas;
    int64_t n_vox;
    const int64_t *row_block_ptr;   /* [m+1]                                */
    const int64_t *row_block_rows;  /* measurement ids of each row block    */
    const int64_t *col_block_ptr;   /* [n_panels+1]                         */
    const int64_t *col_block_vox;   /* voxel ids of each column block       */
    const double *table_values;     /* [m*n_panels], values[i*n_panels+j]   */
    const double *table_totals;     /* [n_panels]                           */
    int32_t panel_begin;            /* panels owned by this context:        */
    int32_t panel_end;              /*   [panel_begin, panel_end)           */
    int32_t dtype;                  /* BCT_F64 | BCT_F32                    */
    int32_t device;                 /* CUDA device ordinal                  */
} bct_system_desc;

/* Parallel-beam strip geometry of SURVEY §8c, traced on the device. */
typedef struct {
    int64_t n, views, bins;
    int32_t m, nc;
    const double *cos_views;        /* [views] numpy cos(pi*a/views)        */
    const double *sin_views;        /* [views]                              */
    int32_t panel_begin, panel_end;
    int32_t dtype;
    int32_t device;
} bct_pb_desc;

/* General scan (fan / cone beam, any pose list) traced on the device:
 * geometry.py:42-312 (grid, flat detector, poses) and the blocked store of
 * projector.py:563-626.  The partition and the silhouette probability table
 * (geometry.py:586-672) come from the host (paper_1709_00953_b200/scan.py). */
typedef struct {
    int64_t dims[3];                /* voxel grid; a 2D grid has dims[2]=1  */
    double voxel_size[3];
    double origin[3];               /* low corner of voxel (0,0,0)          */
    int64_t det_nu, det_nv;         /* pixel g = view*nu*nv + iv*nu + iu    */
    double det_du, det_dv;
    int64_t n_views;
    const double *poses;            /* [n_views*12]: source, detector centre,
                                       det_u, det_v                         */
    int32_t m;                      /* row blocks, <= 256                   */
    int32_t n_panels;               /* column blocks (voxel boxes)          */
    const int64_t *row_block_ptr;   /* [m+1]                                */
    const int64_t *row_block_rows;  /* measurement ids of each row block    */
    const int64_t *box_lo;          /* [n_panels*3] voxel index bounds      */
    const int64_t *box_hi;
    const double *table_values;     /* [m*n_panels]                         */
    const double *table_totals;     /* [n_panels]                           */
    int32_t panel_begin, panel_end;
    int32_t dtype;
    int32_t device;
} bct_scan_desc;

typedef struct {
    int64_t n_tasks;
    int64_t n_visits;
    int64_t n_degenerate;           /* tasks with status != 0               */
    double resid_sq;    /* ||y - sum_j z^j||^2 (this context's rows)        */
    double x_sq;        /* ||x||^2 over owned voxels (after commit)         */
    double err_sq;      /* ||x_true - x||^2 over owned voxels, NaN if unset */
    double kernel_ms;   /* device time of the epoch kernel (CUDA events)    */
} bct_epoch_result;

const char *bct_last_error(const bct_ctx *ctx);
int bct_version(void);

int bct_create(const bct_system_desc *desc, const bct_panel *panels, bct_ctx **out);
int bct_create_parallel_beam(const bct_pb_desc *desc, bct_ctx **out);
/* Errors: BCT_EINVAL for a degenerate ray or a source inside a voxel box
 * (projector.py:278-284, 591-592: GeometryError in the reference). */
int bct_create_scan(const bct_scan_desc *desc, bct_ctx **out);
int bct_destroy(bct_ctx *ctx);

/* Sizes: n_meas, n_vox, m, n_panels, owned range, nnz (owned), z length. */
int bct_info(const bct_ctx *ctx, int64_t *out8);
int bct_panel_info(const bct_ctx *ctx, int32_t j, int64_t *n_rows, int64_t *nnz,
                   int64_t *n_cols);
/* The panel in the reference's cached layout (projector.py:474-488); any
 * output may be NULL; with data, cols and indptr all NULL only the row maps
 * (rbp, l2g) are produced, without merging the stored entries. */
int bct_get_panel(bct_ctx *ctx, int32_t j, double *data, int32_t *cols, int64_t *indptr,
                  int64_t *rbp, int64_t *l2g);
int bct_get_table(bct_ctx *ctx, double *values, double *totals);
/* CUDA stream of the context (cudaStream_t). */
int bct_get_stream(bct_ctx *ctx, void **stream);

/* State (solvers.py:50-82), global order. */
int bct_set_y(bct_ctx *ctx, const double *y);
int bct_set_x(bct_ctx *ctx, const double *x);
int bct_get_x(bct_ctx *ctx, double *x);
int bct_set_r(bct_ctx *ctx, const double *r);
int bct_get_r(bct_ctx *ctx, double *r);
int bct_set_z(bct_ctx *ctx, int32_t j, const double *z_j);   /* [n_rows(j)] */
int bct_get_z(bct_ctx *ctx, int32_t j, double *z_j);
int bct_get_xhat(bct_ctx *ctx, double *xhat);
int bct_set_x_true(bct_ctx *ctx, const double *x_true);      /* NULL clears */
int bct_reset_accumulators(bct_ctx *ctx);                    /* xhat=0, counts=0 */
/* Cold start on the device: x = 0, z = 0, xhat = 0, counts = 0
 * (SolverState.initialize with x0=None, solvers.py:70-76, without uploads). */
int bct_clear_state(bct_ctx *ctx);
int bct_get_counts(bct_ctx *ctx, int64_t *counts);            /* [n_panels] */

/* _commit_epoch (solvers.py:180-185): x_J = xhat_J / counts[j], reset. */
int bct_commit_epoch(bct_ctx *ctx);
/* r = y - sum_j z^j over all measurements (SolverState.initialize). */
int bct_reset_residual(bct_ctx *ctx);
/* Solver start with x0 = 0 (SolverState.initialize + set_x_true of
 * src/solvers.py:188-230 in one call): y uploaded, x = z = xhat = 0,
 * counts = 0, r = y, x_true uploaded (NULL: none).  Enqueued on the
 * context's stream with no host wait when y and x_true are page-locked: the
 * caller keeps them unchanged until its next synchronising call (an epoch
 * result, a state read). */
int bct_begin_solve(bct_ctx *ctx, const double *y, const double *x_true);

/* z^j = A_:j x_J for owned panels (projector.py:756-765, bitwise order). */
int bct_fill_z_from_image(bct_ctx *ctx);
/* out = sum_j z^j over all measurements (projector.py:767-777). */
int bct_projection_sum(bct_ctx *ctx, double *out);
/* y_out = A x (projector.py:692-702, bitwise order). */
int bct_forward(bct_ctx *ctx, const double *x, double *y_out);
/* max|r - (y - sum z)| / max|y| (solvers.py:154-166). */
int bct_audit(bct_ctx *ctx, double *drift);

/*
 * One epoch of the plan `loops` (executor.py:225-253).  Tasks are listed in
 * execution order: task_j[k] the column block, task_visit[k] a visit id
 * (consecutive tasks with the same id form one volume-block visit, sharing
 * the visit-start x_J snapshot and, in serial mode, one refresh), the group
 * sel[task_gptr[k]:task_gptr[k+1]] (row-block ids in draw order) and betas[k].
 * Asynchronous; results via bct_wait_epoch.  Flags: BCT_COMMIT applies
 * _commit_epoch afterwards, BCT_METRICS fills the result norms,
 * BCT_SHARDED writes partial projection sums to the exchange buffer instead
 * of refreshing r (finish with bct_finish_sharded after an all-reduce).
 * Divergence guard (solvers.py:251-258, for pipelined drivers that submit
 * epoch e+1 before reading epoch e): BCT_GUARD_REF (with BCT_COMMIT) records
 * max(|x|, 1e-12) after the epoch as the reference norm; BCT_GUARD makes the
 * epoch a no-op when the previous epoch left |x| non-finite or above
 * factor * reference (bct_set_divergence_factor), so the state stays at the
 * diverged epoch like the reference's when it raises DivergenceError.
 * Invalid plans fail with BCT_ESCHEDULE before any device state changes.
 */
int bct_run_epoch(bct_ctx *ctx, int32_t mode, int64_t n_tasks, const int32_t *task_j,
                  const int32_t *task_visit, const int64_t *task_gptr, const int64_t *sel,
                  const double *betas, int32_t flags);

/*
 * Device-side selection (sampling.py:80-157): visit_j[v] are the visited
 * column blocks in draw order (rng.choice on the host), exp_variates the
 * host rng.exponential stream consumed in visit order (scope_n(j) values per
 * visit), draws[v] the per-visit draw count.  Weights follow the strategy
 * (mixed_weights with theta); betas = b * sum(values[ids,j]) / totals[j]
 * with numpy's pairwise summation.  Builds the device plan and runs the
 * epoch like bct_run_epoch.  plan_ids_out (optional, host) receives the
 * drawn ids per visit in draw order (sum(draws) entries).
 */
int bct_sample_epoch(bct_ctx *ctx, int32_t mode, int32_t n_visits, const int32_t *visit_j,
                     const double *exp_variates, int64_t n_variates, const int32_t *draws,
                     int32_t group_size, double b, int32_t strategy, double theta,
                     int32_t flags, int64_t *plan_ids_out);

/* Factor of the divergence guard (SolverParams.divergence_factor, 1e6). */
int bct_set_divergence_factor(bct_ctx *ctx, double factor);

/* Blocks until the last epoch finished; mus/statuses optional [n_tasks]. */
int bct_wait_epoch(bct_ctx *ctx, bct_epoch_result *out, double *mus, int32_t *statuses);

/* Sharded parallel mode: the device exchange buffer holds
 * n_meas partial projection sums followed by x_sq and err_sq. */
int bct_exchange_buffer(bct_ctx *ctx, double **dev_ptr, int64_t *len);
/* Profiling only: per-block phase timestamps of the last epoch when the
 * environment sets BCT_TIMELINE=1 ([2][task][8][grid] globaltimer ns: phase
 * marks, then per-task sub-phase marks; out holds 16 * n_tasks * grid). */
int bct_debug_timeline(bct_ctx *ctx, long long *out, int64_t n_tasks, int32_t *grid);
/* After the all-reduce of the exchange buffer (enqueued on the context's
 * stream): r = y - S on the drawn rows; the last epoch's result (bct_wait_epoch)
 * then holds the global |y - S|^2, |x|^2, |x_t - x|^2.  Asynchronous when
 * resid_sq is NULL, else it synchronises and returns |y - S|^2.  flags: the
 * epoch's BCT_GUARD / BCT_GUARD_REF (the guard acts on the global |x|). */
int bct_finish_sharded(bct_ctx *ctx, int32_t flags, double *resid_sq);

/*
 * Whole-system cyclic baselines, replacing run_row_action /
 * run_column_action (solvers.py:317-379) on the context's own A (every panel
 * must be owned).  bct_baseline_init assembles A as a device CSR + CSC in
 * BlockSystem.to_scipy's order (projector.py:779-793) on first use, computes
 * the scaling (rows for BCT_ROW_ACTION, columns for BCT_COLUMN_ACTION; m_rule
 * as BaselineParams.m_rule) and resets the baseline state: x = 0 and, for the
 * column action, r = y (bct_set_y first).  bct_baseline_epoch runs one sweep
 * over every block in partition order and returns |y|^2, |y - y_est|^2,
 * |x_t|^2, |x_t - x|^2 (y_est = A x for the row action, y - r for the column
 * action; the x_t terms are NaN without bct_set_x_true).  bct_baseline_get_x
 * copies x out in global voxel order.  Results are bitwise equal to the
 * reference's scipy sweeps.  The GCSGD state (x, r, z) is not touched.
 */
int bct_baseline_init(bct_ctx *ctx, int32_t kind, int32_t m_rule);
int bct_baseline_epoch(bct_ctx *ctx, double omega, double *norms4);
int bct_baseline_get_x(bct_ctx *ctx, double *x);

#ifdef __cplusplus
}
#endif
#endif /* BLOCKCT_H */
