// Internal layout of libblockct_cuda.so (not part of the C ABI).
//
// HBM layout per context (owned panels lp = 0..P-1, global id j = begin+lp):
//   forward CSR  vals[T] / cols[i32] / indptr[i32, panel-relative]     (nnz, rows+1)
//   CSC panel    tvals[T] / trows[i32 global measurement id]            (nnz)
//                cptr[i32] = (|J|) x (m+1) segment starts per (column, row block)
//   rbp[i32]     (m+1) per panel;  l2g[i32] per local row
//   z store      f64, panel-major over local rows (the reference's z list)
//   x, xhat      f64, panel-major over the panel's voxels (x_J contiguous)
//   y, r         f64, global measurement order (replicated across ranks)
//   inverse map  inv_ptr[n_meas+1] / inv_z[i32 flat z offset], panel-ascending
//   row blocks   rb_ptr[m+1] / rb_rows / rb_of_row[n_meas]
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <string>
#include <vector>

// Row-block sets are bitsets of mask_words(m) 64-bit words in a per-epoch
// device array (EpochParams::masks): the epoch's drawn blocks first, then per
// task its group and its visit's union.  m is bounded by the 12 bits the
// layout's band keys give the row block (layout.cu band_key_k).
#define BCT_MAX_M 4096
__host__ __device__ __forceinline__ int mask_words(int m) { return (m + 63) >> 6; }

// One owned column panel in HBM (see layout.cu for the design).
struct PanelDev {
    // forward store: SELL-32 slices of (row, super tile) segments (phase 2)
    const void *fvals;         // T; vector k of lane l of slice s at slice_start[s] + (k*32+l)*4
    const uint16_t *fidx;      // voxel index inside the slice's super tile
    const int32_t *slice_start;// [n_slices+1] entry offset of each slice
    const int32_t *sl_seg;     // [n_slices*32] segment of each lane (-1: empty)
    const int32_t *stbs;       // [n_st*(m+1)] first slice of (tile, row block >= i)
    const int32_t *st_ptr;     // [n_st+1] device voxel range of each super tile
    const int32_t *seg_key;    // tile * n_rows + local row
    const int32_t *seg_len;    // entries of each segment
    const int32_t *seg_slice;  // slice / lane holding each segment
    const int32_t *seg_lane;
    const int32_t *rseg_ptr;   // [n_rows+1] row -> its segments (tile order) in rseg
    const int32_t *rseg;
    const int32_t *rpos;       // [n_seg] SELL position (slice*32+lane) of rseg's segments:
                               // where the epoch kernel stores each segment's partial
    // panel CSC with tile bands (phase 1): slices of 32 columns of a tile,
    // entry e of lane l of slice s at csl_start[s] + ((e/8)*32 + l)*8 + e%8
    const void *tvals;         // T
    const uint16_t *tloc;      // slot of the entry's row in its tile's band (null when
                               // the delta form below is used)
    const uint8_t *toff;       // delta form: slot = tbase[e / 8] + toff[e] (a lane's 8
    const uint16_t *tbase;     // entries span < 256 slots on strip tiles)
    const int32_t *csl_start;  // [n_cslices+1]
    const int32_t *cptr;       // [n_cols*(m+1)] column-local start of each row block
    const int32_t *corder;     // tile order of device columns, tile_cols per tile
    const int32_t *band_ptr;   // [n_tiles+1] ranges of each tile
    const int2 *band_meta;     // per range: (first measurement id, slot << 16 | length)
    const uint16_t *band_rb;   // row block of each range
    // rows / voxels
    const int32_t *rbp;        // [m+1]
    const int32_t *l2g;        // [n_rows] global measurement ids
    const int32_t *d2c;        // device voxel position -> reference local column
    int64_t row_off;           // rows of the panel in z / t_ax
    int64_t x_off;             // voxels of the panel in x / xhat / x_true / gx order
    int64_t fwd_cap, csc_cap;
    int32_t n_rows, n_cols, nnz, j;
    int32_t n_seg, n_slices, n_st, n_tiles;
    int32_t band_max, st_max;
    int32_t mdiv;              // reference order = (c / mdiv, tile, c) for bitwise merges
    int32_t tile_cols;         // columns per phase-1 tile (multiple of 32)
    int32_t n_cslices;
    int32_t swz_shift;         // phase-2 super tile swizzle (see swz_idx)
    int32_t seg_cap;           // set-up input: max entries per forward segment (0: 64)
    // step-coded voxel indices of the forward store (strip panels; phase B):
    // a segment's entries are stored in walk order, so each entry is its
    // predecessor moved by one of {0, s, w, w + s} (s = +-1 the row step, w =
    // the super tile's row length): 2 bits per entry instead of 16
    const uint32_t *fcode;     // word (slice_start[sl]/16 + 24*sl) + (k/4)*32 + lane holds
                               // vectors k..k+3 of the lane, a byte per vector
    const int32_t *fq0;        // per SELL slot: first voxel (logical) | (s < 0) << 16
    const int32_t *rq;         // per SELL slot: its segment's position in rseg (-1: empty
                               // lane): the batched phase B stores partials in row order
    int32_t st_h;              // set-up input: strip height (0: generic placement)
};

struct TaskDev {
    int32_t lp;        // owned panel index
    int32_t j;         // global column block id
    int32_t flags;     // TASK_* bits
    int32_t visit;
    double beta;
    // epoch-batched parallel path (full-panel tasks): flattened work prefixes
    // and the task's slices of the batch scratch buffers
    int32_t tile_pre, slice_pre, row_pre, vox_pre;   // exclusive prefixes over tasks
    int64_t gx_off;    // (g, x) pairs of the task: gx_batch + gx_off
    int64_t seg_off;   // segment partials: seg_batch + seg_off
    int64_t tax_off;   // (t, ax) per local row: tax_batch + tax_off
    int64_t ent_pre;   // forward-store entries of the tasks before this one
};

enum { TASK_LAST_OF_VISIT = 1, TASK_FIRST_OF_VISIT = 2, TASK_FULL = 4 };  // FULL: every row block

// the masks of task k in EpochParams::masks (after the epoch mask)
__host__ __device__ __forceinline__ int64_t task_mask_off(int64_t k, int mw) { return (1 + 2 * k) * mw; }
__host__ __device__ __forceinline__ int64_t visit_mask_off(int64_t k, int mw) { return (2 + 2 * k) * mw; }

struct EpochHeader {
    int32_t n_tasks;
    int32_t mode;
    int32_t flags;
    int32_t batched;   // 1: parallel epoch of full-panel tasks, phase-by-phase over all tasks
    int32_t n_tiles_total, n_slices_total, n_rows_total, n_vox_total;
    int64_t n_ent_total;             // forward-store entries of the batched tasks
    int32_t host_prep;               // 1: EpochParams::prep holds every task's record
    int32_t r32_valid;               // FP32 mode: r32 == (float)r on every row (every
                                     // writer of r in a launch keeps it so)
    int32_t fuse_tail;               // batched: no phase D; phase C keeps (t, ax) per
                                     // panel row (z in (t, ax) form, EpochParams::zt),
                                     // the tail forms z = ax + mu t where it sums z and
                                     // updates x-hat; the per-panel tables fit in
                                     // dynamic shared memory
    int32_t pad_;
    // divergence guard (solvers.py:251-258): BCT_GUARD_REF records the
    // reference norm max(|x|, 1e-12) after this epoch; BCT_GUARD skips the
    // whole epoch when the previous one left |x| non-finite or above
    // guard_factor * reference, so a pipelined run stops at the diverged
    // epoch's state like the reference
    double guard_factor;
};

// Device-side per-epoch outputs.
struct EpochOut {
    double resid_sq, x_sq, err_sq, pad;
    int32_t n_degenerate;
    int32_t pad2[7];
};

// ---- per-task path set-up (epoch.cu per-task loop; built by api.cu when the
// masks are host-known) ----
// Everything a task of the per-task path needs before phase 1: its TaskDev,
// its panel, the contiguous runs of its row-block mask (with their local row
// ranges and the task's SELL slices per super tile) and its visit's drawn
// row blocks (serial refresh).  Fixed header + int arrays sized by the
// context (PrepDims); each CTA copies a task's record into dynamic shared
// memory.  On the device one thread builds it (sampled epochs: a chain of
// dependent loads); when the host knows the masks (bct_run_epoch) it builds
// every task's with the plan.
struct alignas(16) PrepHdr {
    TaskDev T;
    PanelDev P;
    int32_t n_runs;    // contiguous runs of set bits of the task's mask
    int32_t nst;       // super tiles of the panel
    int32_t full;      // the task covers every row block
    int32_t nvb;       // drawn row blocks of the visit
};
// int arrays after the header: i0, i1, rows0 [rc], pre [rc+1], st_pre [sc+1],
// vb [m], vpre [m+1] (rc = max runs = m/2+1, sc = max super tiles per panel)
struct PrepDims {
    int32_t rc, sc, m, pad_;
    __host__ __device__ int words() const { return 4 * rc + 1 + sc + 1 + 2 * m + 1; }
    __host__ __device__ int64_t bytes() const   // record stride, 16-byte multiple
    {
        return ((int64_t)sizeof(PrepHdr) + 4 * (int64_t)words() + 15) & ~15ll;
    }
};
// views of a record's arrays
struct PrepView {
    PrepHdr *h;
    int *i0, *i1, *rows0, *pre, *st_pre, *vb, *vpre;
    __host__ __device__ PrepView(void *rec, const PrepDims &d)
    {
        h = static_cast<PrepHdr *>(rec);
        int *a = reinterpret_cast<int *>(static_cast<char *>(rec) + sizeof(PrepHdr));
        i0 = a; a += d.rc;
        i1 = a; a += d.rc;
        rows0 = a; a += d.rc;
        pre = a; a += d.rc + 1;
        st_pre = a; a += d.sc + 1;
        vb = a; a += d.m;
        vpre = a;
    }
};

struct EpochParams {
    const PanelDev *panels;
    int32_t n_panels_owned;
    int32_t m;
    int64_t n_meas;
    int64_t z_len;
    int64_t x_len;
    // refresh / metrics
    const int32_t *inv_ptr;
    const int32_t *inv_z;
    const int32_t *invt;       // interleaved inverse map: groups of 32 measurements,
    const int32_t *invt_off;   //   slot s of lane l at invt_off[G] + s*32 + l (-1: none)
    const int32_t *rb_ptr;
    const int32_t *rb_rows;
    const int32_t *rb_of_row;
    // state
    const double *y;
    double *r;
    float *r32;                // FP32 mode: copy of r for the batched phase-A bands
    double *z;
    double *x;
    double *xhat;
    int32_t *counts;           // per owned panel (tasks this epoch)
    const double *x_true;      // panel order, may be null
    // plan
    const EpochHeader *hdr;
    const TaskDev *tasks;
    const uint64_t *masks;     // [mw] epoch's drawn blocks, then per task [mw] group, [mw] visit
    int32_t mw;                // mask words per set
    int32_t prep_smem_off;     // byte offset of the task record in dynamic shared memory
    PrepDims prep_dims;
    // scratch
    double *gx;                // 2 buffers x (2*max_cols) : (g, x_J) interleaved, device order
    int64_t gx_stride;
    double *t_ax;              // (t, ax) interleaved per local row of the widest panel
    double *seg_part;          // (t, ax) partial per segment of the widest panel
    double *gx_batch;          // batched path scratch (see TaskDev offsets)
    double *seg_batch;
    double *tax_batch;
    double *part_task;         // [n_tasks][2][grid] gg / denom partials (batched)
    // z in (t, ax) form (fused batched tail): panel lp's z is ax + mu t from
    // zt[row_off..) with zl_mu / zl_st[lp] while zl_on[lp] (api.cu materialize_z)
    void *zt;
    int32_t *zl_on, *zl_st;
    double *zl_mu;
    int32_t band_cap;          // shared-memory slots per band buffer
    int32_t band_dbuf;         // 1: two band buffers (copy next tile while computing)
    double *part;              // per-block partials: [4][grid]
    double *mus;
    int32_t *statuses;
    EpochOut *out;
    char *res_host;            // the epoch's result block in mapped pinned host memory
                               // [EpochOut | mus | statuses], written by the last block
    double *exchange;          // sharded: n_meas partial sums + 2
    double *guard_ref;         // divergence guard: reference |x| (device scalar)
    unsigned int *bar;         // grid barrier word
    unsigned int *ticket;      // last-block counter
    long long *timeline;       // optional phase timestamps (BCT_TIMELINE=1)
    int64_t tl_tasks;          // tasks per half of the timeline buffer
    const int32_t *cta_split;  // per owned panel [grid+1]: phase-2a slice split (full tasks)
    const char *prep;          // per-task path: host-built records (hdr.host_prep), prep_dims.bytes() apart
};

struct bct_ctx_s;

// divergence guard of the sharded finish (see EpochHeader::guard_factor): the
// previous epoch's global |x|^2 is still in EpochOut when the finish of a
// guarded epoch runs; a diverged predecessor makes the finish a no-op too
struct FinishGuard {
    const double *x_sq_prev;   // EpochOut::x_sq
    double *ref;               // reference |x| (written with set_ref)
    double factor;
    int32_t check, set_ref;
    EpochOut *host_out;        // mapped result block of the epoch (norms written there too)
};
__device__ __forceinline__ bool guard_tripped(const FinishGuard &g)
{
    if (!g.check) return false;
    const double nx = sqrt(*(volatile const double *)g.x_sq_prev);
    return !isfinite(nx) || nx > g.factor * *(volatile const double *)g.ref;
}

// builder / launch helpers implemented in the .cu files
// Position of super-tile voxel q in the staged (g, x) array: the low four bits
// are XORed with the voxel's pseudo-row (q >> shift, shift = log2 of the super
// tile's row length), so the lanes of a slice that read one voxel column of
// consecutive image rows (rays along the strip) hit distinct shared-memory
// bank pairs.  An involution for shift >= 4.
__host__ __device__ __forceinline__ int swz_idx(int q, int shift)
{
    return q ^ ((q >> shift) & 15);
}

// general scan geometry for the device tracer (builder.cu)
struct ScanDev {
    double origin[3], vsize[3];
    int64_t nu, nv;
    double du, dv;
    const double *poses;     // [views * 12]: source, detector centre, det_u, det_v
};
struct Box {
    int64_t lo[3], hi[3];    // voxel index bounds of a column block
};

namespace bct {
constexpr int RES_HEAD_BYTES = 64;   // EpochOut at the start of an epoch's result block

// whole-system baselines (baseline.cu): A as a device CSR and CSC, global
// measurement rows x global voxel columns, in BlockSystem.to_scipy's order
struct BaselineMat {
    int64_t nnz = 0, n_meas = 0, n_vox = 0;
    int64_t *row_ptr = nullptr, *col_ptr = nullptr;
    int32_t *csr_col = nullptr, *csc_row = nullptr;
    double *csr_val = nullptr, *csc_val = nullptr;
};
cudaError_t baseline_build(int dtype, const PanelDev *h_panels, int np, const int32_t *d_gvox,
                           int64_t n_meas, int64_t n_vox, BaselineMat &M, cudaStream_t s);
void baseline_free(BaselineMat &M);
cudaError_t baseline_scale(const BaselineMat &M, int kind, int rule, double *diag, cudaStream_t s);
// (lo, hi): the block's ids as one range [lo, hi) when they form one, else -1
cudaError_t baseline_row_block(const BaselineMat &M, const int32_t *rows, int64_t n_rows, int blk,
                               int32_t g_lo, int32_t g_hi, const int32_t *rb_of_row, double omega,
                               const double *y, const double *mdiag, double *res, double *x,
                               cudaStream_t s);
cudaError_t baseline_col_block(const BaselineMat &M, const int64_t *vox, int64_t n_vox_blk,
                               int blk, int32_t v_lo, int32_t v_hi, const int32_t *cb_of_vox,
                               double omega, const double *ddiag, double *dx, double *x,
                               double *r, cudaStream_t s);
cudaError_t baseline_norms(const BaselineMat &M, const double *y, const double *r, const double *x,
                           const double *x_true, const int32_t *gvox, int64_t x_len, int use_r,
                           double *part, double *out4, cudaStream_t s);

cudaError_t scan_trace_counts(const ScanDev &S, const int32_t *L, int64_t n, const Box &B,
                              int32_t *counts, int32_t *bad, cudaStream_t s);
cudaError_t scan_fill(const ScanDev &S, const int32_t *l2g, const int32_t *indptr, int64_t n_hit,
                      const Box &B, double *data, int32_t *cols, cudaStream_t s);
cudaError_t gather_i32(const int32_t *src, const int32_t *idx, int64_t n, int32_t *dst,
                       cudaStream_t s);

// band ranges start at multiples of this many slots / measurement ids, so a
// range is staged in 16-byte granules of 4 FP32 or 2 FP64 residuals
constexpr int BAND_ALIGN = 4;

// epoch-batched path: at most this many tasks (task tables live in shared memory)
constexpr int MAX_BATCH_TASKS = 256;
// fused batched tail: shared-memory bytes per owned panel (z / x offsets,
// task, (g, x) offset, z form: mu / status)
constexpr int FT_PANEL_BYTES = 36;

// device sampler (sampler.cu)
struct SampleVisit {
    int32_t j, draws;
    int32_t var_off;     // first exponential variate of the visit
    int32_t id_off;      // first drawn id of the visit in the plan record
    int32_t task_base;   // first task of the visit, -1 when another rank owns j
    int32_t pad_;
};
struct SamplerParams {
    const double *values;    // [m * n_panels] table values (row-major, values[i*n+j])
    const double *totals;    // [n_panels]
    int32_t n_panels, m;
    const SampleVisit *visits;
    const double *exp;       // exponential variates, visit order
    int32_t strategy, group_size;
    double theta, b;
    TaskDev *tasks;          // the epoch's device task array (betas written)
    uint64_t *masks;         // EpochParams::masks layout: epoch mask ORed, task masks written
    int32_t mw;
    int32_t *plan_ids;       // drawn ids, visit order, draw order
};
void launch_sampler(const SamplerParams &p, int n_visits, cudaStream_t s, cudaError_t *err);

// phase-1 tile reduction areas in dynamic shared memory (2 x epoch.cu RED_DOUBLES)
// per-task phase 2a: at most this many work units (parts) per SELL slice; the
// segment-partial scratch holds that many partials per slot
#ifndef BCT_TASK_PARTS_MAX
#define BCT_TASK_PARTS_MAX 16
#endif
constexpr int TASK_PARTS_MAX = BCT_TASK_PARTS_MAX;
constexpr size_t PHASE1_RED_BYTES = 2 * 32 * 256 / 8 * 8;
std::string cuda_err(cudaError_t e);
void launch_epoch(const EpochParams &p, int dtype, int grid, int block, size_t smem,
                  cudaStream_t s, cudaError_t *err);
int epoch_grid_size(int dtype, int device, size_t smem, int *block);
size_t epoch_static_smem(int dtype);   // the epoch kernel's static shared arrays
// z in (t, ax) form (EpochParams::zt): bytes per pair, and the pass that
// writes such panels' z out and returns them to the stored form
size_t zt_pair_bytes(int dtype);
cudaError_t z_materialize(int dtype, const PanelDev *panels, int np, const void *zt,
                          const double *mu, const int32_t *st, int32_t *on, double *z,
                          cudaStream_t s);
int layout_panel_v2(int dtype, int m, int32_t n_rows, int32_t n_cols, int64_t nnz,
                    const double *vals64, const int32_t *cols_c, const int32_t *indptr_c,
                    const int32_t *l2g, const int32_t *rbp, const std::vector<int32_t> &c2d_h,
                    const std::vector<int32_t> &st_ptr_h, const std::vector<int32_t> &corder_h,
                    int tile_cols, PanelDev &P, std::vector<void *> &keep, std::string &err,
                    cudaStream_t s);
}
