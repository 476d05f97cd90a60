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

#define BCT_MASKW 4                 // up to 256 row blocks
#define BCT_MAX_M (64 * BCT_MASKW)

// Rows of the forward CSR and columns of the CSC start on 4-entry (16-byte
// for int32/f32) boundaries so the kernels can use 128-bit loads; the
// padding entries are never read as data (lengths mask them).
struct PanelDev {
    int64_t fwd_off;   // first (padded) entry of the panel in vals/cols
    int64_t csc_off;   // first (padded) entry of the panel in tvals/trows
    int64_t row_off;   // first local row of the panel in z/l2g/rlen/scratch; rptr at row_off+lp
    int64_t x_off;     // first voxel of the panel in x/xhat/corder
    int64_t cptr_off;  // start of the (|J|)*(m+1) segment table
    int64_t unit_off;  // first row unit of the panel in urow/uend
    int32_t n_rows;
    int32_t n_cols;
    int32_t nnz;
    int32_t j;         // global column block id
};

struct TaskDev {
    int32_t lp;        // owned panel index
    int32_t j;         // global column block id
    int32_t flags;     // bit0: last task of its visit; bit1: first task of its visit
    int32_t visit;
    double beta;
    uint64_t mask[BCT_MASKW];        // row blocks of the task's group
    uint64_t visit_mask[BCT_MASKW];  // union over the visit (serial refresh set)
};

enum { TASK_LAST_OF_VISIT = 1, TASK_FIRST_OF_VISIT = 2 };

struct EpochHeader {
    int32_t n_tasks;
    int32_t mode;
    int32_t flags;
    int32_t pad;
    uint64_t epoch_mask[BCT_MASKW];  // union of all drawn blocks (parallel refresh)
};

// Device-side per-epoch outputs.
struct EpochOut {
    double resid_sq, x_sq, err_sq, pad;
    int32_t n_degenerate;
    int32_t pad2[7];
};

struct EpochParams {
    // store
    const void *vals;          // double* or float*
    const int32_t *cols;
    const int32_t *rptr;       // padded row starts (panel-relative), n_rows+1 per panel
    const int32_t *rlen;       // true row lengths
    const void *tvals;
    const int32_t *trows;
    const int32_t *cptr;       // absolute (panel-relative) CSC positions per (column, block)
    const int32_t *corder;     // column processing order (2D voxel tiles)
    const uint32_t *vbits;     // row-start bit per 4-entry forward vector (word = fwd_off/128)
    const int32_t *urow;       // row units: [urow[u], uend[u]) whole rows of one row block
    const int32_t *uend;
    const int32_t *ubp;        // (m+1) per panel: units of row block i = [ubp[i], ubp[i+1])
    const int32_t *rbp;
    const PanelDev *panels;
    int32_t n_panels_owned;
    int32_t m;
    int64_t n_meas;
    int64_t z_len;
    int64_t x_len;
    // refresh / metrics
    const int32_t *inv_ptr;
    const int32_t *inv_z;
    const int32_t *rb_ptr;
    const int32_t *rb_rows;
    const int32_t *rb_of_row;
    // state
    const double *y;
    double *r;
    double *z;
    double *x;
    double *xhat;
    int32_t *counts;           // per owned panel (tasks this epoch)
    const double *x_true;      // panel order, may be null
    // plan
    const EpochHeader *hdr;
    const TaskDev *tasks;
    // scratch
    double *gx;                // 2 buffers x (2*max_cols) : (g, x_J) interleaved
    int64_t gx_stride;
    double *t_ax;              // (t, ax) interleaved per local row of the widest panel
    double *part;              // per-block partials: [4][grid]
    double *mus;
    int32_t *statuses;
    EpochOut *out;
    double *exchange;          // sharded: n_meas partial sums + 2
    unsigned int *bar;         // grid barrier word
    unsigned int *ticket;      // last-block counter
    long long *timeline;       // optional phase timestamps (BCT_TIMELINE=1)
};

struct bct_ctx_s;

// builder / launch helpers implemented in the .cu files
namespace bct {
std::string cuda_err(cudaError_t e);
void launch_epoch(const EpochParams &p, int dtype, int grid, int block, cudaStream_t s,
                  cudaError_t *err);
int epoch_grid_size(int dtype, int device, int *block);
}
