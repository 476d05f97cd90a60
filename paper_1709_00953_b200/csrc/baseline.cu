// baseline.cu -- the whole-system cyclic baselines on the device
// (run_row_action / run_column_action, solvers.py:317-379).
//
// The reference assembles A once as a scipy CSR (projector.py:779-793,
// BlockSystem.to_scipy: COO of every panel -> canonical CSR, columns sorted
// within each row) and its CSC, then sweeps:
//   row action, per measurement block I:  x += w * A_I^T (M (y_I - A_I x))
//   column action, per volume block J:    dx = w * (D (A_J^T r)); x_J += dx;
//                                          r -= A_J dx
// with M / D the inverse row / column sums (or sums of squares, or 1).
//
// Here the same CSR and CSC are assembled on the device from the context's
// panels (every stored SELL entry -> (row, global voxel, value), two radix
// sorts), and each sweep is a pair of kernels that reproduce scipy's
// operation order: csr_matvec (a row's entries in column order, from 0.0),
// csc_matvec (each output accumulates its inputs in order, from 0.0),
// separate IEEE multiplies and adds (no contraction), and numpy's pairwise
// np.add.reduceat for the scaling sums (sparse .sum(axis) on the minor axis,
// scipy/_compressed.py _minor_reduce).  Results are bitwise equal to the
// reference on the same A (tests/test_baselines.py).
#include <cstdint>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "../../include/blockct.h"
#include "internal.h"

namespace {

// one thread per (row, super tile) segment: its entries -> COO triplets
__global__ void emit_k(PanelDev P, const int32_t *gvox, const int64_t *seg_off, int64_t base,
                       int64_t n_vox, int64_t n_meas, int f32, uint64_t *key_rc, uint64_t *key_cr,
                       double *val)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= P.n_seg) return;
    const int key = P.seg_key[s];
    const int lr = key % P.n_rows, st = key / P.n_rows;
    const int64_t g = P.l2g[lr];
    const int vb = P.st_ptr[st];
    const int sl = P.seg_slice[s], ln = P.seg_lane[s], len = P.seg_len[s];
    const int64_t s0 = P.slice_start[sl];
    int64_t o = base + seg_off[s];
    for (int e = 0; e < len; ++e, ++o) {
        const int64_t pos = s0 + ((int64_t)(e >> 2) * 32 + ln) * 4 + (e & 3);
        const int64_t col = gvox[P.x_off + vb + swz_idx(P.fidx[pos], P.swz_shift)];
        const double v = f32 ? (double)static_cast<const float *>(P.fvals)[pos]
                             : static_cast<const double *>(P.fvals)[pos];
        key_rc[o] = (uint64_t)g * (uint64_t)n_vox + (uint64_t)col;
        key_cr[o] = (uint64_t)col * (uint64_t)n_meas + (uint64_t)g;
        val[o] = v;
    }
}

// ptr[q] = first sorted key >= q * stride (q in [0, n])
__global__ void ptr_k(const uint64_t *keys, int64_t nnz, uint64_t stride, int64_t n, int64_t *ptr)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q > n) return;
    const uint64_t k = (uint64_t)q * stride;
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < k) lo = mid + 1; else hi = mid;
    }
    ptr[q] = lo;
}

__global__ void minor_k(const uint64_t *keys, int64_t nnz, uint64_t stride, int32_t *minor)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < nnz) minor[e] = (int32_t)(keys[e] % stride);
}

// numpy pairwise_sum (loops_utils.h.src) of a[0..n), stride 1
__device__ double pairwise(const double *a, int64_t n, bool square)
{
    auto at = [&](int64_t i) { return square ? __dmul_rn(a[i], a[i]) : a[i]; };
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, at(i));
        return r;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = at(j);
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], at(i + j));
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, at(i));
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pairwise(a, n2, square), pairwise(a + n2, n - n2, square));
}

// inverse scaling per row (CSR) or column (CSC): np.add.reduceat of the
// (squared) entries = first entry + pairwise sum of the rest; empty -> 0
__global__ void scale_k(const int64_t *ptr, const double *val, int64_t n, int rule, double *out)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    if (rule == BCT_M_IDENTITY) {
        out[q] = 1.0;
        return;
    }
    const int64_t a = ptr[q], b = ptr[q + 1];
    const bool sq = rule == BCT_M_NORM_INVERSE;
    double s = 0.0;
    if (b > a) {
        const double first = sq ? __dmul_rn(val[a], val[a]) : val[a];
        s = __dadd_rn(first, pairwise(val + a + 1, b - a - 1, sq));
    }
    out[q] = s > 0.0 ? __ddiv_rn(1.0, s) : 0.0;
}

// row action, step 1: res[g] = M[g] * (y[g] - (A_I x)[g]) for the block's rows
__global__ void ra_res_k(const int64_t *row_ptr, const int32_t *col, const double *val,
                         const int32_t *rows, int64_t n, const double *y, const double *x,
                         const double *mdiag, double *res)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int g = rows[q];
    double s = 0.0;
    for (int64_t e = row_ptr[g]; e < row_ptr[g + 1]; ++e) s = __dadd_rn(s, __dmul_rn(val[e], x[col[e]]));
    res[g] = __dmul_rn(mdiag[g], __dsub_rn(y[g], s));
}

// row action, step 2: x[c] += w * sum over the block's rows (ascending) of
// A[g, c] res[g]  (csc_matvec of A_I^T: rows of A_I in order, from 0.0)
// First entry in [a, b) of a sorted index list with idx >= key.
__device__ __forceinline__ int64_t lb_idx(const int32_t *idx, int64_t a, int64_t b, int32_t key)
{
    while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (idx[mid] < key) a = mid + 1; else b = mid;
    }
    return a;
}

// (g_lo >= 0: the block's rows are the id range [g_lo, g_hi), so a column's
// entries of the block are one run of its row-sorted list, found by binary
// search -- O(entries of the block) per pass instead of the whole matrix)
__global__ void ra_upd_k(const int64_t *col_ptr, const int32_t *row, const double *val,
                         const int32_t *rb_of_row, int blk, int32_t g_lo, int32_t g_hi,
                         int64_t n_vox, double omega, const double *res, double *x)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_vox) return;
    double s = 0.0;
    if (g_lo >= 0) {
        const int64_t e1 = col_ptr[c + 1];
        for (int64_t e = lb_idx(row, col_ptr[c], e1, g_lo); e < e1 && row[e] < g_hi; ++e)
            s = __dadd_rn(s, __dmul_rn(val[e], res[row[e]]));
    } else {
        for (int64_t e = col_ptr[c]; e < col_ptr[c + 1]; ++e) {
            const int g = row[e];
            if (rb_of_row[g] == blk) s = __dadd_rn(s, __dmul_rn(val[e], res[g]));
        }
    }
    x[c] = __dadd_rn(x[c], __dmul_rn(omega, s));
}

// column action, step 1 (per voxel of block J, in order): dx = w * (D g),
// g = the column's entries against r (csr_matvec of A_J^T); x_J += dx
__global__ void ca_dx_k(const int64_t *col_ptr, const int32_t *row, const double *val,
                        const int64_t *vox, int64_t n, double omega, const double *ddiag,
                        const double *r, double *x, double *dx)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int64_t c = vox[q];
    double s = 0.0;
    for (int64_t e = col_ptr[c]; e < col_ptr[c + 1]; ++e) s = __dadd_rn(s, __dmul_rn(val[e], r[row[e]]));
    const double d = __dmul_rn(omega, __dmul_rn(ddiag[c], s));
    dx[c] = d;
    x[c] = __dadd_rn(x[c], d);
}

// column action, step 2: r[g] -= sum over the row's entries in block J
// (column order, from 0.0) of A[g, c] dx[c]  (csc_matvec of A_J)
// (v_lo >= 0: the block's voxels are the id range [v_lo, v_hi): one run of
// each row's column-sorted list, by binary search)
__global__ void ca_res_k(const int64_t *row_ptr, const int32_t *col, const double *val,
                         const int32_t *cb_of_vox, int blk, int32_t v_lo, int32_t v_hi,
                         int64_t n_meas, const double *dx, double *r)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_meas) return;
    double s = 0.0;
    if (v_lo >= 0) {
        const int64_t e1 = row_ptr[g + 1];
        for (int64_t e = lb_idx(col, row_ptr[g], e1, v_lo); e < e1 && col[e] < v_hi; ++e)
            s = __dadd_rn(s, __dmul_rn(val[e], dx[col[e]]));
    } else {
        for (int64_t e = row_ptr[g]; e < row_ptr[g + 1]; ++e) {
            const int c = col[e];
            if (cb_of_vox[c] == blk) s = __dadd_rn(s, __dmul_rn(val[e], dx[c]));
        }
    }
    r[g] = __dsub_rn(r[g], s);
}

// y_est = A x (csr_matvec) or y - r; per-block sums of squares of y and
// y - y_est, and (device-order x_true against the global-order x) of x_true
// and x_true - x.  Fixed-order per-block partials, reduced by baseline_norms.
__global__ void norms_k(const int64_t *row_ptr, const int32_t *col, const double *val,
                        int64_t n_meas, const double *y, const double *r, const double *x,
                        const double *x_true, const int32_t *gvox, int64_t n_vox, int use_r,
                        double *part)
{
    __shared__ double sh[4][256];
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_meas; g += stride) {
        double est;
        if (use_r) {
            est = __dsub_rn(y[g], r[g]);
        } else {
            est = 0.0;
            for (int64_t e = row_ptr[g]; e < row_ptr[g + 1]; ++e)
                est = __dadd_rn(est, __dmul_rn(val[e], x[col[e]]));
        }
        const double d = __dsub_rn(y[g], est);
        a[0] = fma(y[g], y[g], a[0]);
        a[1] = fma(d, d, a[1]);
    }
    if (x_true)
        for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n_vox; v += stride) {
            const double t = x_true[v], d = __dsub_rn(t, x[gvox[v]]);
            a[2] = fma(t, t, a[2]);
            a[3] = fma(d, d, a[3]);
        }
    for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] = a[k];
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w)
            for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < 4) part[blockIdx.x * 4 + threadIdx.x] = sh[threadIdx.x][0];
}

__global__ void norms_fin_k(const double *part, int nb, double *out)
{
    if (threadIdx.x < 4) {
        double s = 0.0;
        for (int b = 0; b < nb; ++b) s += part[b * 4 + threadIdx.x];
        out[threadIdx.x] = s;
    }
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

namespace bct {

cudaError_t baseline_build(int dtype, const PanelDev *h_panels, int np, const int32_t *d_gvox,
                           int64_t n_meas, int64_t n_vox, BaselineMat &M, cudaStream_t s)
{
    int64_t nnz = 0;
    for (int lp = 0; lp < np; ++lp) nnz += h_panels[lp].nnz;
    M.nnz = nnz;
    M.n_meas = n_meas;
    M.n_vox = n_vox;
    const int64_t nz = nnz > 0 ? nnz : 1;
    uint64_t *krc = nullptr, *kcr = nullptr, *k2 = nullptr;
    double *v0 = nullptr;
    int64_t *seg_off = nullptr;
    int64_t max_seg = 1;
    for (int lp = 0; lp < np; ++lp) max_seg = std::max<int64_t>(max_seg, h_panels[lp].n_seg + 1);
    cudaError_t e;
#define TRY(x)                          \
    do {                                \
        if ((e = (x)) != cudaSuccess) { \
            goto done;                  \
        }                               \
    } while (0)
    {
        TRY(cudaMalloc(&krc, 8 * nz));
        TRY(cudaMalloc(&kcr, 8 * nz));
        TRY(cudaMalloc(&k2, 8 * nz));
        TRY(cudaMalloc(&v0, 8 * nz));
        TRY(cudaMalloc(&M.csr_val, 8 * nz));
        TRY(cudaMalloc(&M.csc_val, 8 * nz));
        TRY(cudaMalloc(&M.csr_col, 4 * nz));
        TRY(cudaMalloc(&M.csc_row, 4 * nz));
        TRY(cudaMalloc(&M.row_ptr, 8 * (n_meas + 1)));
        TRY(cudaMalloc(&M.col_ptr, 8 * (n_vox + 1)));
        TRY(cudaMalloc(&seg_off, 8 * max_seg));
        // segment entry offsets: exclusive scan of seg_len (int32 -> int64)
        void *tmp = nullptr;
        size_t tb = 0, tb2 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, (const int32_t *)nullptr, seg_off, max_seg, s);
        int bits = 1;
        const uint64_t kmax = (uint64_t)n_meas * (uint64_t)n_vox;
        while (bits < 64 && (kmax >> bits) != 0) ++bits;
        cub::DeviceRadixSort::SortPairs(nullptr, tb2, krc, k2, v0, M.csr_val, nz, 0, bits, s);
        TRY(cudaMalloc(&tmp, std::max(tb, tb2)));
        int64_t base = 0;
        for (int lp = 0; lp < np; ++lp) {
            const PanelDev &P = h_panels[lp];
            if (P.n_seg == 0) continue;
            size_t t = std::max(tb, tb2);
            cub::DeviceScan::ExclusiveSum(tmp, t, P.seg_len, seg_off, P.n_seg, s);
            emit_k<<<nblk(P.n_seg, 128), 128, 0, s>>>(P, d_gvox, seg_off, base, n_vox, n_meas,
                                                      dtype != 0, krc, kcr, v0);
            TRY(cudaGetLastError());
            base += P.nnz;
        }
        size_t t = std::max(tb, tb2);
        TRY(cub::DeviceRadixSort::SortPairs(tmp, t, krc, k2, v0, M.csr_val, nz, 0, bits, s));
        ptr_k<<<nblk(n_meas + 1, 256), 256, 0, s>>>(k2, nnz, (uint64_t)n_vox, n_meas, M.row_ptr);
        minor_k<<<nblk(nz, 256), 256, 0, s>>>(k2, nnz, (uint64_t)n_vox, M.csr_col);
        t = std::max(tb, tb2);
        TRY(cub::DeviceRadixSort::SortPairs(tmp, t, kcr, k2, v0, M.csc_val, nz, 0, bits, s));
        ptr_k<<<nblk(n_vox + 1, 256), 256, 0, s>>>(k2, nnz, (uint64_t)n_meas, n_vox, M.col_ptr);
        minor_k<<<nblk(nz, 256), 256, 0, s>>>(k2, nnz, (uint64_t)n_meas, M.csc_row);
        TRY(cudaGetLastError());
        TRY(cudaStreamSynchronize(s));
        cudaFree(tmp);
    }
done:
#undef TRY
    cudaFree(krc);
    cudaFree(kcr);
    cudaFree(k2);
    cudaFree(v0);
    cudaFree(seg_off);
    return e;
}

void baseline_free(BaselineMat &M)
{
    for (void *p : {(void *)M.row_ptr, (void *)M.col_ptr, (void *)M.csr_col, (void *)M.csc_row,
                    (void *)M.csr_val, (void *)M.csc_val})
        if (p) cudaFree(p);
    M = BaselineMat();
}

cudaError_t baseline_scale(const BaselineMat &M, int kind, int rule, double *diag, cudaStream_t s)
{
    if (kind == 0)
        scale_k<<<nblk(M.n_meas, 256), 256, 0, s>>>(M.row_ptr, M.csr_val, M.n_meas, rule, diag);
    else
        scale_k<<<nblk(M.n_vox, 256), 256, 0, s>>>(M.col_ptr, M.csc_val, M.n_vox, rule, diag);
    return cudaGetLastError();
}

cudaError_t baseline_row_block(const BaselineMat &M, const int32_t *rows, int64_t n_rows, int blk,
                               int32_t g_lo, int32_t g_hi, const int32_t *rb_of_row, double omega,
                               const double *y, const double *mdiag, double *res, double *x,
                               cudaStream_t s)
{
    if (n_rows > 0)
        ra_res_k<<<nblk(n_rows, 128), 128, 0, s>>>(M.row_ptr, M.csr_col, M.csr_val, rows, n_rows,
                                                   y, x, mdiag, res);
    ra_upd_k<<<nblk(M.n_vox, 128), 128, 0, s>>>(M.col_ptr, M.csc_row, M.csc_val, rb_of_row, blk,
                                                g_lo, g_hi, M.n_vox, omega, res, x);
    return cudaGetLastError();
}

cudaError_t baseline_col_block(const BaselineMat &M, const int64_t *vox, int64_t n_vox_blk,
                               int blk, int32_t v_lo, int32_t v_hi, const int32_t *cb_of_vox,
                               double omega,
                               const double *ddiag, double *dx, double *x, double *r,
                               cudaStream_t s)
{
    if (n_vox_blk > 0)
        ca_dx_k<<<nblk(n_vox_blk, 128), 128, 0, s>>>(M.col_ptr, M.csc_row, M.csc_val, vox,
                                                     n_vox_blk, omega, ddiag, r, x, dx);
    ca_res_k<<<nblk(M.n_meas, 128), 128, 0, s>>>(M.row_ptr, M.csr_col, M.csr_val, cb_of_vox, blk,
                                                 v_lo, v_hi, M.n_meas, dx, r);
    return cudaGetLastError();
}

cudaError_t baseline_norms(const BaselineMat &M, const double *y, const double *r, const double *x,
                           const double *x_true, const int32_t *gvox, int64_t x_len, int use_r,
                           double *part, double *out4, cudaStream_t s)
{
    constexpr int NB = 148;
    norms_k<<<NB, 256, 0, s>>>(M.row_ptr, M.csr_col, M.csr_val, M.n_meas, y, r, x, x_true, gvox,
                               x_len, use_r, part);
    norms_fin_k<<<1, 32, 0, s>>>(part, NB, out4);
    return cudaGetLastError();
}

}  // namespace bct
