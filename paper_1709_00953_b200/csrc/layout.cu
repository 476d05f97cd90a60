// layout.cu -- the HBM layout of one column panel, built on the device.
//
// The epoch kernel is bound by L1 wavefronts, not bytes, when it gathers the
// dense vectors straight from global memory (one wavefront per distinct
// 128-byte line; a warp-wide gather of residual or image entries touches up to
// 32 lines).  The layout therefore makes every gather a shared-memory access:
//
// Phase 1 (g = A_I^T r_I) reads the panel CSC.  Columns (voxels) are grouped
// into tiles of 16 (4x4 voxels for strips); the rows crossing a tile form a
// narrow "sinogram band" (a few bins per view).  Per tile the band is stored
// as ranges of consecutive measurement ids; the kernel stages r over the band
// in shared memory and every CSC entry carries its 16-bit band slot (tloc).
//
// Phase 2 (t = A_I g, ax = A_I x_J) reads the forward store.  The panel's
// voxels are cut into super tiles of <= 4096 (iy ranges of a strip); each
// row's entries are grouped per super tile into segments (row, tile) padded
// to 4 entries, stored super-tile-major, and carry 16-bit tile-local voxel
// indices (fidx).  The kernel stages one super tile's (g, x) pairs in shared
// memory and streams its segments; per-segment partial sums are combined per
// row in super-tile order (deterministic).  Segments are grouped into units
// of whole segments (<= ~512 entries) that never cross a (tile, row block)
// boundary, so any subset of row blocks maps to whole units.
//
// Entries inside a segment stay in the reference's column order, and a row's
// segments in tile order, so the bitwise set-up kernels (builder.cu) recover
// the reference's summation order by merging a row's segments by column.
#include <cstdint>
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <string>
#include <vector>

#include "internal.h"

namespace {

inline unsigned nb(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

int bits_for(int64_t v)
{
    int b = 1;
    while ((1ll << b) <= v) ++b;
    return b;
}

__device__ __forceinline__ int64_t lb_i32(const int32_t *a, int64_t lo, int64_t hi, int32_t key)
{
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int64_t lb_u64(const uint64_t *a, int64_t lo, int64_t hi, uint64_t key)
{
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void row_of_entry_k(const int32_t *indptr, int32_t n_rows, int32_t *rowid)
{
    int lr = blockIdx.x * blockDim.x + threadIdx.x;
    if (lr >= n_rows) return;
    for (int p = indptr[lr]; p < indptr[lr + 1]; ++p) rowid[p] = lr;
}

__global__ void iota_k(int32_t *v, int64_t n)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = (int32_t)i;
}

// ---- forward store (phase 2) -------------------------------------------------

// key of entry p = st(d(c)) * n_rows + row
__global__ void fwd_key_k(const int32_t *cols_c, const int32_t *rowid, const int32_t *c2d,
                          const int32_t *d2st, int32_t n_rows, int64_t nnz, int32_t *key)
{
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= nnz) return;
    key[p] = d2st[c2d[cols_c[p]]] * n_rows + rowid[p];
}

// 1 where a new segment starts in sorted order
__global__ void seg_flag_k(const int32_t *skey, int64_t nnz, int32_t *flag)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    flag[q] = (q == 0 || skey[q] != skey[q - 1]) ? 1 : 0;
}

// segment s: first sorted position, key; (seg id = inclusive scan - 1)
__global__ void seg_first_k(const int32_t *flag, const int32_t *incl, const int32_t *skey,
                            int64_t nnz, int32_t *seg_first, int32_t *seg_key)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnz || !flag[q]) return;
    int s = incl[q] - 1;
    seg_first[s] = (int32_t)q;
    seg_key[s] = skey[q];
}

__global__ void seg_len4_k(const int32_t *seg_first, int32_t n_seg, int64_t nnz, int32_t *len4)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s > n_seg) return;
    if (s == n_seg) { len4[s] = 0; return; }
    int64_t e = (s + 1 < n_seg) ? seg_first[s + 1] : nnz;
    len4[s] = (int32_t)(((e - seg_first[s]) + 3) & ~3);
}

// scatter sorted entries into padded segment slots
template <typename V>
__global__ void fwd_scatter_k(const int32_t *perm, const int32_t *incl, const int32_t *seg_first,
                              const int32_t *seg_start, const int32_t *seg_key,
                              const double *vals64, const int32_t *cols_c, const int32_t *c2d,
                              const int32_t *st_ptr, int32_t n_rows, int64_t nnz, V *fvals,
                              uint16_t *fidx)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    int s = incl[q] - 1;
    int p = perm[q];
    int st = seg_key[s] / n_rows;
    int64_t dst = seg_start[s] + (q - seg_first[s]);
    fvals[dst] = (V)vals64[p];
    fidx[dst] = (uint16_t)(c2d[cols_c[p]] - st_ptr[st]);
}

// padding: zero value on the segment's last voxel; row-start bitmap; seg_row
template <typename V>
__global__ void fwd_pad_k(const int32_t *seg_first, const int32_t *seg_start, const int32_t *seg_key,
                          int32_t n_seg, int64_t nnz, int32_t n_rows, V *fvals, uint16_t *fidx,
                          uint32_t *bits, int32_t *seg_row)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    int64_t len = ((s + 1 < n_seg) ? seg_first[s + 1] : nnz) - seg_first[s];
    int64_t a = seg_start[s] + len, e = seg_start[s + 1];
    uint16_t last = fidx[a - 1];
    for (int64_t q = a; q < e; ++q) {
        fvals[q] = (V)0;
        fidx[q] = last;
    }
    uint32_t v = (uint32_t)seg_start[s] >> 2;
    atomicOr(&bits[v >> 5], 1u << (v & 31));
    seg_row[s] = seg_key[s] % n_rows;
}

// units: segment s opens a unit when it is the first of its (tile, row
// block) group or its start enters a new 512-entry window of the group
__global__ void unit_flag_k(const int32_t *seg_key, const int32_t *seg_start, int32_t n_seg,
                            int32_t n_rows, const int32_t *rbp, int m, int unit_entries,
                            int32_t *grp, int32_t *flag)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    int st = seg_key[s] / n_rows, lr = seg_key[s] % n_rows;
    int i = (int)lb_i32(rbp, 0, m + 1, lr + 1) - 1;  // block of lr
    grp[s] = st * (m + 1) + i;
    __syncwarp();
}

__global__ void unit_flag2_k(const int32_t *grp, const int32_t *seg_start, int32_t n_seg,
                             int unit_entries, const int32_t *grp_first_pos, int32_t *flag)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    if (s == 0 || grp[s] != grp[s - 1]) { flag[s] = 1; return; }
    int g0 = grp_first_pos[s];
    flag[s] = ((seg_start[s] - g0) / unit_entries != (seg_start[s - 1] - g0) / unit_entries) ? 1 : 0;
}

// first segment start of every segment's group (segments of a group are contiguous)
__global__ void grp_first_k(const int32_t *grp, const int32_t *seg_start, int32_t n_seg,
                            int32_t *grp_first_pos)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    // binary search the first segment with the same group
    int lo = 0, hi = s;
    while (lo < hi) {
        int mid = (lo + hi) / 2;
        if (grp[mid] < grp[s]) lo = mid + 1; else hi = mid;
    }
    grp_first_pos[s] = seg_start[lo];
}

__global__ void unit_collect_k(const int32_t *flag, const int32_t *incl, int32_t n_seg,
                               int32_t *u_seg)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg || !flag[s]) return;
    u_seg[incl[s] - 1] = s;
}

__global__ void unit_st_k(const int32_t *u_seg, const int32_t *seg_key, int32_t n_units,
                          int32_t n_rows, int32_t *u_st)
{
    int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n_units) return;
    u_st[u] = seg_key[u_seg[u]] / n_rows;
}

// stbu[st*(m+1)+i] = first unit of (tile st, block >= i)
__global__ void stbu_k(const int32_t *seg_key, int32_t n_seg, const int32_t *u_seg, int32_t n_units,
                       const int32_t *rbp, int m, int32_t n_st, int32_t n_rows, int32_t *stbu)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_st * (m + 1)) return;
    int st = t / (m + 1), i = t % (m + 1);
    int32_t key = st * n_rows + rbp[i];
    int64_t s = lb_i32(seg_key, 0, n_seg, key);
    stbu[t] = (int32_t)lb_i32(u_seg, 0, n_units, (int32_t)s);
}

// rows -> segments in tile order: sort segment ids by row*n_st + tile
__global__ void rkey_k(const int32_t *seg_key, int32_t n_seg, int32_t n_rows, int32_t n_st,
                       int32_t *rkey)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    rkey[s] = (seg_key[s] % n_rows) * n_st + seg_key[s] / n_rows;
}

__global__ void rseg_ptr_k(const int32_t *srkey, int32_t n_seg, int32_t n_rows, int32_t n_st,
                           int32_t *rseg_ptr)
{
    int lr = blockIdx.x * blockDim.x + threadIdx.x;
    if (lr > n_rows) return;
    rseg_ptr[lr] = (int32_t)lb_i32(srkey, 0, n_seg, lr * n_st);
}

// ---- CSC with tile bands (phase 1) ----------------------------------------------

__global__ void csc_key_k(const int32_t *cols_c, const int32_t *c2d, int64_t nnz, int32_t *dkey)
{
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < nnz) dkey[p] = c2d[cols_c[p]];
}

__global__ void colcount_k(const int32_t *sorted_d, int64_t nnz, int32_t n_cols, int32_t *colstart,
                           int32_t *len8)
{
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > n_cols) return;
    int64_t s = lb_i32(sorted_d, 0, nnz, c);
    colstart[c] = (int32_t)s;
    if (c < n_cols) {
        int64_t e = lb_i32(sorted_d, s, nnz, c + 1);
        len8[c] = (int32_t)(((e - s) + 7) & ~7);
    } else {
        len8[c] = 0;
    }
}

// band keys: (tile of column) << 32 | global row, per CSC entry in sorted order
__global__ void band_key_k(const int32_t *perm, const int32_t *rowid, const int32_t *l2g,
                           const int32_t *sorted_d, const int32_t *tile_of_d, int64_t nnz,
                           uint64_t *bkey, int32_t *grow)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    int32_t g = l2g[rowid[perm[q]]];
    grow[q] = g;
    bkey[q] = ((uint64_t)(uint32_t)tile_of_d[sorted_d[q]] << 32) | (uint32_t)g;
}

__global__ void uniq_flag_k(const uint64_t *k, int64_t n, int32_t *flag)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < n) flag[q] = (q == 0 || k[q] != k[q - 1]) ? 1 : 0;
}

__global__ void uniq_collect_k(const uint64_t *k, const int32_t *flag, const int32_t *incl,
                               int64_t n, uint64_t *u)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < n && flag[q]) u[incl[q] - 1] = k[q];
}

// range starts among unique keys: new tile or non-consecutive row
__global__ void range_flag_k(const uint64_t *u, int64_t nu, int32_t *flag)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nu) return;
    flag[q] = (q == 0 || (u[q] >> 32) != (u[q - 1] >> 32) || u[q] != u[q - 1] + 1) ? 1 : 0;
}

// per tile: first unique index (tile_u0) and first range (band_ptr)
__global__ void tile_bounds_k(const uint64_t *u, int64_t nu, const int32_t *rflag_incl,
                              int32_t n_tiles, int32_t *tile_u0, int32_t *band_ptr)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > n_tiles) return;
    int64_t q = lb_u64(u, 0, nu, (uint64_t)(uint32_t)t << 32);
    tile_u0[t] = (int32_t)q;
    // ranges before q = number of range starts in [0, q)
    band_ptr[t] = q == 0 ? 0 : rflag_incl[q - 1];
}

__global__ void ranges_k(const uint64_t *u, int64_t nu, const int32_t *rflag, const int32_t *rincl,
                         const int32_t *tile_u0, int32_t *band_start, int32_t *band_pre,
                         int32_t *band_len)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nu || !rflag[q]) return;
    int k = rincl[q] - 1;
    int t = (int)(u[q] >> 32);
    band_start[k] = (int32_t)(uint32_t)u[q];
    band_pre[k] = (int32_t)(q - tile_u0[t]);
    // length: up to the next range start
    int64_t e = q + 1;
    while (e < nu && !rflag[e]) ++e;
    band_len[k] = (int32_t)(e - q);
}

template <typename V>
__global__ void csc_scatter_k(const int32_t *perm, const double *vals64, const int32_t *sorted_d,
                              const int32_t *grow, const int32_t *tile_of_d, const uint64_t *u,
                              const int32_t *tile_u0, const int32_t *colstart, const int32_t *cpad,
                              int64_t nnz, V *tvals, uint16_t *tloc)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    int d = sorted_d[q];
    int t = tile_of_d[d];
    uint64_t key = ((uint64_t)(uint32_t)t << 32) | (uint32_t)grow[q];
    int64_t pos = lb_u64(u, tile_u0[t], tile_u0[t + 1], key);
    int64_t dst = cpad[d] + (q - colstart[d]);
    tvals[dst] = (V)vals64[perm[q]];
    tloc[dst] = (uint16_t)(pos - tile_u0[t]);
}

template <typename V>
__global__ void csc_pad_k(const int32_t *colstart, const int32_t *cpad, int32_t n_cols, V *tvals,
                          uint16_t *tloc)
{
    int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_cols) return;
    int64_t a = cpad[d] + (colstart[d + 1] - colstart[d]);
    uint16_t last = a > cpad[d] ? tloc[a - 1] : 0;
    for (int64_t q = a; q < cpad[d + 1]; ++q) {
        tvals[q] = (V)0;
        tloc[q] = last;
    }
}

// cptr[d*(m+1)+i] = padded position of column d's first entry with local row >= rbp[i]
__global__ void cptr_k(const int32_t *colstart, const int32_t *cpad, const int32_t *tlocal_sorted,
                       const int32_t *rbp, int m, int32_t n_cols, int32_t *cptr)
{
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)n_cols * (m + 1)) return;
    int d = (int)(t / (m + 1)), i = (int)(t % (m + 1));
    int64_t lb = lb_i32(tlocal_sorted, colstart[d], colstart[d + 1], rbp[i]);
    cptr[t] = (int32_t)(cpad[d] + (lb - colstart[d]));
}

__global__ void gather_rows_k(const int32_t *perm, const int32_t *rowid, int64_t nnz, int32_t *out)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < nnz) out[q] = rowid[perm[q]];
}

}  // namespace

namespace bct {

struct Alloc {
    std::vector<void *> *list;
    std::string *err;
    template <typename T>
    T *get(int64_t n)
    {
        void *p = nullptr;
        size_t bytes = (size_t)std::max<int64_t>(n, 1) * sizeof(T);
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            *err = "cudaMalloc failed in layout (" + std::to_string(bytes) + " bytes)";
            return nullptr;
        }
        list->push_back(p);
        return (T *)p;
    }
};

static void release(std::vector<void *> &tmp)
{
    for (void *p : tmp) cudaFree(p);
    tmp.clear();
}

#define LCK(x)                                                                   \
    do {                                                                         \
        cudaError_t _e = (x);                                                    \
        if (_e != cudaSuccess) {                                                 \
            err = std::string(#x) + ": " + cudaGetErrorString(_e);               \
            release(tmp);                                                        \
            return -1;                                                           \
        }                                                                        \
    } while (0)
#define LNN(p)                     \
    do {                           \
        if (!(p)) {                \
            release(tmp);          \
            return -1;             \
        }                          \
    } while (0)

// exclusive (incl=false) / inclusive scan of int32
static cudaError_t scan_i32(const int32_t *in, int32_t *out, int64_t n, bool inclusive,
                            std::vector<void *> &tmp, cudaStream_t s)
{
    size_t b = 0;
    if (inclusive) cub::DeviceScan::InclusiveSum(nullptr, b, in, out, (int)n, s);
    else cub::DeviceScan::ExclusiveSum(nullptr, b, in, out, (int)n, s);
    void *t = nullptr;
    cudaError_t e = cudaMalloc(&t, std::max<size_t>(b, 16));
    if (e != cudaSuccess) return e;
    tmp.push_back(t);
    if (inclusive) return cub::DeviceScan::InclusiveSum(t, b, in, out, (int)n, s);
    return cub::DeviceScan::ExclusiveSum(t, b, in, out, (int)n, s);
}

template <typename K>
static cudaError_t sort_pairs(const K *kin, K *kout, const int32_t *vin, int32_t *vout, int64_t n,
                              int end_bit, std::vector<void *> &tmp, cudaStream_t s)
{
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, kin, kout, vin, vout, (int)n, 0, end_bit, s);
    void *t = nullptr;
    cudaError_t e = cudaMalloc(&t, std::max<size_t>(b, 16));
    if (e != cudaSuccess) return e;
    tmp.push_back(t);
    return cub::DeviceRadixSort::SortPairs(t, b, kin, kout, vin, vout, (int)n, 0, end_bit, s);
}

static cudaError_t sort_keys_u64(const uint64_t *kin, uint64_t *kout, int64_t n, int end_bit,
                                 std::vector<void *> &tmp, cudaStream_t s)
{
    size_t b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b, kin, kout, (int)n, 0, end_bit, s);
    void *t = nullptr;
    cudaError_t e = cudaMalloc(&t, std::max<size_t>(b, 16));
    if (e != cudaSuccess) return e;
    tmp.push_back(t);
    return cub::DeviceRadixSort::SortKeys(t, b, kin, kout, (int)n, 0, end_bit, s);
}

template <typename T>
static T read1(const T *d, cudaStream_t s)
{
    T h{};
    cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return h;
}

// Builds every array of PanelDev for one panel from its compact forward CSR in
// the reference's order.  Device inputs: vals64, cols_c, indptr_c, l2g, rbp.
// Host inputs: c2d (column -> device position), st_ptr (super tiles over
// device positions), corder (tile order of device positions, 16 per tile).
// Persistent arrays are appended to `keep`; returns 0 or -1 with `err`.
int layout_panel_v2(int dtype, int m, int32_t n_rows, int32_t n_cols, int64_t nnz,
                    const double *vals64, const int32_t *cols_c, const int32_t *indptr_c,
                    const int32_t *l2g, const int32_t *rbp, const std::vector<int32_t> &c2d_h,
                    const std::vector<int32_t> &st_ptr_h, const std::vector<int32_t> &corder_h,
                    int unit_entries, PanelDev &P, std::vector<void *> &keep, std::string &err,
                    cudaStream_t s)
{
    std::vector<void *> tmp;
    Alloc K{&keep, &err}, T{&tmp, &err};
    const int vs = dtype == 0 ? 8 : 4;
    const int32_t n_st = (int32_t)st_ptr_h.size() - 1;
    const int32_t n_tiles = (int32_t)((corder_h.size() + 15) / 16);

    // host tables -> device
    std::vector<int32_t> d2st_h(n_cols), tile_of_d_h(n_cols);
    for (int st = 0; st < n_st; ++st)
        for (int d = st_ptr_h[st]; d < st_ptr_h[st + 1]; ++d) d2st_h[d] = st;
    for (size_t q = 0; q < corder_h.size(); ++q) tile_of_d_h[corder_h[q]] = (int32_t)(q / 16);
    int32_t *c2d = T.get<int32_t>(n_cols), *d2st = T.get<int32_t>(n_cols);
    int32_t *tile_of_d = T.get<int32_t>(n_cols);
    int32_t *st_ptr = K.get<int32_t>(n_st + 1), *corder = K.get<int32_t>(n_cols);
    LNN(c2d); LNN(d2st); LNN(tile_of_d); LNN(st_ptr); LNN(corder);
    LCK(cudaMemcpyAsync(c2d, c2d_h.data(), 4 * n_cols, cudaMemcpyHostToDevice, s));
    LCK(cudaMemcpyAsync(d2st, d2st_h.data(), 4 * n_cols, cudaMemcpyHostToDevice, s));
    LCK(cudaMemcpyAsync(tile_of_d, tile_of_d_h.data(), 4 * n_cols, cudaMemcpyHostToDevice, s));
    LCK(cudaMemcpyAsync(st_ptr, st_ptr_h.data(), 4 * (n_st + 1), cudaMemcpyHostToDevice, s));
    LCK(cudaMemcpyAsync(corder, corder_h.data(), 4 * n_cols, cudaMemcpyHostToDevice, s));

    int32_t *rowid = T.get<int32_t>(nnz), *iota = T.get<int32_t>(nnz);
    int32_t *key = T.get<int32_t>(nnz), *skey = T.get<int32_t>(nnz), *perm = T.get<int32_t>(nnz);
    int32_t *flag = T.get<int32_t>(nnz), *incl = T.get<int32_t>(nnz);
    LNN(rowid); LNN(iota); LNN(key); LNN(skey); LNN(perm); LNN(flag); LNN(incl);
    if (nnz > 0) {
        row_of_entry_k<<<nb(n_rows, 128), 128, 0, s>>>(indptr_c, n_rows, rowid);
        iota_k<<<nb(nnz, 256), 256, 0, s>>>(iota, nnz);
    }

    // ================= forward segments =================
    int32_t n_seg = 0;
    if (nnz > 0) {
        fwd_key_k<<<nb(nnz, 256), 256, 0, s>>>(cols_c, rowid, c2d, d2st, n_rows, nnz, key);
        LCK(sort_pairs<int32_t>(key, skey, iota, perm, nnz, bits_for((int64_t)n_st * n_rows), tmp, s));
        seg_flag_k<<<nb(nnz, 256), 256, 0, s>>>(skey, nnz, flag);
        LCK(scan_i32(flag, incl, nnz, true, tmp, s));
        n_seg = read1(incl + nnz - 1, s);
    }
    int32_t *seg_first = T.get<int32_t>(n_seg + 1), *seg_key = K.get<int32_t>(n_seg + 1);
    int32_t *len4 = T.get<int32_t>(n_seg + 1), *seg_start = K.get<int32_t>(n_seg + 1);
    LNN(seg_first); LNN(seg_key); LNN(len4); LNN(seg_start);
    int64_t fwd_cap = 0;
    if (n_seg > 0) {
        seg_first_k<<<nb(nnz, 256), 256, 0, s>>>(flag, incl, skey, nnz, seg_first, seg_key);
        seg_len4_k<<<nb(n_seg + 1, 256), 256, 0, s>>>(seg_first, n_seg, nnz, len4);
        LCK(scan_i32(len4, seg_start, n_seg + 1, false, tmp, s));
        fwd_cap = read1(seg_start + n_seg, s);
    } else {
        LCK(cudaMemsetAsync(seg_start, 0, 4, s));
    }
    void *fvals = K.get<char>(std::max<int64_t>(fwd_cap, 1) * vs);
    uint16_t *fidx = K.get<uint16_t>(fwd_cap);
    int64_t nwords = fwd_cap / 128 + 1;
    uint32_t *fbits = K.get<uint32_t>(nwords);
    int32_t *seg_row = K.get<int32_t>(n_seg + 1);
    LNN(fvals); LNN(fidx); LNN(fbits); LNN(seg_row);
    LCK(cudaMemsetAsync(fbits, 0, 4 * nwords, s));
    if (n_seg > 0) {
        if (dtype == 0) {
            fwd_scatter_k<double><<<nb(nnz, 256), 256, 0, s>>>(perm, incl, seg_first, seg_start,
                seg_key, vals64, cols_c, c2d, st_ptr, n_rows, nnz, (double *)fvals, fidx);
            fwd_pad_k<double><<<nb(n_seg, 256), 256, 0, s>>>(seg_first, seg_start, seg_key, n_seg,
                nnz, n_rows, (double *)fvals, fidx, fbits, seg_row);
        } else {
            fwd_scatter_k<float><<<nb(nnz, 256), 256, 0, s>>>(perm, incl, seg_first, seg_start,
                seg_key, vals64, cols_c, c2d, st_ptr, n_rows, nnz, (float *)fvals, fidx);
            fwd_pad_k<float><<<nb(n_seg, 256), 256, 0, s>>>(seg_first, seg_start, seg_key, n_seg,
                nnz, n_rows, (float *)fvals, fidx, fbits, seg_row);
        }
    }
    // units
    int32_t *grp = T.get<int32_t>(n_seg + 1), *gfirst = T.get<int32_t>(n_seg + 1);
    int32_t *uflag = T.get<int32_t>(n_seg + 1), *uincl = T.get<int32_t>(n_seg + 1);
    LNN(grp); LNN(gfirst); LNN(uflag); LNN(uincl);
    int32_t n_units = 0;
    if (n_seg > 0) {
        unit_flag_k<<<nb(n_seg, 256), 256, 0, s>>>(seg_key, seg_start, n_seg, n_rows, rbp, m,
                                                   unit_entries, grp, uflag);
        grp_first_k<<<nb(n_seg, 256), 256, 0, s>>>(grp, seg_start, n_seg, gfirst);
        unit_flag2_k<<<nb(n_seg, 256), 256, 0, s>>>(grp, seg_start, n_seg, unit_entries, gfirst,
                                                    uflag);
        LCK(scan_i32(uflag, uincl, n_seg, true, tmp, s));
        n_units = read1(uincl + n_seg - 1, s);
    }
    int32_t *u_seg = K.get<int32_t>(n_units + 1), *u_st = K.get<int32_t>(n_units + 1);
    int32_t *stbu = K.get<int32_t>((int64_t)n_st * (m + 1) + 1);
    LNN(u_seg); LNN(u_st); LNN(stbu);
    if (n_units > 0) {
        unit_collect_k<<<nb(n_seg, 256), 256, 0, s>>>(uflag, uincl, n_seg, u_seg);
        unit_st_k<<<nb(n_units, 256), 256, 0, s>>>(u_seg, seg_key, n_units, n_rows, u_st);
    }
    LCK(cudaMemcpyAsync(u_seg + n_units, &n_seg, 4, cudaMemcpyHostToDevice, s));
    LCK(cudaStreamSynchronize(s));  // &n_seg is a host stack value
    stbu_k<<<nb((int64_t)n_st * (m + 1), 128), 128, 0, s>>>(seg_key, n_seg, u_seg, n_units, rbp, m,
                                                           n_st, n_rows, stbu);
    // rows -> segments (tile order)
    int32_t *rkey = T.get<int32_t>(n_seg + 1), *srkey = T.get<int32_t>(n_seg + 1);
    int32_t *sid = T.get<int32_t>(n_seg + 1), *rseg = K.get<int32_t>(n_seg + 1);
    int32_t *rseg_ptr = K.get<int32_t>(n_rows + 1);
    LNN(rkey); LNN(srkey); LNN(sid); LNN(rseg); LNN(rseg_ptr);
    if (n_seg > 0) {
        rkey_k<<<nb(n_seg, 256), 256, 0, s>>>(seg_key, n_seg, n_rows, n_st, rkey);
        iota_k<<<nb(n_seg, 256), 256, 0, s>>>(sid, n_seg);
        LCK(sort_pairs<int32_t>(rkey, srkey, sid, rseg, n_seg,
                                bits_for((int64_t)n_rows * n_st), tmp, s));
    }
    rseg_ptr_k<<<nb(n_rows + 1, 256), 256, 0, s>>>(srkey, n_seg, n_rows, n_st, rseg_ptr);
    LCK(cudaGetLastError());

    // ================= CSC with tile bands =================
    int32_t *sd = T.get<int32_t>(nnz), *cperm = T.get<int32_t>(nnz);
    int32_t *colstart = T.get<int32_t>(n_cols + 1), *cpad = T.get<int32_t>(n_cols + 1);
    int32_t *len8 = T.get<int32_t>(n_cols + 1);
    LNN(sd); LNN(cperm); LNN(colstart); LNN(cpad); LNN(len8);
    if (nnz > 0) {
        csc_key_k<<<nb(nnz, 256), 256, 0, s>>>(cols_c, c2d, nnz, key);
        LCK(sort_pairs<int32_t>(key, sd, iota, cperm, nnz, bits_for(n_cols), tmp, s));
    }
    colcount_k<<<nb(n_cols + 1, 256), 256, 0, s>>>(sd, nnz, n_cols, colstart, len8);
    LCK(scan_i32(len8, cpad, n_cols + 1, false, tmp, s));
    int64_t csc_cap = read1(cpad + n_cols, s);
    // bands
    uint64_t *bkey = T.get<uint64_t>(nnz), *bsorted = T.get<uint64_t>(nnz);
    int32_t *grow = T.get<int32_t>(nnz);
    LNN(bkey); LNN(bsorted); LNN(grow);
    int64_t nu = 0;
    if (nnz > 0) {
        band_key_k<<<nb(nnz, 256), 256, 0, s>>>(cperm, rowid, l2g, sd, tile_of_d, nnz, bkey, grow);
        LCK(sort_keys_u64(bkey, bsorted, nnz, 32 + bits_for(n_tiles), tmp, s));
        uniq_flag_k<<<nb(nnz, 256), 256, 0, s>>>(bsorted, nnz, flag);
        LCK(scan_i32(flag, incl, nnz, true, tmp, s));
        nu = read1(incl + nnz - 1, s);
    }
    uint64_t *uk = T.get<uint64_t>(nu + 1);
    int32_t *rflag = T.get<int32_t>(nu + 1), *rincl = T.get<int32_t>(nu + 1);
    int32_t *tile_u0 = T.get<int32_t>(n_tiles + 1);
    LNN(uk); LNN(rflag); LNN(rincl); LNN(tile_u0);
    int32_t n_ranges = 0;
    if (nu > 0) {
        uniq_collect_k<<<nb(nnz, 256), 256, 0, s>>>(bsorted, flag, incl, nnz, uk);
        range_flag_k<<<nb(nu, 256), 256, 0, s>>>(uk, nu, rflag);
        LCK(scan_i32(rflag, rincl, nu, true, tmp, s));
        n_ranges = read1(rincl + nu - 1, s);
    }
    int32_t *band_ptr = K.get<int32_t>(n_tiles + 1), *band_start = K.get<int32_t>(n_ranges + 1);
    int32_t *band_pre = K.get<int32_t>(n_ranges + 1), *band_len = K.get<int32_t>(n_ranges + 1);
    LNN(band_ptr); LNN(band_start); LNN(band_pre); LNN(band_len);
    tile_bounds_k<<<nb(n_tiles + 1, 128), 128, 0, s>>>(uk, nu, rincl, n_tiles, tile_u0, band_ptr);
    if (n_ranges > 0)
        ranges_k<<<nb(nu, 256), 256, 0, s>>>(uk, nu, rflag, rincl, tile_u0, band_start, band_pre,
                                             band_len);
    // the widest band sets the shared-memory size
    std::vector<int32_t> tu(n_tiles + 1);
    LCK(cudaMemcpyAsync(tu.data(), tile_u0, 4 * (n_tiles + 1), cudaMemcpyDeviceToHost, s));
    LCK(cudaStreamSynchronize(s));
    int32_t band_max = 0;
    for (int t = 0; t < n_tiles; ++t) band_max = std::max(band_max, tu[t + 1] - tu[t]);
    if (band_max > 65535) {
        err = "a column tile touches more than 65535 measurement rows";
        release(tmp);
        return -1;
    }
    void *tvals = K.get<char>(std::max<int64_t>(csc_cap, 1) * vs);
    uint16_t *tloc = K.get<uint16_t>(csc_cap);
    int32_t *cptr = K.get<int32_t>((int64_t)n_cols * (m + 1));
    int32_t *tls = T.get<int32_t>(nnz);
    LNN(tvals); LNN(tloc); LNN(cptr); LNN(tls);
    if (nnz > 0) {
        if (dtype == 0)
            csc_scatter_k<double><<<nb(nnz, 256), 256, 0, s>>>(cperm, vals64, sd, grow, tile_of_d, uk,
                tile_u0, colstart, cpad, nnz, (double *)tvals, tloc);
        else
            csc_scatter_k<float><<<nb(nnz, 256), 256, 0, s>>>(cperm, vals64, sd, grow, tile_of_d, uk,
                tile_u0, colstart, cpad, nnz, (float *)tvals, tloc);
        gather_rows_k<<<nb(nnz, 256), 256, 0, s>>>(cperm, rowid, nnz, tls);
    }
    if (dtype == 0)
        csc_pad_k<double><<<nb(n_cols, 256), 256, 0, s>>>(colstart, cpad, n_cols, (double *)tvals, tloc);
    else
        csc_pad_k<float><<<nb(n_cols, 256), 256, 0, s>>>(colstart, cpad, n_cols, (float *)tvals, tloc);
    cptr_k<<<nb((int64_t)n_cols * (m + 1), 256), 256, 0, s>>>(colstart, cpad, tls, rbp, m, n_cols,
                                                             cptr);
    LCK(cudaGetLastError());
    LCK(cudaStreamSynchronize(s));
    release(tmp);

    P.fvals = fvals;
    P.fidx = fidx;
    P.fbits = fbits;
    P.seg_start = seg_start;
    P.seg_key = seg_key;
    P.u_seg = u_seg;
    P.u_st = u_st;
    P.stbu = stbu;
    P.st_ptr = st_ptr;
    P.rseg_ptr = rseg_ptr;
    P.rseg = rseg;
    P.seg_row = seg_row;
    P.tvals = tvals;
    P.tloc = tloc;
    P.cptr = cptr;
    P.corder = corder;
    P.band_ptr = band_ptr;
    P.band_start = band_start;
    P.band_pre = band_pre;
    P.band_len = band_len;
    P.n_seg = n_seg;
    P.n_units = n_units;
    P.n_st = n_st;
    P.n_tiles = n_tiles;
    P.band_max = band_max;
    int32_t st_max = 0;
    for (int st = 0; st < n_st; ++st) st_max = std::max(st_max, st_ptr_h[st + 1] - st_ptr_h[st]);
    P.st_max = st_max;
    P.fwd_cap = fwd_cap;
    P.csc_cap = csc_cap;
    return 0;
}

}  // namespace bct
