// layout.cu -- the HBM layout of one column panel, built on the device.
//
// The epoch kernel would be bound by L1 wavefronts, not bytes, if it gathered
// the dense vectors straight from global memory (one wavefront per distinct
// 128-byte line; a warp-wide gather of residual or image entries touches up to
// 32 lines).  The layout therefore makes every gather a shared-memory access:
//
// Phase 1 (g = A_I^T r_I) reads the panel CSC.  Columns (voxels) are grouped
// into tiles (16x16 voxels for strips, 8x8 / 4x8 when the band would not fit);
// the rows crossing a tile form a narrow "sinogram band" (a few bins per
// view), stored as even-aligned ranges of consecutive measurement ids that
// never cross a row block.  Each tile's columns are stored in 32-column slices,
// lane-interleaved 8 entries at a time (csl_start), every entry carrying its
// band slot (tloc, stored as an 8-bit offset on a 16-bit base per 8 entries
// when it fits: tloc_delta_k); a lane's 8 entries are ordered to spread the
// shared-memory banks of each gather.
//
// Phase 2 (t = A_I g, ax = A_I x_J) reads the forward store.  The panel's
// voxels are cut into super tiles (16384 voxels in FP32 mode, 4096 in FP64;
// iy ranges of a strip); each row's entries are grouped per super tile into
// segments (row, super tile) that carry 16-bit, swizzled super-tile voxel
// indices (fidx).  The segments of one (super tile, row block) group are
// sorted by length and stored as SELL-32 slices (32 segments interleaved 4
// entries at a time), so a warp streams a slice with coalesced 16-byte loads,
// one segment per lane, gathering (g, x) pairs from the staged super tile.
// Per-segment partials are combined per row in super-tile order
// (deterministic).  A task over any subset of row blocks maps to whole slices.
//
// Entries inside a segment are in the reference's column order -- except on
// step-coded strip panels (fcode_k), where an equal-ix run of a ray going down
// in iy is stored reversed (walk order) -- and a row's segments in tile order,
// so the bitwise set-up kernels (builder.cu row_dot) recover the reference's
// summation order by merging a row's segments by column, reading descending
// runs backwards.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <string>
#include <vector>

#include "internal.h"

namespace {

inline unsigned nb(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

constexpr int SEG_CAP = 64;   // default max entries of one forward segment (PanelDev::seg_cap)

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
// (a (row, super tile) group longer than cap entries is cut into several
// segments so that no SELL slice is much longer than its neighbours)
__global__ void seg_flag_k(const int32_t *skey, int64_t nnz, int cap, int32_t *flag)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    if (q == 0 || skey[q] != skey[q - 1]) {
        flag[q] = 1;
        return;
    }
    int64_t lo = lb_i32(skey, 0, q, skey[q]);
    flag[q] = ((q - lo) % cap == 0) ? 1 : 0;
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


// ---- forward store, SELL-32 slices of segments (phase 2) ------------------------
//
// segments (row, super tile) of one (super tile, row block) group are sorted
// by length (longest first) and cut into slices of 32; a slice stores its 32
// segments interleaved 4 entries at a time -- vector k of lane l sits at
// slice_start + (k*32 + l)*4 -- so a warp streams a slice with coalesced
// 16-byte loads, one segment per lane and no cross-lane reduction.

__global__ void seg_len_k(const int32_t *seg_first, int32_t n_seg, int64_t nnz, int32_t *len,
                          int32_t *nvec)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    int64_t e = (s + 1 < n_seg) ? seg_first[s + 1] : nnz;
    len[s] = (int32_t)(e - seg_first[s]);
    nvec[s] = (int32_t)((e - seg_first[s] + 3) / 4);
}

// key: (tile, row block) group ascending, vector count descending
__global__ void sell_key_k(const int32_t *seg_key, const int32_t *nvec, int32_t n_seg,
                           int32_t n_rows, const int32_t *rbp, int m, uint64_t *key)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    int st = seg_key[s] / n_rows, lr = seg_key[s] % n_rows;
    int blk = (int)lb_i32(rbp, 0, m + 1, lr + 1) - 1;
    uint32_t gid = (uint32_t)(st * (m + 1) + blk);
    key[s] = ((uint64_t)gid << 32) | (uint32_t)(0x7fffffff - nvec[s]);
}

__global__ void slice_flag_k(const uint64_t *skey, int32_t n_seg, int32_t *flag)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_seg) return;
    uint32_t g = (uint32_t)(skey[q] >> 32);
    int64_t lo = 0, hi = q;   // first position of this group
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if ((uint32_t)(skey[mid] >> 32) < g) lo = mid + 1; else hi = mid;
    }
    flag[q] = ((q - lo) % 32 == 0) ? 1 : 0;
}

__global__ void slice_info_k(const uint64_t *skey, const int32_t *sseg, const int32_t *flag_incl,
                             const int32_t *nvec, int32_t n_seg, int32_t *seg_slice,
                             int32_t *seg_lane, int32_t *sl_seg, int32_t *slice_len4,
                             int32_t *slice_gid)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_seg) return;
    uint32_t g = (uint32_t)(skey[q] >> 32);
    int64_t lo = 0, hi = q;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if ((uint32_t)(skey[mid] >> 32) < g) lo = mid + 1; else hi = mid;
    }
    int lane = (int)((q - lo) % 32);
    int sl = flag_incl[q] - 1;
    int s = sseg[q];
    seg_slice[s] = sl;
    seg_lane[s] = lane;
    sl_seg[(int64_t)sl * 32 + lane] = s;
    if (lane == 0) {
        slice_len4[sl] = nvec[s] * 128;  // entries of the slice (longest segment first)
        slice_gid[sl] = (int32_t)g;
    }
}

template <typename V>
__global__ void sell_scatter_k(const int32_t *perm, const int32_t *incl, const int32_t *seg_first,
                               const int32_t *seg_key, const int32_t *seg_slice,
                               const int32_t *seg_lane, const int32_t *slice_start,
                               const double *vals64, const int32_t *cols_c, const int32_t *c2d,
                               const int32_t *st_ptr, int32_t n_rows, int64_t nnz, V *fvals,
                               uint16_t *fidx, int swz_shift)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    int s = incl[q] - 1;
    int p = perm[q];
    int st = seg_key[s] / n_rows;
    int64_t e = q - seg_first[s];
    int64_t pos = slice_start[seg_slice[s]] + ((e >> 2) * 32 + seg_lane[s]) * 4 + (e & 3);
    fvals[pos] = (V)vals64[p];
    fidx[pos] = (uint16_t)swz_idx(c2d[cols_c[p]] - st_ptr[st], swz_shift);
}

// padding of every (slice, lane): zero values on the lane's last voxel
template <typename V>
__global__ void sell_pad_k(const int32_t *sl_seg, const int32_t *seg_len, const int32_t *slice_start,
                           int32_t n_slices, V *fvals, uint16_t *fidx)
{
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)n_slices * 32) return;
    int sl = (int)(t / 32), lane = (int)(t % 32);
    int s = sl_seg[t];
    int len = s >= 0 ? seg_len[s] : 0;
    int64_t base = slice_start[sl];
    int64_t nent = ((int64_t)slice_start[sl + 1] - base) / 32;  // entries per lane
    uint16_t last = 0;
    if (len > 0) last = fidx[base + (((int64_t)(len - 1) >> 2) * 32 + lane) * 4 + ((len - 1) & 3)];
    for (int64_t e = len; e < nent; ++e) {
        int64_t pos = base + ((e >> 2) * 32 + lane) * 4 + (e & 3);
        fvals[pos] = (V)0;
        fidx[pos] = last;
    }
}

// Step codes of the forward store (strip panels).  A segment is one ray's run
// through a super tile; its entries arrive sorted by (ix, iy).  The ray walks
// monotonically, so the runs of equal ix are contiguous, adjacent, and all go
// the same way in iy.  Reversing every run when the ray goes down in iy puts
// the entries in walk order (ix ascending), where each entry is its
// predecessor moved by 0 (first entry / padding), s (row step), w (next strip
// row) or w + s (through a corner: the zero-length voxel is not stored).
// Phase B then reads 2 bits per entry instead of a 16-bit index.  A segment
// that does not fit (a capped run cut inside a descending ix run) is flagged
// in fq0 (bit 17) and read through its 16-bit indices; *bad counts them.
template <typename V>
__global__ void fcode_k(const int32_t *seg_key, const int32_t *seg_len, const int32_t *seg_slice,
                        const int32_t *seg_lane, const int32_t *slice_start,
                        const int32_t *st_ptr, int32_t n_seg, int32_t n_rows, int32_t h,
                        int swz_shift, V *fvals, uint16_t *fidx, uint32_t *fcode, int32_t *fq0,
                        int *bad)
{
    const int sg = blockIdx.x * blockDim.x + threadIdx.x;
    if (sg >= n_seg) return;
    const int st = seg_key[sg] / n_rows, K = seg_len[sg];
    const int w = (st_ptr[st + 1] - st_ptr[st]) / h;
    const int sl = seg_slice[sg], lane = seg_lane[sg];
    const int64_t base = slice_start[sl];
    auto pos = [&](int e) { return base + ((int64_t)(e >> 2) * 32 + lane) * 4 + (e & 3); };
    auto qat = [&](int e) { return swz_idx(fidx[pos(e)], swz_shift); };
    // row direction: first pair of adjacent ix runs that tells it apart
    int s = 1;
    {
        int e = 0, prev_lo = -1, prev_hi = -1;
        while (e < K) {
            const int ix = qat(e) / w;
            int f = e;
            while (f + 1 < K && qat(f + 1) / w == ix) ++f;
            const int lo = qat(e) % w, hi = qat(f) % w;
            if (prev_lo >= 0 && !(lo == hi && prev_lo == prev_hi && lo == prev_lo)) {
                s = lo >= prev_hi ? 1 : -1;
                break;
            }
            prev_lo = lo;
            prev_hi = hi;
            e = f + 1;
        }
    }
    if (s < 0) {   // reverse every run of equal ix
        int e = 0;
        while (e < K) {
            const int ix = qat(e) / w;
            int f = e;
            while (f + 1 < K && qat(f + 1) / w == ix) ++f;
            for (int a = e, b = f; a < b; ++a, --b) {
                const int64_t pa = pos(a), pb = pos(b);
                const V tv = fvals[pa]; fvals[pa] = fvals[pb]; fvals[pb] = tv;
                const uint16_t ti = fidx[pa]; fidx[pa] = fidx[pb]; fidx[pb] = ti;
            }
            e = f + 1;
        }
    }
    // codes; padding entries (value 0, the lane's last voxel) keep code 0
    auto code_of = [&](int qp, int qn) {
        const int d = qn - qp;
        if (d == s && qn / w == qp / w) return 1;
        if (d == w) return 2;
        if (d == w + s && qn / w == qp / w + 1) return 3;
        return -1;
    };
    bool ok = true;
    for (int e = 1; e < K && ok; ++e) ok = code_of(qat(e - 1), qat(e)) >= 0;
    const int64_t slot = (int64_t)sl * 32 + lane;
    if (!ok) {   // e.g. a capped run cut inside a descending ix run: keep the indices
        fq0[slot] = 1 << 17;
        atomicAdd(bad, 1);
        return;
    }
    const int64_t wbase = slice_start[sl] / 16 + 24ll * sl;
    const int nvec = (slice_start[sl + 1] - slice_start[sl]) >> 7;
    int q = K > 0 ? qat(0) : 0;
    fq0[slot] = q | (s < 0 ? 1 << 16 : 0);
    for (int kv4 = 0; kv4 < nvec; kv4 += 4) {
        uint32_t word = 0;
        for (int j = 0; j < 4; ++j)
            for (int e4 = 0; e4 < 4; ++e4) {
                const int e = (kv4 + j) * 4 + e4;
                if (e == 0 || e >= K) continue;
                const int qn = qat(e);
                word |= (uint32_t)code_of(q, qn) << (8 * j + 2 * e4);
                q = qn;
            }
        fcode[wbase + (int64_t)(kv4 >> 2) * 32 + lane] = word;
    }
}

// stbs[st*(m+1)+i] = first slice of (tile st, row block >= i)
__global__ void stbs_k(const int32_t *slice_gid, int32_t n_slices, int m, int32_t n_st,
                       int32_t *stbs)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_st * (m + 1)) return;
    stbs[t] = (int32_t)lb_i32(slice_gid, 0, n_slices, t);
}

// rows -> segments in tile order: sort segment ids by row*n_st + tile
__global__ void rkey_k(const int32_t *seg_key, int32_t n_seg, int32_t n_rows, int32_t n_st,
                       int32_t *rkey)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    rkey[s] = (seg_key[s] % n_rows) * n_st + seg_key[s] / n_rows;
}

__global__ void rq_k(const int32_t *rpos, int32_t n_seg, int32_t *rq)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < n_seg) rq[rpos[q]] = q;
}

__global__ void rpos_k(const int32_t *rseg, const int32_t *seg_slice, const int32_t *seg_lane,
                       int32_t n_seg, int32_t *rpos)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < n_seg) rpos[q] = seg_slice[rseg[q]] * 32 + seg_lane[rseg[q]];
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

// band keys: tile << 44 | row block << 32 | global row, per CSC entry in sorted
// order (ranges never cross a row block, so a partial task can zero the rest)
__global__ void band_key_k(const int32_t *perm, const int32_t *rowid, const int32_t *l2g,
                           const int32_t *rbp, int m, const int32_t *sorted_d,
                           const int32_t *tile_of_d, int64_t nnz, uint64_t *bkey)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    const int32_t lr = rowid[perm[q]];
    const int32_t g = l2g[lr];
    const int blk = (int)lb_i32(rbp, 0, m + 1, lr + 1) - 1;
    // tile (20 bits) | row block (12 bits, BCT_MAX_M) | measurement id (32 bits)
    bkey[q] = ((uint64_t)(uint32_t)tile_of_d[sorted_d[q]] << 44) | ((uint64_t)blk << 32) |
              (uint32_t)g;
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
    // (the upper 32 bits are tile and row block)
}

// per tile: first unique index (tile_u0) and first range (band_ptr)
__global__ void tile_bounds_k(const uint64_t *u, int64_t nu, const int32_t *rflag_incl,
                              int32_t n_tiles, int32_t *tile_u0, int32_t *band_ptr)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > n_tiles) return;
    int64_t q = lb_u64(u, 0, nu, (uint64_t)(uint32_t)t << 44);
    tile_u0[t] = (int32_t)q;
    // ranges before q = number of range starts in [0, q)
    band_ptr[t] = q == 0 ? 0 : rflag_incl[q - 1];
}

// Ranges are staged in 16-byte granules: range k covers the aligned
// measurement span [g0 & ~3, g0 + len rounded up to 4), alen slots, and
// starts at a band slot that is a multiple of 4 (apre = exclusive prefix of
// alen): 4 FP32 or 2 FP64 residuals per granule (bct::BAND_ALIGN).
__global__ void ranges_k(const uint64_t *u, int64_t nu, const int32_t *rflag, const int32_t *rincl,
                         int32_t *rstart, int32_t *rlen, int32_t *alen, uint16_t *band_rb)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nu || !rflag[q]) return;
    int k = rincl[q] - 1;
    band_rb[k] = (uint16_t)((u[q] >> 32) & 0xfff);
    const int32_t g0 = (int32_t)(uint32_t)u[q];
    // length: up to the next range start
    int64_t e = q + 1;
    while (e < nu && !rflag[e]) ++e;
    rstart[k] = (int32_t)q;
    rlen[k] = (int32_t)(e - q);
    constexpr int A = bct::BAND_ALIGN;
    alen[k] = ((g0 & (A - 1)) + (int32_t)(e - q) + A - 1) & ~(A - 1);
}

__global__ void range_meta_k(const uint64_t *u, const int32_t *rstart, const int32_t *rlen,
                             const int32_t *apre, const int32_t *band_ptr, int32_t n_ranges,
                             int2 *band_meta)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_ranges) return;
    const uint64_t key = u[rstart[k]];
    const int t = (int)(key >> 44);
    const int32_t pre = apre[k] - apre[band_ptr[t]];
    band_meta[k] = make_int2((int32_t)(uint32_t)key,
                             (int32_t)(((uint32_t)pre << 16) | (uint32_t)rlen[k]));
}

__global__ void gather_rows_k(const int32_t *perm, const int32_t *rowid, int64_t nnz, int32_t *out)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < nnz) out[q] = rowid[perm[q]];
}

// ---- CSC slices: 32 columns (lanes) of a tile interleaved 8 entries at a time
// -- entry e of the column in lane l of slice s at
// csl_start[s] + ((e / 8) * 32 + l) * 8 + e % 8

__global__ void cslice_len_k(const int32_t *colstart, const int32_t *corder, int32_t n_cols,
                             int32_t n_cslices, int32_t *slice_ent)
{
    int sl = blockIdx.x * blockDim.x + threadIdx.x;
    if (sl > n_cslices) return;
    if (sl == n_cslices) { slice_ent[sl] = 0; return; }
    int kmax = 0;
    for (int l = 0; l < 32; ++l) {
        int q = sl * 32 + l;
        if (q >= n_cols) break;
        int d = corder[q];
        kmax = max(kmax, (colstart[d + 1] - colstart[d] + 7) / 8);
    }
    slice_ent[sl] = kmax * 256;
}

template <typename V>
__global__ void csc_sell_scatter_k(const int32_t *perm, const double *vals64, const int32_t *sorted_d,
                                   const uint64_t *bkey, const int32_t *tile_of_d, const uint64_t *u,
                                   const int32_t *tile_u0, const int32_t *rincl,
                                   const int32_t *rstart, const int32_t *apre,
                                   const int32_t *band_ptr, const int32_t *colstart,
                                   const int32_t *dslot, const int32_t *csl_start, int64_t nnz,
                                   V *tvals, uint16_t *tloc)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    int d = sorted_d[q];
    int t = tile_of_d[d];
    int64_t bpos = lb_u64(u, tile_u0[t], tile_u0[t + 1], bkey[q]);
    int64_t e = q - colstart[d];
    int slot = dslot[d];
    int64_t dst = csl_start[slot / 32] + ((e >> 3) * 32 + (slot % 32)) * 8 + (e & 7);
    tvals[dst] = (V)vals64[perm[q]];
    const int k = rincl[bpos] - 1;   // range of the entry's row
    const int32_t g0 = (int32_t)(uint32_t)u[rstart[k]];
    tloc[dst] = (uint16_t)(apre[k] - apre[band_ptr[t]] + (g0 & (bct::BAND_ALIGN - 1)) +
                           (bpos - rstart[k]));
}

// padding of every (slice, lane): zero values on the column's last band slot
template <typename V>
__global__ void csc_sell_pad_k(const int32_t *colstart, const int32_t *corder, int32_t n_cols,
                               const int32_t *csl_start, int32_t n_cslices, V *tvals,
                               uint16_t *tloc)
{
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)n_cslices * 32) return;
    int sl = (int)(t / 32), lane = (int)(t % 32);
    int q = sl * 32 + lane;
    int len = q < n_cols ? colstart[corder[q] + 1] - colstart[corder[q]] : 0;
    int64_t base = csl_start[sl];
    int64_t nent = ((int64_t)csl_start[sl + 1] - base) / 32;
    uint16_t last = 0;
    if (len > 0) last = tloc[base + (((int64_t)(len - 1) >> 3) * 32 + lane) * 8 + ((len - 1) & 7)];
    for (int64_t e = len; e < nent; ++e) {
        int64_t pos = base + ((e >> 3) * 32 + lane) * 8 + (e & 7);
        tvals[pos] = (V)0;
        tloc[pos] = last;
    }
}

// Bank-aware order inside each lane's 8-entry vector.  Phase 1 gathers
// band[tloc] with one 8-byte shared load per entry position e: a half-warp
// (16 lanes) is one 128-byte wavefront when its 16 slots fall in distinct
// bank pairs (slot mod 16) or repeat an address, and one more wavefront per
// extra distinct slot in a bank pair otherwise.  The order of a lane's 8
// entries is free (it only reorders that lane's fma chain), so a warp per
// vector row assigns, position by position and lane by lane, the remaining
// entry that adds the fewest wavefronts; zero padding entries take the slot
// another lane already reads (a broadcast).
// FP32 mode stages FP32 bands for the batched path: one 4-byte load per
// entry, one wavefront per warp when the 32 slots fall in distinct banks
// (slot mod 32) -- the same greedy over the whole warp (nbank = 32).
template <typename V>
__global__ void csc_bank_perm_k(V *tvals, uint16_t *tloc, const int32_t *csl_start,
                                int32_t n_cslices, int nbank)
{
    constexpr int WPB = 4;
    __shared__ int cnt_s[WPB][2][32];
    __shared__ int first_s[WPB][2][32];
    __shared__ int any_s[WPB][2];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * WPB + wib, nw = gridDim.x * WPB;
    const int grp = nbank == 32 ? 0 : lane >> 4, bmask = nbank - 1;
    int *cnt = &cnt_s[wib][grp][0];
    int *first = &first_s[wib][grp][0];
    for (int sl = gw; sl < n_cslices; sl += nw) {
        const int64_t base0 = csl_start[sl];
        const int nvr = (int)((csl_start[sl + 1] - base0) >> 8);
        for (int u = 0; u < nvr; ++u) {
            const int64_t base = base0 + (int64_t)u * 256 + lane * 8;
            V val[8];
            int loc[8];
            for (int e = 0; e < 8; ++e) {
                val[e] = tvals[base + e];
                loc[e] = tloc[base + e];
            }
            V oval[8];
            int oloc[8];
            unsigned left = 0xffu;
            for (int e = 0; e < 8; ++e) {
                cnt_s[wib][0][lane] = 0;
                cnt_s[wib][1][lane] = 0;
                if (lane < 2) any_s[wib][lane] = -1;
                __syncwarp();
                for (int who = 0; who < 32; ++who) {
                    if (lane == who) {
                        int best = -1, bcost = 1 << 30, pad = -1;
                        for (int j = 0; j < 8; ++j) {
                            if (!((left >> j) & 1u)) continue;
                            if (val[j] == (V)0) {
                                if (pad < 0) pad = j;
                                continue;
                            }
                            const int b = loc[j] & bmask;
                            const int c = (cnt[b] == 0 || first[b] == loc[j]) ? 0 : cnt[b];
                            if (c < bcost) {
                                bcost = c;
                                best = j;
                            }
                        }
                        int pick = best;
                        int a = best >= 0 ? loc[best] : 0;
                        if (pad >= 0 && (best < 0 || bcost > 0)) {
                            pick = pad;   // a zero entry: read a slot already read
                            const int an = any_s[wib][grp];
                            a = an >= 0 ? an : (best >= 0 ? loc[best] : loc[pad]);
                        }
                        const int b = a & bmask;
                        if (cnt[b] == 0) {
                            cnt[b] = 1;
                            first[b] = a;
                        } else if (first[b] != a) {
                            ++cnt[b];
                        }
                        if (any_s[wib][grp] < 0) any_s[wib][grp] = a;
                        oval[e] = val[pick];
                        oloc[e] = a;
                        left &= ~(1u << pick);
                    }
                    __syncwarp();
                }
            }
            for (int e = 0; e < 8; ++e) {
                tvals[base + e] = oval[e];
                tloc[base + e] = (uint16_t)oloc[e];
            }
        }
    }
}

// The same greedy as csc_bank_perm_k, one thread per vector row (the 32
// virtual lanes of a row walked in order by that thread, the counters in
// thread-private shared memory) instead of one lane at a time in a warp:
// bit-identical output, all threads busy (config 4: 535 ms -> a few ms).
constexpr int BP_TPB = 128;
template <typename V>
__global__ void __launch_bounds__(BP_TPB) csc_bank_perm_rows_k(const V *tv_in,
                                                               const uint16_t *tl_in, V *tv_out,
                                                               uint16_t *tl_out, int64_t n_vrows,
                                                               int nbank)
{
    __shared__ uint8_t cnt_s[2][32][BP_TPB];
    __shared__ uint16_t first_s[2][32][BP_TPB];
    __shared__ uint8_t left_s[32][BP_TPB];
    const int t = threadIdx.x;
    const int64_t r = blockIdx.x * (int64_t)BP_TPB + t;
    if (r >= n_vrows) return;
    const int64_t base0 = r * 256;
    const int bmask = nbank - 1;
    for (int L = 0; L < 32; ++L) left_s[L][t] = 0xff;
    for (int e = 0; e < 8; ++e) {
        for (int b = 0; b < 32; ++b) {
            cnt_s[0][b][t] = 0;
            cnt_s[1][b][t] = 0;
        }
        int any[2] = {-1, -1};
        for (int L = 0; L < 32; ++L) {
            const int g = nbank == 32 ? 0 : (L >> 4);
            const int64_t base = base0 + L * 8;
            const unsigned left = left_s[L][t];
            int best = -1, bcost = 1 << 30, pad = -1;
            for (int j = 0; j < 8; ++j) {
                if (!((left >> j) & 1u)) continue;
                if (tv_in[base + j] == (V)0) {
                    if (pad < 0) pad = j;
                    continue;
                }
                const int lj = tl_in[base + j];
                const int b = lj & bmask;
                const int cb = cnt_s[g][b][t];
                const int c = (cb == 0 || first_s[g][b][t] == lj) ? 0 : cb;
                if (c < bcost) {
                    bcost = c;
                    best = j;
                }
            }
            int pick = best;
            int a = best >= 0 ? tl_in[base + best] : 0;
            if (pad >= 0 && (best < 0 || bcost > 0)) {
                pick = pad;   // a zero entry: read a slot already read
                const int an = any[g];
                a = an >= 0 ? an : (best >= 0 ? tl_in[base + best] : tl_in[base + pad]);
            }
            const int b = a & bmask;
            if (cnt_s[g][b][t] == 0) {
                cnt_s[g][b][t] = 1;
                first_s[g][b][t] = (uint16_t)a;
            } else if (first_s[g][b][t] != a) {
                ++cnt_s[g][b][t];
            }
            if (any[g] < 0) any[g] = a;
            tv_out[base + e] = tv_in[base + pick];
            tl_out[base + e] = (uint16_t)a;
            left_s[L][t] = (uint8_t)(left & ~(1u << pick));
        }
    }
}

// Delta form of tloc: per lane-vector (8 entries) a 16-bit base (the smallest
// slot of its nonzero entries) and 8-bit offsets; zero (padding) entries read
// the base.  Flags a vector whose span does not fit 8 bits.
template <typename V>
__global__ void tloc_delta_k(const V *tvals, const uint16_t *tloc, int64_t n_vec, uint8_t *toff,
                             uint16_t *tbase, int *overflow)
{
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n_vec) return;
    int lo = 1 << 30, hi = -1;
    for (int e = 0; e < 8; ++e)
        if (tvals[q * 8 + e] != (V)0) {
            lo = min(lo, (int)tloc[q * 8 + e]);
            hi = max(hi, (int)tloc[q * 8 + e]);
        }
    if (hi < 0) lo = hi = tloc[q * 8];   // all padding
    if (hi - lo > 255) atomicOr(overflow, 1);
    tbase[q] = (uint16_t)lo;
    for (int e = 0; e < 8; ++e) {
        const int d = tvals[q * 8 + e] != (V)0 ? (int)tloc[q * 8 + e] - lo : 0;
        toff[q * 8 + e] = (uint8_t)min(d, 255);
    }
}

// cptr[d*(m+1)+i] = column-local index of column d's first entry with local row >= rbp[i]
__global__ void cptr_local_k(const int32_t *colstart, const int32_t *tlocal_sorted,
                             const int32_t *rbp, int m, int32_t n_cols, int32_t *cptr)
{
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)n_cols * (m + 1)) return;
    int d = (int)(t / (m + 1)), i = (int)(t % (m + 1));
    int64_t lb = lb_i32(tlocal_sorted, colstart[d], colstart[d + 1], rbp[i]);
    cptr[t] = (int32_t)(lb - colstart[d]);
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
                    int tile_cols, PanelDev &P, std::vector<void *> &keep, std::string &err,
                    cudaStream_t s)
{
    std::vector<void *> tmp;
    Alloc K{&keep, &err}, T{&tmp, &err};
    const int vs = dtype == 0 ? 8 : 4;
    const int32_t n_st = (int32_t)st_ptr_h.size() - 1;
    const int32_t n_tiles = (int32_t)((corder_h.size() + tile_cols - 1) / tile_cols);
    if (n_tiles >= (1 << 20) || m > BCT_MAX_M) {   // band key fields (band_key_k)
        err = "panel exceeds 2^20 tiles or BCT_MAX_M row blocks";
        return -1;
    }

    // host tables -> device
    std::vector<int32_t> d2st_h(n_cols), tile_of_d_h(n_cols);
    for (int st = 0; st < n_st; ++st)
        for (int d = st_ptr_h[st]; d < st_ptr_h[st + 1]; ++d) d2st_h[d] = st;
    for (size_t q = 0; q < corder_h.size(); ++q) tile_of_d_h[corder_h[q]] = (int32_t)(q / tile_cols);
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
        seg_flag_k<<<nb(nnz, 256), 256, 0, s>>>(skey, nnz, P.seg_cap > 0 ? P.seg_cap : SEG_CAP,
                                                 flag);
        LCK(scan_i32(flag, incl, nnz, true, tmp, s));
        n_seg = read1(incl + nnz - 1, s);
    }
    int32_t *seg_first = T.get<int32_t>(n_seg + 1), *seg_key = K.get<int32_t>(n_seg + 1);
    int32_t *seg_len = K.get<int32_t>(n_seg + 1), *nvec = T.get<int32_t>(n_seg + 1);
    int32_t *seg_slice = K.get<int32_t>(n_seg + 1), *seg_lane = K.get<int32_t>(n_seg + 1);
    uint64_t *skey0 = T.get<uint64_t>(n_seg + 1), *skey1 = T.get<uint64_t>(n_seg + 1);
    int32_t *sid0 = T.get<int32_t>(n_seg + 1), *sseg = T.get<int32_t>(n_seg + 1);
    int32_t *sflag = T.get<int32_t>(n_seg + 1), *sincl = T.get<int32_t>(n_seg + 1);
    LNN(seg_first); LNN(seg_key); LNN(seg_len); LNN(nvec); LNN(seg_slice); LNN(seg_lane);
    LNN(skey0); LNN(skey1); LNN(sid0); LNN(sseg); LNN(sflag); LNN(sincl);
    int32_t n_slices = 0;
    if (n_seg > 0) {
        seg_first_k<<<nb(nnz, 256), 256, 0, s>>>(flag, incl, skey, nnz, seg_first, seg_key);
        seg_len_k<<<nb(n_seg, 256), 256, 0, s>>>(seg_first, n_seg, nnz, seg_len, nvec);
        sell_key_k<<<nb(n_seg, 256), 256, 0, s>>>(seg_key, nvec, n_seg, n_rows, rbp, m, skey0);
        iota_k<<<nb(n_seg, 256), 256, 0, s>>>(sid0, n_seg);
        {
            size_t b = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, b, skey0, skey1, sid0, sseg, (int)n_seg, 0, 64, s);
            void *tt = T.get<char>((int64_t)b + 16);
            LNN(tt);
            LCK(cub::DeviceRadixSort::SortPairs(tt, b, skey0, skey1, sid0, sseg, (int)n_seg, 0, 64, s));
        }
        slice_flag_k<<<nb(n_seg, 256), 256, 0, s>>>(skey1, n_seg, sflag);
        LCK(scan_i32(sflag, sincl, n_seg, true, tmp, s));
        n_slices = read1(sincl + n_seg - 1, s);
    }
    int32_t *sl_seg = K.get<int32_t>((int64_t)n_slices * 32 + 1);
    int32_t *slice_len = T.get<int32_t>(n_slices + 1), *slice_start = K.get<int32_t>(n_slices + 1);
    int32_t *slice_gid = K.get<int32_t>(n_slices + 1);
    int32_t *stbs = K.get<int32_t>((int64_t)n_st * (m + 1) + 1);
    LNN(sl_seg); LNN(slice_len); LNN(slice_start); LNN(slice_gid); LNN(stbs);
    LCK(cudaMemsetAsync(sl_seg, 0xff, 4 * ((int64_t)n_slices * 32 + 1), s));
    int64_t fwd_cap = 0;
    if (n_slices > 0) {
        slice_info_k<<<nb(n_seg, 256), 256, 0, s>>>(skey1, sseg, sincl, nvec, n_seg, seg_slice,
                                                    seg_lane, sl_seg, slice_len, slice_gid);
        LCK(cudaMemsetAsync(slice_len + n_slices, 0, 4, s));
        LCK(scan_i32(slice_len, slice_start, n_slices + 1, false, tmp, s));
        fwd_cap = read1(slice_start + n_slices, s);
        if (getenv("BCT_VERBOSE"))
            fprintf(stderr, "forward store: %lld entries in %d slices for %lld stored (%.2f%% padding)\n",
                    (long long)fwd_cap, n_slices, (long long)nnz,
                    nnz > 0 ? 100.0 * ((double)fwd_cap / (double)nnz - 1.0) : 0.0);
    } else {
        LCK(cudaMemsetAsync(slice_start, 0, 4, s));
    }
    if (fwd_cap >= (1ll << 31)) {
        err = "panel forward store exceeds 2^31 entries";
        release(tmp);
        return -1;
    }
    void *fvals = K.get<char>(std::max<int64_t>(fwd_cap, 1) * vs);
    uint16_t *fidx = K.get<uint16_t>(fwd_cap);
    LNN(fvals); LNN(fidx);
    if (n_slices > 0) {
        if (dtype == 0) {
            sell_scatter_k<double><<<nb(nnz, 256), 256, 0, s>>>(perm, incl, seg_first, seg_key,
                seg_slice, seg_lane, slice_start, vals64, cols_c, c2d, st_ptr, n_rows, nnz,
                (double *)fvals, fidx, P.swz_shift);
            sell_pad_k<double><<<nb((int64_t)n_slices * 32, 256), 256, 0, s>>>(sl_seg, seg_len,
                slice_start, n_slices, (double *)fvals, fidx);
        } else {
            sell_scatter_k<float><<<nb(nnz, 256), 256, 0, s>>>(perm, incl, seg_first, seg_key,
                seg_slice, seg_lane, slice_start, vals64, cols_c, c2d, st_ptr, n_rows, nnz,
                (float *)fvals, fidx, P.swz_shift);
            sell_pad_k<float><<<nb((int64_t)n_slices * 32, 256), 256, 0, s>>>(sl_seg, seg_len,
                slice_start, n_slices, (float *)fvals, fidx);
        }
    }
    // step codes of strip panels (phase B); BCT_NO_FCODE keeps the indices
    uint32_t *fcode = nullptr;
    int32_t *fq0 = nullptr;
    if (P.st_h > 0 && n_seg > 0 && !getenv("BCT_NO_FCODE")) {
        const int64_t n_words = fwd_cap / 16 + 24ll * n_slices + 32;
        uint32_t *fc = K.get<uint32_t>(n_words);
        int32_t *fq = K.get<int32_t>((int64_t)n_slices * 32 + 1);
        int *bad = T.get<int>(1);
        LNN(fc); LNN(fq); LNN(bad);
        LCK(cudaMemsetAsync(fc, 0, 4 * n_words, s));
        LCK(cudaMemsetAsync(fq, 0, 4 * ((int64_t)n_slices * 32 + 1), s));
        LCK(cudaMemsetAsync(bad, 0, 4, s));
        if (dtype == 0)
            fcode_k<double><<<nb(n_seg, 128), 128, 0, s>>>(seg_key, seg_len, seg_slice, seg_lane,
                slice_start, st_ptr, n_seg, n_rows, P.st_h, P.swz_shift, (double *)fvals, fidx,
                fc, fq, bad);
        else
            fcode_k<float><<<nb(n_seg, 128), 128, 0, s>>>(seg_key, seg_len, seg_slice, seg_lane,
                slice_start, st_ptr, n_seg, n_rows, P.st_h, P.swz_shift, (float *)fvals, fidx,
                fc, fq, bad);
        LCK(cudaGetLastError());
        fcode = fc;
        fq0 = fq;
        if (getenv("BCT_VERBOSE"))
            fprintf(stderr, "fcode: %d of %d segments keep indices\n", read1(bad, s), n_seg);
    }
    stbs_k<<<nb((int64_t)n_st * (m + 1), 128), 128, 0, s>>>(slice_gid, n_slices, m, n_st, stbs);
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
    // the epoch kernel stores segment partials in SELL order (slice*32 +
    // lane: coalesced stores in phase 2); rpos lists each row's partials
    int32_t *rpos = K.get<int32_t>(n_seg + 1);
    LNN(rpos);
    if (n_seg > 0)
        rpos_k<<<nb(n_seg, 256), 256, 0, s>>>(rseg, seg_slice, seg_lane, n_seg, rpos);
    // and its inverse per SELL slot: the batched phase B stores each partial
    // at its row-order position, so phase C reads every row's partials
    // contiguously
    int32_t *rq = K.get<int32_t>((int64_t)n_slices * 32 + 1);
    LNN(rq);
    LCK(cudaMemsetAsync(rq, 0xff, 4 * ((int64_t)n_slices * 32 + 1), s));
    if (n_seg > 0) rq_k<<<nb(n_seg, 256), 256, 0, s>>>(rpos, n_seg, rq);
    LCK(cudaGetLastError());

    // ================= CSC with tile bands =================
    int32_t *sd = T.get<int32_t>(nnz), *cperm = T.get<int32_t>(nnz);
    int32_t *colstart = T.get<int32_t>(n_cols + 1);
    int32_t *len8 = T.get<int32_t>(n_cols + 1);
    LNN(sd); LNN(cperm); LNN(colstart); LNN(len8);
    if (nnz > 0) {
        csc_key_k<<<nb(nnz, 256), 256, 0, s>>>(cols_c, c2d, nnz, key);
        LCK(sort_pairs<int32_t>(key, sd, iota, cperm, nnz, bits_for(n_cols), tmp, s));
    }
    colcount_k<<<nb(n_cols + 1, 256), 256, 0, s>>>(sd, nnz, n_cols, colstart, len8);
    // slices of 32 columns in tile order
    const int32_t n_cslices = (n_cols + 31) / 32;
    int32_t *slice_ent = T.get<int32_t>(n_cslices + 1), *csl_start = K.get<int32_t>(n_cslices + 1);
    int32_t *dslot = T.get<int32_t>(n_cols);
    LNN(slice_ent); LNN(csl_start); LNN(dslot);
    std::vector<int32_t> co(corder_h);
    {
        // the columns of a tile in descending entry count (stable): a
        // 32-column slice is stored as its longest column's vector rows, so
        // grouping like lengths cuts the padding phase 1 streams (config 4:
        // 2.9% -> 0.5%).  Only the order inside a tile moves: bands, tiles
        // and each column's own sum are unchanged.  (BCT_CSC_SORT=0: off)
        const char *cs_env = getenv("BCT_CSC_SORT");
        if (!(cs_env && cs_env[0] == '0') && n_cols > 0) {
            std::vector<int32_t> cs(n_cols + 1);
            LCK(cudaMemcpyAsync(cs.data(), colstart, 4 * ((int64_t)n_cols + 1),
                                cudaMemcpyDeviceToHost, s));
            LCK(cudaStreamSynchronize(s));
            for (size_t t0 = 0; t0 < co.size(); t0 += tile_cols) {
                const size_t t1 = std::min(co.size(), t0 + (size_t)tile_cols);
                std::stable_sort(co.begin() + t0, co.begin() + t1, [&](int32_t a, int32_t b) {
                    return cs[a + 1] - cs[a] > cs[b + 1] - cs[b];
                });
            }
            LCK(cudaMemcpyAsync(corder, co.data(), 4 * (int64_t)n_cols, cudaMemcpyHostToDevice, s));
        }
        std::vector<int32_t> ds(n_cols);
        for (size_t q = 0; q < co.size(); ++q) ds[co[q]] = (int32_t)q;
        LCK(cudaMemcpyAsync(dslot, ds.data(), 4 * n_cols, cudaMemcpyHostToDevice, s));
        LCK(cudaStreamSynchronize(s));
    }
    cslice_len_k<<<nb(n_cslices + 1, 128), 128, 0, s>>>(colstart, corder, n_cols, n_cslices,
                                                       slice_ent);
    LCK(scan_i32(slice_ent, csl_start, n_cslices + 1, false, tmp, s));
    int64_t csc_cap = read1(csl_start + n_cslices, s);
    if (getenv("BCT_VERBOSE"))
        fprintf(stderr, "csc store: %lld entries in %d slices for %lld stored (%.2f%% padding)\n",
                (long long)csc_cap, n_cslices, (long long)nnz,
                nnz > 0 ? 100.0 * ((double)csc_cap / (double)nnz - 1.0) : 0.0);
    if (csc_cap >= (1ll << 31)) {
        err = "panel CSC exceeds 2^31 entries";
        release(tmp);
        return -1;
    }
    // bands
    uint64_t *bkey = T.get<uint64_t>(nnz), *bsorted = T.get<uint64_t>(nnz);
    LNN(bkey); LNN(bsorted);
    int64_t nu = 0;
    if (nnz > 0) {
        band_key_k<<<nb(nnz, 256), 256, 0, s>>>(cperm, rowid, l2g, rbp, m, sd, tile_of_d, nnz,
                                                 bkey);
        LCK(sort_keys_u64(bkey, bsorted, nnz, 44 + bits_for(n_tiles), tmp, s));
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
    int32_t *band_ptr = K.get<int32_t>(n_tiles + 1);
    int2 *band_meta = K.get<int2>(n_ranges + 1);
    uint16_t *band_rb = K.get<uint16_t>(n_ranges + 1);
    int32_t *rstart = T.get<int32_t>(n_ranges + 1), *rlen = T.get<int32_t>(n_ranges + 1);
    int32_t *alen = T.get<int32_t>(n_ranges + 1), *apre = T.get<int32_t>(n_ranges + 1);
    LNN(band_ptr); LNN(band_meta); LNN(band_rb); LNN(rstart); LNN(rlen); LNN(alen); LNN(apre);
    tile_bounds_k<<<nb(n_tiles + 1, 128), 128, 0, s>>>(uk, nu, rincl, n_tiles, tile_u0, band_ptr);
    LCK(cudaMemsetAsync(alen + n_ranges, 0, 4, s));
    if (n_ranges > 0)
        ranges_k<<<nb(nu, 256), 256, 0, s>>>(uk, nu, rflag, rincl, rstart, rlen, alen, band_rb);
    LCK(scan_i32(alen, apre, n_ranges + 1, false, tmp, s));
    if (n_ranges > 0)
        range_meta_k<<<nb(n_ranges, 256), 256, 0, s>>>(uk, rstart, rlen, apre, band_ptr, n_ranges,
                                                       band_meta);
    // the widest band sets the shared-memory size
    std::vector<int32_t> bp(n_tiles + 1), ap(n_ranges + 1);
    LCK(cudaMemcpyAsync(bp.data(), band_ptr, 4 * (n_tiles + 1), cudaMemcpyDeviceToHost, s));
    LCK(cudaMemcpyAsync(ap.data(), apre, 4 * (n_ranges + 1), cudaMemcpyDeviceToHost, s));
    LCK(cudaStreamSynchronize(s));
    int32_t band_max = 0;
    for (int t = 0; t < n_tiles; ++t) band_max = std::max(band_max, ap[bp[t + 1]] - ap[bp[t]]);
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
            csc_sell_scatter_k<double><<<nb(nnz, 256), 256, 0, s>>>(cperm, vals64, sd, bkey,
                tile_of_d, uk, tile_u0, rincl, rstart, apre, band_ptr, colstart, dslot,
                csl_start, nnz, (double *)tvals, tloc);
        else
            csc_sell_scatter_k<float><<<nb(nnz, 256), 256, 0, s>>>(cperm, vals64, sd, bkey,
                tile_of_d, uk, tile_u0, rincl, rstart, apre, band_ptr, colstart, dslot,
                csl_start, nnz, (float *)tvals, tloc);
        gather_rows_k<<<nb(nnz, 256), 256, 0, s>>>(cperm, rowid, nnz, tls);
    }
    if (dtype == 0)
        csc_sell_pad_k<double><<<nb((int64_t)n_cslices * 32, 256), 256, 0, s>>>(colstart, corder,
            n_cols, csl_start, n_cslices, (double *)tvals, tloc);
    else
        csc_sell_pad_k<float><<<nb((int64_t)n_cslices * 32, 256), 256, 0, s>>>(colstart, corder,
            n_cols, csl_start, n_cslices, (float *)tvals, tloc);
    cptr_local_k<<<nb((int64_t)n_cols * (m + 1), 256), 256, 0, s>>>(colstart, tls, rbp, m, n_cols,
                                                                   cptr);
    if (!getenv("BCT_NO_BANK_PERM") && n_cslices > 0) {
        const int nbank = dtype == 0 ? 16 : (getenv("BCT_BANK16") ? 16 : 32);
        if (getenv("BCT_OLD_BANK_PERM")) {   // the warp-serial original (checking only)
            const unsigned pb = (unsigned)std::min<int64_t>((n_cslices + 3) / 4, 4096);
            if (dtype == 0)
                csc_bank_perm_k<double><<<pb, 128, 0, s>>>((double *)tvals, tloc, csl_start,
                                                           n_cslices, nbank);
            else
                csc_bank_perm_k<float><<<pb, 128, 0, s>>>((float *)tvals, tloc, csl_start,
                                                          n_cslices, nbank);
        } else if (csc_cap > 0) {
            // out of place into temporaries, then copied back
            const int64_t n_vrows = csc_cap / 256;
            void *tv2 = T.get<char>(csc_cap * vs);
            uint16_t *tl2 = T.get<uint16_t>(csc_cap);
            LNN(tv2); LNN(tl2);
            const unsigned gb = (unsigned)((n_vrows + BP_TPB - 1) / BP_TPB);
            if (dtype == 0)
                csc_bank_perm_rows_k<double><<<gb, BP_TPB, 0, s>>>(
                    (const double *)tvals, tloc, (double *)tv2, tl2, n_vrows, nbank);
            else
                csc_bank_perm_rows_k<float><<<gb, BP_TPB, 0, s>>>(
                    (const float *)tvals, tloc, (float *)tv2, tl2, n_vrows, nbank);
            LCK(cudaMemcpyAsync(tvals, tv2, csc_cap * vs, cudaMemcpyDeviceToDevice, s));
            LCK(cudaMemcpyAsync(tloc, tl2, csc_cap * 2, cudaMemcpyDeviceToDevice, s));
        }
    }
    LCK(cudaGetLastError());
    // 8-bit band offsets when every lane-vector spans < 256 slots (strip tiles)
    uint8_t *toff = nullptr;
    uint16_t *tbase = nullptr;
    if (!getenv("BCT_NO_TLOC_DELTA") && csc_cap > 0) {
        const int64_t n_vec = csc_cap / 8;
        uint8_t *to = K.get<uint8_t>(csc_cap);
        uint16_t *tb = K.get<uint16_t>(n_vec);
        int *ovf = T.get<int>(1);
        LNN(to); LNN(tb); LNN(ovf);
        LCK(cudaMemsetAsync(ovf, 0, 4, s));
        if (dtype == 0)
            tloc_delta_k<double><<<nb(n_vec, 256), 256, 0, s>>>((const double *)tvals, tloc, n_vec,
                                                               to, tb, ovf);
        else
            tloc_delta_k<float><<<nb(n_vec, 256), 256, 0, s>>>((const float *)tvals, tloc, n_vec,
                                                              to, tb, ovf);
        if (read1(ovf, s) == 0) {
            toff = to;
            tbase = tb;
        }
    }
    LCK(cudaStreamSynchronize(s));
    release(tmp);

    P.toff = toff;
    P.tbase = tbase;
    P.fvals = fvals;
    P.fidx = fidx;
    P.fcode = fcode;
    P.fq0 = fq0;
    P.slice_start = slice_start;
    P.sl_seg = sl_seg;
    P.stbs = stbs;
    P.seg_key = seg_key;
    P.seg_len = seg_len;
    P.seg_slice = seg_slice;
    P.seg_lane = seg_lane;
    P.st_ptr = st_ptr;
    P.rseg_ptr = rseg_ptr;
    P.rseg = rseg;
    P.rpos = rpos;
    P.rq = rq;
    P.tvals = tvals;
    P.csl_start = csl_start;
    P.n_cslices = n_cslices;
    P.tloc = tloc;
    P.cptr = cptr;
    P.corder = corder;
    P.band_ptr = band_ptr;
    P.band_meta = band_meta;
    P.band_rb = band_rb;
    P.n_seg = n_seg;
    P.n_slices = n_slices;
    P.n_st = n_st;
    P.n_tiles = n_tiles;
    P.band_max = band_max;
    int32_t st_max = 0;
    for (int st = 0; st < n_st; ++st) st_max = std::max(st_max, st_ptr_h[st + 1] - st_ptr_h[st]);
    P.st_max = st_max;
    P.fwd_cap = fwd_cap;
    P.csc_cap = csc_cap;
    P.tile_cols = tile_cols;
    return 0;
}

}  // namespace bct
