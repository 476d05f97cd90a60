// builder.cu -- device construction of the blocked store (compiled with
// -fmad=false: the tracer must round exactly like the reference).
//
//   pb_count_kernel / pb_fill_kernel
//       the Siddon/Amanatides-Woo traversal of projector.py:51-198 on one
//       (ray, strip) pair, with the same half-open boundary rule, probe
//       offset, step order and segment arithmetic.  The reference finishes
//       with an insertion sort by local index; local ids (ix-x0)*n + iy are
//       distinct and the traversal is monotone in ix and, within one ix
//       column, monotone in iy, so pb_fill_kernel writes every entry straight
//       to its sorted slot instead (same result, O(len) instead of O(len^2)).
//   inverse row map and the bitwise forward / z-fill / projection-sum
//   kernels used for state set-up (projector.py:220-244, 756-777); the panel
//   layout itself is built in layout.cu.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "internal.h"

namespace {

constexpr double REL_EPS = 1e-12;

struct RayTrace {
    double length, t0, t1, t;
    double tmax[3], tdel[3];
    int64_t iv[3], step[3];
    int64_t lo[3], hi[3];
    int64_t max_steps;
    bool hit;
};

__device__ __forceinline__ void pb_endpoints(int64_t n, int64_t bins, double c, double s,
                                             int64_t k, double *src, double *dst)
{
    double u = (double)k - (double)(bins - 1) / 2.0;
    double L = 4.0 * (double)n;
    double cx = u * (-s), cy = u * c;
    double lc = L * c, ls = L * s;
    src[0] = cx - lc; src[1] = cy - ls; src[2] = 0.0;
    dst[0] = cx + lc; dst[1] = cy + ls; dst[2] = 0.0;
}

// Set-up half of the traversal (projector.py:59-145).  Returns false on a miss.
// vsize = 1 on the parallel-beam harness; the general scan passes the grid's.
template <bool UNIT>
__device__ bool trace_init_t(const double *src, const double *dst, const double *origin,
                             const double *vsize, const int64_t *lo, const int64_t *hi,
                             RayTrace &T, double *dv)
{
    dv[0] = dst[0] - src[0];
    dv[1] = dst[1] - src[1];
    dv[2] = dst[2] - src[2];
    T.length = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
    if (T.length == 0.0) return false;
    double scale = fabs(dv[0]);
    if (fabs(dv[1]) > scale) scale = fabs(dv[1]);
    if (fabs(dv[2]) > scale) scale = fabs(dv[2]);
    double eps_d = REL_EPS * scale;
    double t0 = 0.0, t1 = 1.0;
    for (int a = 0; a < 3; ++a) {
        const double vs = UNIT ? 1.0 : vsize[a];
        double d = dv[a], s = src[a];
        double blo = origin[a] + (double)lo[a] * vs;
        double bhi = origin[a] + (double)hi[a] * vs;
        if (fabs(d) > eps_d) {
            double ta = (blo - s) / d, tb = (bhi - s) / d;
            if (ta > tb) { double t = ta; ta = tb; tb = t; }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        } else if (!(blo <= s && s < bhi)) {
            return false;
        }
    }
    if (t1 - t0 <= REL_EPS) return false;
    double probe = t0 + 1e-9 * (t1 - t0);
    for (int a = 0; a < 3; ++a) {
        int64_t c = (int64_t)floor((src[a] + probe * dv[a] - origin[a]) / (UNIT ? 1.0 : vsize[a]));
        if (c < lo[a]) c = lo[a];
        if (c > hi[a] - 1) c = hi[a] - 1;
        T.iv[a] = c;
        T.lo[a] = lo[a];
        T.hi[a] = hi[a];
    }
    for (int a = 0; a < 3; ++a) {
        T.step[a] = 0;
        T.tmax[a] = INFINITY;
        T.tdel[a] = INFINITY;
        if (fabs(dv[a]) > eps_d) {
            bool pos = dv[a] > 0.0;
            T.step[a] = pos ? 1 : -1;
            int64_t plane = pos ? T.iv[a] + 1 : T.iv[a];
            const double vs = UNIT ? 1.0 : vsize[a];
            T.tmax[a] = (origin[a] + (double)plane * vs - src[a]) / dv[a];
            T.tdel[a] = vs / fabs(dv[a]);
        }
    }
    T.t0 = t0;
    T.t1 = t1;
    T.t = t0;
    T.max_steps = (hi[0] - lo[0]) + (hi[1] - lo[1]) + (hi[2] - lo[2]) + 3;
    return true;
}

__device__ __forceinline__ bool trace_init(const double *src, const double *dst,
                                           const double *origin, const int64_t *lo,
                                           const int64_t *hi, RayTrace &T, double *dv)
{
    return trace_init_t<true>(src, dst, origin, nullptr, lo, hi, T, dv);
}

// One traversal; calls emit(ix, iy, seg) for every positive segment.
template <typename F>
__device__ void trace_walk(RayTrace &T, F emit)
{
    for (int64_t it = 0; it < T.max_steps; ++it) {
        int a = 0;
        double tm = T.tmax[0];
        if (T.tmax[1] < tm) { a = 1; tm = T.tmax[1]; }
        if (T.tmax[2] < tm) { a = 2; tm = T.tmax[2]; }
        double tn = tm < T.t1 ? tm : T.t1;
        double seg = (tn - T.t) * T.length;
        if (seg > 0.0) emit(T.iv[0], T.iv[1], seg);
        if (tm >= T.t1) break;
        T.iv[a] += T.step[a];
        if (T.iv[a] < T.lo[a] || T.iv[a] >= T.hi[a]) break;
        T.tmax[a] += T.tdel[a];
        T.t = tn;
    }
}

__global__ void pb_count_kernel(int64_t n, int64_t views, int64_t bins, const double *cosv,
                                const double *sinv, int64_t x0, int64_t x1, int32_t *counts)
{
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= views * bins) return;
    double src[3], dst[3], dv[3];
    int64_t a = r / bins, k = r % bins;
    pb_endpoints(n, bins, cosv[a], sinv[a], k, src, dst);
    double origin[3] = {-0.5 * (double)n, -0.5 * (double)n, -0.5};
    int64_t lo[3] = {x0, 0, 0}, hi[3] = {x1, n, 1};
    RayTrace T;
    int cnt = 0;
    if (trace_init(src, dst, origin, lo, hi, T, dv))
        trace_walk(T, [&](int64_t, int64_t, double) { ++cnt; });
    counts[r] = cnt;
}

// trace_walk one positive segment at a time (the same arithmetic in the same
// order); false when the traversal has ended.
struct TraceIter {
    int64_t it = 0;
    bool done = false;
};

__device__ __forceinline__ bool trace_next(RayTrace &T, TraceIter &I, int64_t &ix, int64_t &iy,
                                           double &seg_out)
{
    while (!I.done && I.it < T.max_steps) {
        ++I.it;
        int a = 0;
        double tm = T.tmax[0];
        if (T.tmax[1] < tm) { a = 1; tm = T.tmax[1]; }
        if (T.tmax[2] < tm) { a = 2; tm = T.tmax[2]; }
        double tn = tm < T.t1 ? tm : T.t1;
        double seg = (tn - T.t) * T.length;
        const int64_t cx = T.iv[0], cy = T.iv[1];
        if (tm >= T.t1) {
            I.done = true;
        } else {
            T.iv[a] += T.step[a];
            if (T.iv[a] < T.lo[a] || T.iv[a] >= T.hi[a]) {
                I.done = true;
            } else {
                T.tmax[a] += T.tdel[a];
                T.t = tn;
            }
        }
        if (seg > 0.0) {
            ix = cx;
            iy = cy;
            seg_out = seg;
            return true;
        }
    }
    return false;
}

// Writes the sorted row of every hit ray: entries ordered by ix, then iy.
// Along a ray ix and iy are each monotone, so the sorted slot of an entry
// follows from its position in the walk: the walk order itself (ix and iy
// both ascending), its mirror image (both descending), or, when the two run
// in opposite directions, the walk's ix runs (in order or mirrored) with each
// run reversed -- a second walker runs one ix run ahead to give the run's
// length.  No per-column table: any strip width.
__global__ void pb_fill_kernel(int64_t n, int64_t views, int64_t bins, const double *cosv,
                               const double *sinv, int64_t x0, int64_t x1, const int32_t *l2g,
                               const int32_t *indptr, int64_t n_hit, double *data,
                               int32_t *cols)
{
    int64_t lr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (lr >= n_hit) return;
    double src[3], dst[3], dv[3];
    int64_t r = l2g[lr], a = r / bins, k = r % bins;
    pb_endpoints(n, bins, cosv[a], sinv[a], k, src, dst);
    double origin[3] = {-0.5 * (double)n, -0.5 * (double)n, -0.5};
    int64_t lo[3] = {x0, 0, 0}, hi[3] = {x1, n, 1};
    RayTrace T;
    if (!trace_init(src, dst, origin, lo, hi, T, dv)) return;
    const bool xdown = T.step[0] < 0, ydown = T.step[1] < 0;
    const int base = indptr[lr], len = indptr[lr + 1] - base;
    int p = 0;
    if (xdown == ydown) {
        trace_walk(T, [&](int64_t ix, int64_t iy, double seg) {
            const int slot = xdown ? len - 1 - p : p;
            data[base + slot] = seg;
            cols[base + slot] = (int32_t)((ix - x0) * n + iy);
            ++p;
        });
        return;
    }
    RayTrace S = T;   // scout: one ix run ahead
    TraceIter si, wi;
    int64_t six = 0, siy = 0, ix = 0, iy = 0;
    double sseg = 0.0, seg = 0.0;
    bool have = trace_next(S, si, six, siy, sseg);
    while (have) {
        const int64_t gx = six;
        int run_len = 0;
        while (have && six == gx) {
            ++run_len;
            have = trace_next(S, si, six, siy, sseg);
        }
        for (int q = 0; q < run_len; ++q) {
            if (!trace_next(T, wi, ix, iy, seg)) return;
            const int w = p + (run_len - 1 - q);
            const int slot = xdown ? len - 1 - w : w;
            data[base + slot] = seg;
            cols[base + slot] = (int32_t)((ix - x0) * n + iy);
        }
        p += run_len;
    }
}

// ---- general scan geometry (fan / cone beam, geometry.py + projector.py) ----
//
// Measurement g = view * nu*nv + iv*nu + iu; its ray runs from the view's
// source to the pixel centre dc + off_u*det_u + off_v*det_v, offsets
// (i - (n-1)/2) * spacing (geometry.py:144-153, 234-240).  The column block is
// a voxel box [lo, hi); local index ((i0-lo0)*bny + (i1-lo1))*bnz + (i2-lo2)
// (projector.py:164).  Rays are traced in the row-block order of the
// partition (list L: every row block's measurement ids in turn), which is the
// reference's panel row order (projector.py:563-626).

__device__ __forceinline__ void scan_endpoints(const ScanDev &S, int64_t g, double *src,
                                               double *dst)
{
    const int64_t ppv = S.nu * S.nv;
    const int64_t view = g / ppv, pix = g % ppv;
    const int64_t iv = pix / S.nu, iu = pix % S.nu;
    const double ou = ((double)iu - (double)(S.nu - 1) / 2.0) * S.du;
    const double ov = ((double)iv - (double)(S.nv - 1) / 2.0) * S.dv;
    const double *p = S.poses + 12 * view;
    for (int a = 0; a < 3; ++a) {
        src[a] = p[a];
        dst[a] = (p[3 + a] + ou * p[6 + a]) + ov * p[9 + a];
    }
}

template <typename F>
__device__ void trace_walk3(RayTrace &T, F emit)
{
    for (int64_t it = 0; it < T.max_steps; ++it) {
        int a = 0;
        double tm = T.tmax[0];
        if (T.tmax[1] < tm) { a = 1; tm = T.tmax[1]; }
        if (T.tmax[2] < tm) { a = 2; tm = T.tmax[2]; }
        double tn = tm < T.t1 ? tm : T.t1;
        double seg = (tn - T.t) * T.length;
        if (seg > 0.0) emit(T.iv[0], T.iv[1], T.iv[2], seg);
        if (tm >= T.t1) break;
        T.iv[a] += T.step[a];
        if (T.iv[a] < T.lo[a] || T.iv[a] >= T.hi[a]) break;
        T.tmax[a] += T.tdel[a];
        T.t = tn;
    }
}

// counts[q] = entries of ray L[q] in the box; a degenerate ray (source on
// the pixel centre) sets *bad (projector.py:591-592 raises GeometryError).
__global__ void scan_count_kernel(ScanDev S, const int32_t *L, int64_t n, Box B, int32_t *counts,
                                  int32_t *bad)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    double src[3], dst[3], dv[3];
    scan_endpoints(S, L[q], src, dst);
    RayTrace T;
    int cnt = 0;
    if (trace_init_t<false>(src, dst, S.origin, S.vsize, B.lo, B.hi, T, dv))
        trace_walk3(T, [&](int64_t, int64_t, int64_t, double) { ++cnt; });
    else if (T.length == 0.0)
        atomicExch(bad, 1);
    counts[q] = cnt;
}

__device__ __forceinline__ void rev_range(double *d, int32_t *c, int a, int b)
{
    for (--b; a < b; ++a, --b) {
        double td = d[a]; d[a] = d[b]; d[b] = td;
        int32_t tc = c[a]; c[a] = c[b]; c[b] = tc;
    }
}

// Reverses every maximal run of equal key c / div in [a, b).
__device__ void rev_runs(double *d, int32_t *c, int a, int b, int32_t div)
{
    while (a < b) {
        int e = a + 1;
        const int32_t k = c[a] / div;
        while (e < b && c[e] / div == k) ++e;
        rev_range(d, c, a, e);
        a = e;
    }
}

// Writes the row of every hit ray sorted by local index.  The reference
// traverses, then insertion-sorts (projector.py:185-197).  The traversal is
// monotone along every axis, so the sorted order is reached in O(len) by
// reversing the whole row when it runs backwards in i0, then each equal-i0
// run backwards in i1, then each equal-(i0, i1) run backwards in i2 (local
// indices are distinct, so the order is the same).
__global__ void scan_fill_kernel(ScanDev S, const int32_t *l2g, const int32_t *indptr,
                                 int64_t n_hit, Box B, double *data, int32_t *cols)
{
    int64_t lr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (lr >= n_hit) return;
    double src[3], dst[3], dv[3];
    scan_endpoints(S, l2g[lr], src, dst);
    RayTrace T;
    if (!trace_init_t<false>(src, dst, S.origin, S.vsize, B.lo, B.hi, T, dv)) return;
    const int64_t bny = B.hi[1] - B.lo[1], bnz = B.hi[2] - B.lo[2];
    const int base = indptr[lr];
    int k = 0;
    const int64_t s0 = T.step[0], s1 = T.step[1], s2 = T.step[2];
    trace_walk3(T, [&](int64_t i0, int64_t i1, int64_t i2, double seg) {
        data[base + k] = seg;
        cols[base + k] = (int32_t)(((i0 - B.lo[0]) * bny + (i1 - B.lo[1])) * bnz + (i2 - B.lo[2]));
        ++k;
    });
    const int e = base + k;
    int dir = 1;
    if (s0 < 0) { rev_range(data, cols, base, e); dir = -dir; }
    if (s1 * dir < 0) { rev_runs(data, cols, base, e, (int32_t)(bny * bnz)); dir = -dir; }
    if (s2 * dir < 0) rev_runs(data, cols, base, e, (int32_t)bnz);
}

__global__ void gather_i32_kernel(const int32_t *src, const int32_t *idx, int64_t n, int32_t *dst)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < n) dst[q] = src[idx[q]];
}


__global__ void flag_hits_kernel(const int32_t *counts, int64_t n, int32_t *flags)
{
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < n) flags[r] = counts[r] > 0;
}

__global__ void compact_hits_kernel(const int32_t *counts, const int32_t *pos, int64_t n,
                                    int32_t *l2g, int32_t *rowlen)
{
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < n && counts[r] > 0) {
        l2g[pos[r]] = (int32_t)r;
        rowlen[pos[r]] = counts[r];
    }
}

__global__ void rbp_kernel(const int32_t *l2g, int64_t n_hit, const int64_t *edges, int m,
                           int32_t *rbp)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > m) return;
    int64_t key = edges[i];
    int64_t lo = 0, hi = n_hit;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (l2g[mid] < key) lo = mid + 1; else hi = mid;
    }
    rbp[i] = (int32_t)lo;
}

// ---- inverse row map -----------------------------------------------------

__global__ void inv_count_kernel(const int32_t *l2g, int32_t n_rows, int32_t *cnt)
{
    int lr = blockIdx.x * blockDim.x + threadIdx.x;
    if (lr < n_rows) atomicAdd(&cnt[l2g[lr]], 1);
}

__global__ void inv_fill_kernel(const int32_t *l2g, int32_t n_rows, int64_t row_off,
                                const int32_t *inv_ptr, int32_t *fill, int32_t *inv_z)
{
    int lr = blockIdx.x * blockDim.x + threadIdx.x;
    if (lr >= n_rows) return;
    int g = l2g[lr];  // unique within one panel
    inv_z[inv_ptr[g] + fill[g]] = (int32_t)(row_off + lr);
    fill[g] += 1;
}

// ---- bitwise state kernels (reference operation order, no contraction) --

// Interleaved copy of the inverse row map for the epoch tail: groups of 32
// consecutive measurements, slot s of lane l at off[G] + s*32 + l (padding -1
// after a lane's list), so a warp reads its lists with coalesced loads.
__global__ void invt_len_kernel(const int32_t *inv_ptr, int64_t n_meas, int32_t *glen)
{
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int len = g < n_meas ? inv_ptr[g + 1] - inv_ptr[g] : 0;
    int mx = len;
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && g < ((n_meas + 31) & ~31ll)) glen[g >> 5] = mx * 32;
}

__global__ void invt_fill_kernel(const int32_t *inv_ptr, const int32_t *inv_z, int64_t n_meas,
                                 const int32_t *goff, int32_t *invt)
{
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= ((n_meas + 31) & ~31ll)) return;
    const int64_t G = g >> 5;
    const int lane = (int)(g & 31);
    const int nmax = (goff[G + 1] - goff[G]) / 32;
    const int e0 = g < n_meas ? inv_ptr[g] : 0, len = g < n_meas ? inv_ptr[g + 1] - e0 : 0;
    for (int s = 0; s < nmax; ++s) invt[goff[G] + s * 32 + lane] = s < len ? inv_z[e0 + s] : -1;
}

__device__ __forceinline__ int panel_of_off(const PanelDev *panels, int np, int64_t off)
{
    int lo = 0, hi = np - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) / 2;
        if (panels[mid].row_off <= off) lo = mid; else hi = mid - 1;
    }
    return lo;
}

constexpr int MAX_ROW_SEGS = 64;

// Row dot in the reference's order (ascending local column, projector.py:220-244)
// over the row's super-tile segments: merge them by (c / mdiv, tile, c).
template <typename V>
__device__ double row_dot(const PanelDev &P, int64_t lr, const double *xj)
{
    const V *fv = static_cast<const V *>(P.fvals);
    const int q0 = P.rseg_ptr[lr], ns = min(P.rseg_ptr[lr + 1] - q0, MAX_ROW_SEGS);
    int cur[MAX_ROW_SEGS], len[MAX_ROW_SEGS], base[MAX_ROW_SEGS], lane[MAX_ROW_SEGS];
    int64_t sb[MAX_ROW_SEGS];
    for (int k = 0; k < ns; ++k) {
        const int sg = P.rseg[q0 + k];
        cur[k] = 0;
        len[k] = P.seg_len[sg];
        base[k] = P.st_ptr[P.seg_key[sg] / P.n_rows];
        sb[k] = P.slice_start[P.seg_slice[sg]];
        lane[k] = P.seg_lane[sg];
    }
    auto pos = [&](int k) { return sb[k] + ((int64_t)(cur[k] >> 2) * 32 + lane[k]) * 4 + (cur[k] & 3); };
    double acc = 0.0;
    for (;;) {
        int gmin = INT_MAX;
        for (int k = 0; k < ns; ++k)
            if (cur[k] < len[k]) gmin = min(gmin, P.d2c[base[k] + swz_idx(P.fidx[pos(k)], P.swz_shift)] / P.mdiv);
        if (gmin == INT_MAX) break;
        // a segment's run of equal c / mdiv is stored ascending, or descending
        // when the step-coded layout keeps it in walk order (layout.cu fcode_k)
        auto col = [&](int k, int e) {
            const int64_t ps = sb[k] + ((int64_t)(e >> 2) * 32 + lane[k]) * 4 + (e & 3);
            return P.d2c[base[k] + swz_idx(P.fidx[ps], P.swz_shift)];
        };
        for (int k = 0; k < ns; ++k) {
            int e1 = cur[k];
            while (e1 < len[k] && col(k, e1) / P.mdiv == gmin) ++e1;
            const int e0 = cur[k];
            const bool down = e1 - e0 >= 2 && col(k, e0) > col(k, e0 + 1);
            for (int u = 0; u < e1 - e0; ++u) {
                const int e = down ? e1 - 1 - u : e0 + u;
                const int64_t ps = sb[k] + ((int64_t)(e >> 2) * 32 + lane[k]) * 4 + (e & 3);
                acc = __dadd_rn(acc, __dmul_rn((double)fv[ps], xj[base[k] + swz_idx(P.fidx[ps], P.swz_shift)]));
            }
            cur[k] = e1;
        }
    }
    return acc;
}

// z^j = A_:j x_J (projector.py:220-226 via fill_z_from_image)
template <typename V>
__global__ void fill_z_kernel(const PanelDev *panels, int np, int64_t z_len, const double *x,
                              double *z)
{
    int64_t off = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (off >= z_len) return;
    int lp = panel_of_off(panels, np, off);
    const PanelDev &P = panels[lp];
    z[off] = row_dot<V>(P, off - P.row_off, x + P.x_off);
}

// y = A x with per-panel row dots accumulated in ascending j (projector.py:237-244)
template <typename V>
__global__ void forward_kernel(const PanelDev *panels, int np, const int32_t *inv_ptr,
                               const int32_t *inv_z, int64_t n_meas, const double *x, double *out)
{
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= n_meas) return;
    double acc = 0.0;
    for (int e = inv_ptr[g]; e < inv_ptr[g + 1]; ++e) {
        int64_t off = inv_z[e];
        int lp = panel_of_off(panels, np, off);
        const PanelDev &P = panels[lp];
        acc = __dadd_rn(acc, row_dot<V>(P, off - P.row_off, x + P.x_off));
    }
    out[g] = acc;
}

// sum_j z^j per measurement, ascending j (projector.py:767-777)
__global__ void zsum_kernel(const int32_t *inv_ptr, const int32_t *inv_z, int64_t n_meas,
                            const double *z, double *out)
{
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= n_meas) return;
    double acc = 0.0;
    for (int e = inv_ptr[g]; e < inv_ptr[g + 1]; ++e) acc = __dadd_rn(acc, z[inv_z[e]]);
    out[g] = acc;
}

__global__ void sub_kernel(const double *y, const double *s, int64_t n, double *r)
{
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g < n) r[g] = __dsub_rn(y[g], s[g]);
}

// audit: max |r - (y - S)| and max |y| (solvers.py:154-166); results as
// ordered bit patterns of non-negative doubles.
__global__ void audit_kernel(const double *y, const double *r, const double *s, int64_t n,
                             unsigned long long *out2)
{
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double d = 0.0, a = 0.0;
    if (g < n) {
        d = fabs(r[g] - (y[g] - s[g]));
        a = fabs(y[g]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
        a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&out2[0], (unsigned long long)__double_as_longlong(d));
        atomicMax(&out2[1], (unsigned long long)__double_as_longlong(a));
    }
}

// _commit_epoch (solvers.py:180-185) for owned panels.
__global__ void commit_kernel(const PanelDev *panels, int np, int32_t *counts, double *x,
                              double *xhat)
{
    for (int lp = 0; lp < np; ++lp) {
        const PanelDev P = panels[lp];
        int cnt = counts[lp];
        if (cnt <= 0) continue;
        for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < P.n_cols;
             c += (int64_t)gridDim.x * blockDim.x) {
            x[P.x_off + c] = xhat[P.x_off + c] / (double)cnt;
            xhat[P.x_off + c] = 0.0;
        }
    }
}

// Sharded tail: r = y - S for rows of drawn blocks; residual norm partials.
// One launch: r = y - S on the drawn rows (+ r32), |y - S|^2 partials per
// block, and the last block to finish (ticket) writes the epoch's global
// result: |y - S|^2 (block order, like the host sum it replaces), |x|^2 and
// |x_t - x|^2 from the all-reduced exchange tail.
constexpr int FIN_U = 4;
template <int U>
__global__ void __launch_bounds__(256, 4) sharded_finish_kernel(const double *y, const double *S, int64_t n,
                                      const int32_t *rb_of_row, const uint64_t *mask, int m,
                                      double *r, float *r32, double *part, const double *tail,
                                      EpochOut *out, unsigned int *ticket, FinishGuard guard)
{
    if (guard_tripped(guard)) return;   // the epoch was skipped: r and the result stay
    __shared__ double sh[32];
    __shared__ bool is_last;
    __shared__ int s_partial;
    // every row block drawn (full-panel plans): no per-row block lookup
    if (threadIdx.x == 0) s_partial = 0;
    __syncthreads();
    for (int w = threadIdx.x; w < (m + 63) / 64; w += blockDim.x) {
        const int nbits = min(64, m - 64 * w);
        const uint64_t want = nbits == 64 ? ~0ull : ((1ull << nbits) - 1);
        if ((__ldg(mask + w) & want) != want) s_partial = 1;
    }
    __syncthreads();
    const bool partial = s_partial != 0;
    double acc = 0.0;
    // one wave of blocks; each thread takes U pairs of consecutive rows per
    // round (16-byte loads of y and S, all issued before the stores)
    auto row = [&](int64_t g, double d, int rb) {
        if (!partial || (rb >= 0 && ((__ldg(mask + (rb >> 6)) >> (rb & 63)) & 1ull))) {
            r[g] = d;
            if (r32) r32[g] = (float)d;   // FP32 mode's band copy stays in step
        }
        acc = fma(d, d, acc);
    };
    const int64_t npair = n >> 1;
    const int64_t step = (int64_t)gridDim.x * blockDim.x * U;
    for (int64_t q0 = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; q0 < npair; q0 += step) {
        double2 d[U];
        int2 rb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = q0 + (int64_t)u * blockDim.x;
            if (q < npair) {
                const double2 yy = __ldg(reinterpret_cast<const double2 *>(y) + q);
                const double2 ss = __ldcg(reinterpret_cast<const double2 *>(S) + q);
                d[u] = make_double2(yy.x - ss.x, yy.y - ss.y);
                rb[u] = partial ? __ldg(reinterpret_cast<const int2 *>(rb_of_row) + q) : make_int2(0, 0);
            } else {
                d[u] = make_double2(0.0, 0.0);
                rb[u] = make_int2(-1, -1);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = q0 + (int64_t)u * blockDim.x;
            if (q >= npair) continue;
            if (r32 && (!partial || (rb[u].x >= 0 && rb[u].x == rb[u].y &&
                                     ((__ldg(mask + (rb[u].x >> 6)) >> (rb[u].x & 63)) & 1ull)))) {
                // both rows stored: one 16-byte r and one 8-byte r32 store
                reinterpret_cast<double2 *>(r)[q] = d[u];
                reinterpret_cast<float2 *>(r32)[q] = make_float2((float)d[u].x, (float)d[u].y);
                acc = fma(d[u].x, d[u].x, acc);
                acc = fma(d[u].y, d[u].y, acc);
            } else {
                row(2 * q, d[u].x, rb[u].x);
                row(2 * q + 1, d[u].y, rb[u].y);
            }
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0)   // odd last row
        row(n - 1, __ldg(y + n - 1) - __ldcg(S + n - 1), __ldg(rb_of_row + n - 1));
    // fixed-order block sum
    auto block_sum = [&](double v) {
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
        __syncthreads();
        double s = 0.0;
        if (threadIdx.x == 0)
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
        return s;
    };
    acc = block_sum(acc);
    if (threadIdx.x == 0) {
        part[blockIdx.x] = acc;
        __threadfence();
        is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    // the last block: every thread sums blocks t, t + blockDim, ... (L2
    // loads), then the fixed-order block sum
    __threadfence();
    double s = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) s += __ldcg(part + b);
    s = block_sum(s);
    if (threadIdx.x != 0) return;
    out->resid_sq = s;
    out->x_sq = tail[0];
    out->err_sq = tail[1];
    if (guard.host_out) {
        guard.host_out->resid_sq = s;
        guard.host_out->x_sq = tail[0];
        guard.host_out->err_sq = tail[1];
    }
    if (guard.set_ref) *guard.ref = fmax(sqrt(tail[0]), 1e-12);
    *ticket = 0;
}

inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

}  // namespace

// ---------------------------------------------------------------------------
// host-side entry points used by api.cu
// ---------------------------------------------------------------------------
namespace bct {

cudaError_t pb_trace_counts(int64_t n, int64_t views, int64_t bins, const double *d_cos,
                            const double *d_sin, int64_t x0, int64_t x1, int32_t *d_counts,
                            cudaStream_t s)
{
    int64_t nm = views * bins;
    pb_count_kernel<<<nblk(nm, 128), 128, 0, s>>>(n, views, bins, d_cos, d_sin, x0, x1,
                                                  d_counts);
    return cudaGetLastError();
}

// Compacts hit rays; returns n_hit through a host pointer (synchronizes).
cudaError_t pb_compact(const int32_t *d_counts, int64_t nm, int32_t *d_tmp_flags,
                       int32_t *d_tmp_pos, void *d_cub, size_t cub_bytes, int32_t *d_l2g,
                       int32_t *d_rowlen, int64_t *n_hit, cudaStream_t s)
{
    flag_hits_kernel<<<nblk(nm, 256), 256, 0, s>>>(d_counts, nm, d_tmp_flags);
    size_t need = cub_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(d_cub, need, d_tmp_flags, d_tmp_pos, (int)nm, s);
    if (e != cudaSuccess) return e;
    compact_hits_kernel<<<nblk(nm, 256), 256, 0, s>>>(d_counts, d_tmp_pos, nm, d_l2g, d_rowlen);
    int32_t last_pos = 0, last_flag = 0;
    cudaMemcpyAsync(&last_pos, d_tmp_pos + nm - 1, 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&last_flag, d_tmp_flags + nm - 1, 4, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    *n_hit = (int64_t)last_pos + last_flag;
    return e;
}

size_t scan_temp_bytes(int64_t n)
{
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, (int32_t *)nullptr, (int32_t *)nullptr, (int)n);
    return b;
}

size_t sort_temp_bytes(int64_t n)
{
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, (int32_t *)nullptr, (int32_t *)nullptr,
                                    (int32_t *)nullptr, (int32_t *)nullptr, (int)n);
    return b;
}

cudaError_t exclusive_scan_i32(const int32_t *in, int32_t *out, int64_t n, void *d_cub,
                               size_t cub_bytes, cudaStream_t s)
{
    size_t need = cub_bytes;
    return cub::DeviceScan::ExclusiveSum(d_cub, need, in, out, (int)n, s);
}

cudaError_t pb_fill(int64_t n, int64_t views, int64_t bins, const double *d_cos,
                    const double *d_sin, int64_t x0, int64_t x1, const int32_t *d_l2g,
                    const int32_t *d_indptr, int64_t n_hit, double *d_data, int32_t *d_cols,
                    cudaStream_t s)
{
    if (n_hit == 0) return cudaSuccess;
    pb_fill_kernel<<<nblk(n_hit, 64), 64, 0, s>>>(n, views, bins, d_cos, d_sin, x0, x1, d_l2g,
                                                  d_indptr, n_hit, d_data, d_cols);
    return cudaGetLastError();
}

cudaError_t scan_trace_counts(const ScanDev &S, const int32_t *L, int64_t n, const Box &B,
                              int32_t *counts, int32_t *bad, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    scan_count_kernel<<<nblk(n, 128), 128, 0, s>>>(S, L, n, B, counts, bad);
    return cudaGetLastError();
}

cudaError_t scan_fill(const ScanDev &S, const int32_t *l2g, const int32_t *indptr, int64_t n_hit,
                      const Box &B, double *data, int32_t *cols, cudaStream_t s)
{
    if (n_hit == 0) return cudaSuccess;
    scan_fill_kernel<<<nblk(n_hit, 64), 64, 0, s>>>(S, l2g, indptr, n_hit, B, data, cols);
    return cudaGetLastError();
}

cudaError_t gather_i32(const int32_t *src, const int32_t *idx, int64_t n, int32_t *dst,
                       cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    gather_i32_kernel<<<nblk(n, 256), 256, 0, s>>>(src, idx, n, dst);
    return cudaGetLastError();
}


cudaError_t pb_rbp(const int32_t *d_l2g, int64_t n_hit, const int64_t *d_edges, int m,
                   int32_t *d_rbp, cudaStream_t s)
{
    rbp_kernel<<<nblk(m + 1, 128), 128, 0, s>>>(d_l2g, n_hit, d_edges, m, d_rbp);
    return cudaGetLastError();
}

cudaError_t invt_len(const int32_t *inv_ptr, int64_t n_meas, int32_t *glen, cudaStream_t s)
{
    const int64_t n = (n_meas + 31) & ~31ll;
    if (n == 0) return cudaSuccess;
    invt_len_kernel<<<nblk(n, 256), 256, 0, s>>>(inv_ptr, n_meas, glen);
    return cudaGetLastError();
}

cudaError_t invt_fill(const int32_t *inv_ptr, const int32_t *inv_z, int64_t n_meas,
                      const int32_t *goff, int32_t *invt, cudaStream_t s)
{
    const int64_t n = (n_meas + 31) & ~31ll;
    if (n == 0) return cudaSuccess;
    invt_fill_kernel<<<nblk(n, 256), 256, 0, s>>>(inv_ptr, inv_z, n_meas, goff, invt);
    return cudaGetLastError();
}

cudaError_t inv_count(const int32_t *d_l2g, int32_t n_rows, int32_t *d_cnt, cudaStream_t s)
{
    if (n_rows == 0) return cudaSuccess;
    inv_count_kernel<<<nblk(n_rows, 256), 256, 0, s>>>(d_l2g, n_rows, d_cnt);
    return cudaGetLastError();
}

cudaError_t inv_fill(const int32_t *d_l2g, int32_t n_rows, int64_t row_off,
                     const int32_t *d_inv_ptr, int32_t *d_fill, int32_t *d_inv_z, cudaStream_t s)
{
    if (n_rows == 0) return cudaSuccess;
    inv_fill_kernel<<<nblk(n_rows, 256), 256, 0, s>>>(d_l2g, n_rows, row_off, d_inv_ptr, d_fill,
                                                      d_inv_z);
    return cudaGetLastError();
}

cudaError_t fill_z(int dtype, const PanelDev *panels, int np, int64_t z_len, const double *x,
                   double *z, cudaStream_t s)
{
    if (z_len == 0) return cudaSuccess;
    if (dtype == 0)
        fill_z_kernel<double><<<nblk(z_len, 128), 128, 0, s>>>(panels, np, z_len, x, z);
    else
        fill_z_kernel<float><<<nblk(z_len, 128), 128, 0, s>>>(panels, np, z_len, x, z);
    return cudaGetLastError();
}

cudaError_t forward(int dtype, const PanelDev *panels, int np, const int32_t *inv_ptr,
                    const int32_t *inv_z, int64_t n_meas, const double *x, double *out,
                    cudaStream_t s)
{
    if (dtype == 0)
        forward_kernel<double><<<nblk(n_meas, 128), 128, 0, s>>>(panels, np, inv_ptr, inv_z,
                                                                 n_meas, x, out);
    else
        forward_kernel<float><<<nblk(n_meas, 128), 128, 0, s>>>(panels, np, inv_ptr, inv_z,
                                                                n_meas, x, out);
    return cudaGetLastError();
}

cudaError_t zsum(const int32_t *inv_ptr, const int32_t *inv_z, int64_t n_meas, const double *z,
                 double *out, cudaStream_t s)
{
    zsum_kernel<<<nblk(n_meas, 256), 256, 0, s>>>(inv_ptr, inv_z, n_meas, z, out);
    return cudaGetLastError();
}

cudaError_t sub(const double *y, const double *sv, int64_t n, double *r, cudaStream_t s)
{
    sub_kernel<<<nblk(n, 256), 256, 0, s>>>(y, sv, n, r);
    return cudaGetLastError();
}

cudaError_t audit(const double *y, const double *r, const double *sv, int64_t n,
                  unsigned long long *out2, cudaStream_t s)
{
    audit_kernel<<<nblk(n, 256), 256, 0, s>>>(y, r, sv, n, out2);
    return cudaGetLastError();
}

cudaError_t commit(const PanelDev *panels, int np, int32_t *counts, double *x, double *xhat,
                   cudaStream_t s)
{
    commit_kernel<<<148, 256, 0, s>>>(panels, np, counts, x, xhat);
    return cudaGetLastError();
}

cudaError_t sharded_finish(const double *y, const double *S, int64_t n, const int32_t *rb_of_row,
                           const uint64_t *mask, int m, double *r, float *r32, double *part, int nb,
                           const double *tail, EpochOut *out, unsigned int *ticket,
                           const FinishGuard &guard, cudaStream_t s)
{
    // U row pairs per thread and round, one wave of resident blocks, at most
    // nb blocks (the partials array's size)
    static int wave = 0, U = FIN_U;
    if (wave == 0) {
        int dev = 0, sms = 148, per = 4;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sharded_finish_kernel<FIN_U>, 256, 0);
        wave = std::max(1, sms * std::max(per, 1));
        if (const char *e = getenv("BCT_FIN_U")) U = atoi(e) == 1 ? 1 : atoi(e) == 2 ? 2 : 4;
    }
    nb = (int)std::min<int64_t>(std::min(nb, wave),
                                std::max<int64_t>(1, (n / 2 + 256 * U - 1) / (256 * U)));
    if (U == 1)
        sharded_finish_kernel<1><<<nb, 256, 0, s>>>(y, S, n, rb_of_row, mask, m, r, r32, part, tail,
                                                    out, ticket, guard);
    else if (U == 2)
        sharded_finish_kernel<2><<<nb, 256, 0, s>>>(y, S, n, rb_of_row, mask, m, r, r32, part, tail,
                                                    out, ticket, guard);
    else
        sharded_finish_kernel<4><<<nb, 256, 0, s>>>(y, S, n, rb_of_row, mask, m, r, r32, part, tail,
                                                    out, ticket, guard);
    return cudaGetLastError();
}

}  // namespace bct
