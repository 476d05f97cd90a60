// api.cu -- the C ABI of libblockct_cuda.so (include/blockct.h).
//
// Owns the device store (one layout per owned column panel, layout.cu), the
// state vectors and the per-epoch plan staging.  Every entry point validates
// its arguments on the host before touching the device, so an invalid plan
// leaves the state untouched (executor.py:158-169: "a failed batch leaves no
// trace").
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include <functional>
#include <string>
#include <vector>

#include "../../include/blockct.h"
#include "internal.h"

namespace bct {
cudaError_t pb_trace_counts(int64_t, int64_t, int64_t, const double *, const double *, int64_t,
                            int64_t, int32_t *, cudaStream_t);
cudaError_t pb_compact(const int32_t *, int64_t, int32_t *, int32_t *, void *, size_t, int32_t *,
                       int32_t *, int64_t *, cudaStream_t);
size_t scan_temp_bytes(int64_t);
cudaError_t exclusive_scan_i32(const int32_t *, int32_t *, int64_t, void *, size_t, cudaStream_t);
cudaError_t pb_fill(int64_t, int64_t, int64_t, const double *, const double *, int64_t, int64_t,
                    const int32_t *, const int32_t *, int64_t, double *, int32_t *, cudaStream_t);
cudaError_t pb_rbp(const int32_t *, int64_t, const int64_t *, int, int32_t *, cudaStream_t);
cudaError_t inv_count(const int32_t *, int32_t, int32_t *, cudaStream_t);
cudaError_t invt_len(const int32_t *, int64_t, int32_t *, cudaStream_t);
cudaError_t invt_fill(const int32_t *, const int32_t *, int64_t, const int32_t *, int32_t *,
                      cudaStream_t);
cudaError_t inv_fill(const int32_t *, int32_t, int64_t, const int32_t *, int32_t *, int32_t *,
                     cudaStream_t);
cudaError_t fill_z(int, const PanelDev *, int, int64_t, const double *, double *, cudaStream_t);
cudaError_t forward(int, const PanelDev *, int, const int32_t *, const int32_t *, int64_t,
                    const double *, double *, cudaStream_t);
cudaError_t zsum(const int32_t *, const int32_t *, int64_t, const double *, double *,
                 cudaStream_t);
cudaError_t sub(const double *, const double *, int64_t, double *, cudaStream_t);
cudaError_t audit(const double *, const double *, const double *, int64_t, unsigned long long *,
                  cudaStream_t);
cudaError_t commit(const PanelDev *, int, int32_t *, double *, double *, cudaStream_t);
cudaError_t sharded_finish(const double *, const double *, int64_t, const int32_t *,
                           const uint64_t *, int, double *, float *, double *, int, const double *,
                           EpochOut *, unsigned int *, const FinishGuard &, cudaStream_t);
}  // namespace bct

namespace {

constexpr int RING = 4;
// voxels per super tile: its (g, x) pairs are staged in shared memory for
// phase 2 -- 16384 x 8 B (float2, 128 KB) in FP32 mode: fewer (row, super
// tile) segments per row for the batched epochs; 8192 x 16 B (128 KB) in
// FP64 mode
inline int st_voxels(int dtype)
{
    if (getenv("BCT_ST_SMALL")) return 4096;
    if (dtype == 1 && getenv("BCT_F32_ACC64")) return 8192;   // measurement variant (epoch.cu)
    // FP64 configs run per-task (small) epochs: a strip panel of up to 8192
    // voxels is one super tile, so its rows are single segments (epoch.cu
    // phase 2a then finishes rows without a grid barrier)
    return dtype == 0 ? 8192 : 16384;
}
constexpr size_t SMEM_BUDGET = 218 * 1024;  // dynamic shared memory per CTA (one CTA per SM;
                                            // 227 KB less the kernel's static arrays)

struct Slot {
    cudaEvent_t done = nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    char *h_res = nullptr;          // mapped pinned result block [out | mus | statuses],
    char *d_hres = nullptr;         // written by the epoch's last block (device view d_hres)
    int64_t n_tasks = 0, n_visits = 0;
    bool pending = false;
    int32_t *h_plan = nullptr;      // pinned: device-sampled ids of the epoch
    int64_t plan_cap = 0, n_plan = 0;
    int64_t *plan_user = nullptr;   // caller's buffer, filled by bct_wait_epoch
};

}  // namespace

struct bct_ctx {
    std::string err;
    int device = 0, dtype = 0, m = 0, n_panels = 0, pb = 0, pe = 0, np = 0;
    int64_t n_meas = 0, n_vox = 0, nnz = 0, z_len = 0, x_len = 0;
    int64_t max_rows = 0, max_cols = 0, max_seg = 0;
    int32_t *d_gvox = nullptr;     // [x_len] global voxel id of each device position
    double *d_xstage = nullptr;    // [n_vox] global-order staging of image transfers
    char *h_pin[2] = {nullptr, nullptr};   // pinned host chunks for state transfers
    cudaEvent_t pin_ev[2] = {nullptr, nullptr};
    size_t smem = 0;                 // dynamic shared memory of the phase buffers
    size_t smem_total = 0;           // + the per-task record
    int32_t band_cap = 0, band_dbuf = 1;
    cudaStream_t stream = nullptr;
    // host mirrors
    std::vector<PanelDev> h_panels;
    std::vector<std::vector<int32_t>> h_d2c;   // per panel: device position -> local column
    std::vector<std::vector<int32_t>> h_rbp;   // per panel
    std::vector<int64_t> col_ptr, col_vox, rb_ptr, rb_rows;
    std::vector<double> table_values, table_totals;
    // device
    PanelDev *d_panels = nullptr;
    int32_t *inv_ptr = nullptr, *inv_z = nullptr, *d_rb_ptr = nullptr, *d_rb_rows = nullptr;
    int32_t *invt = nullptr, *invt_off = nullptr;   // interleaved inverse map (epoch tail)
    int32_t *rb_of_row = nullptr;
    int32_t *cta_split = nullptr;   // per panel [grid+1]: per-task path phase-2 slice split
    double *y = nullptr, *r = nullptr, *z = nullptr, *x = nullptr, *xhat = nullptr;
    float *r32 = nullptr;   // FP32 mode: band staging copy of r (epoch kernel)
    bool r32_valid = false; // r32 == (float)r (every device writer of r keeps r32 in step;
                            // host writes of r clear it)
    double *x_true = nullptr;
    int32_t *counts = nullptr;
    double *gx = nullptr, *t_ax = nullptr, *seg_part = nullptr, *part = nullptr;
    // epoch-batched parallel path scratch (grow-only)
    double *gx_batch = nullptr, *seg_batch = nullptr, *tax_batch = nullptr, *part_task = nullptr;
    int64_t gx_batch_n = 0, seg_batch_n = 0, tax_batch_n = 0, part_task_n = 0;
    // z in (t, ax) form after fused batched epochs (epoch.cu; EpochParams::zt):
    // per-row pairs (allocated at the first such epoch) and per-panel form;
    // z_lazy: some panel may be in that form (materialize_z before z is used)
    void *zt = nullptr;
    int32_t *zl_on = nullptr, *zl_st = nullptr;
    double *zl_mu = nullptr;
    bool z_lazy = false;
    std::vector<std::vector<int32_t>> h_stbs;  // per panel (n_st*(m+1)) first slice table
    double *mus = nullptr, *exchange = nullptr, *vec = nullptr;
    int32_t *statuses = nullptr;
    EpochOut *out = nullptr;
    double *guard_ref = nullptr;     // divergence guard reference norm (device)
    double guard_factor = 1e6;
    unsigned int *bar = nullptr, *ticket = nullptr;
    // one upload per epoch: [EpochHeader | TaskDev x nt | masks | records]
    // (UpLayout), staged in pinned memory; one download of the result block
    // [EpochOut | mus x nt | statuses x nt]: each small copy costs the
    // stream a few microseconds
    // Double-buffered: epoch e uploads into buffer e & 1 on the copy stream
    // while epoch e-1 still runs; d_up / h_up point at the current buffer.
    char *d_up = nullptr, *h_up = nullptr;
    char *d_upb[2] = {nullptr, nullptr}, *h_upb[2] = {nullptr, nullptr};
    int up_i = 0;
    cudaStream_t cstream = nullptr;          // upload copies
    cudaEvent_t staged_b[2] = {nullptr, nullptr};   // upload of buffer b done (copy stream)
    cudaEvent_t free_b[2] = {nullptr, nullptr};     // main-stream work that read buffer b done
    size_t up_cap = 0;
    char *d_res = nullptr;
    uint64_t *cur_masks = nullptr;   // device masks / tasks of the last submitted epoch
    TaskDev *cur_tasks = nullptr;
    int32_t cur_flags = 0;           // flags of the last submitted epoch
    PrepDims pd{};                   // record dimensions (finalize)
    int32_t prep_off = 0;            // byte offset of the record in dynamic shared memory
    int32_t sc_bound = 1;            // bound on super tiles per panel (record size at layout)
    int mw = 1;                      // 64-bit words per row-block set
    unsigned long long *audit2 = nullptr;

    int64_t task_cap = 0;
    // staging

    Slot slots[RING];
    int head = 0, tail = 0;           // ring: tail = oldest pending
    int grid = 0, block = 0;
    bool has_x_true = false;
    // whole-system baselines (baseline.cu)
    bct::BaselineMat bm;
    bool bm_built = false;
    int32_t bl_kind = -1;
    double *bl_diag = nullptr, *bl_x = nullptr, *bl_r = nullptr, *bl_tmp = nullptr;
    double *bl_part = nullptr, *bl_out = nullptr;
    int32_t *bl_cb_of_vox = nullptr;
    int64_t *bl_col_vox = nullptr;
    // device sampler (bct_sample_epoch)
    double *d_values = nullptr, *d_totals = nullptr, *d_exp = nullptr;
    int64_t d_exp_n = 0;
    bct::SampleVisit *d_visits = nullptr;
    int64_t d_visits_n = 0;
    int32_t *d_plan = nullptr;
    int64_t d_plan_n = 0;
    std::vector<void *> allocs;
    long long *timeline = nullptr;    // BCT_TIMELINE=1: [2][task][8][grid] globaltimer stamps
    int64_t timeline_tasks = 0;
};

static std::string g_create_err;

// Every entry point runs on its context's device and leaves the calling
// thread's current device as it found it (one process may hold contexts on
// several GPUs, and the caller -- e.g. torch -- keeps its own current device).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess)
            prev = cur;
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard &) = delete;
    DeviceGuard &operator=(const DeviceGuard &) = delete;
};
#define DEVICE_GUARD(c) DeviceGuard device_guard_((c)->device)

namespace {

int fail(bct_ctx *c, int code, const char *fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf; else g_create_err = buf;
    return code;
}

#define CK(call)                                                                         \
    do {                                                                                 \
        cudaError_t _e = (call);                                                         \
        if (_e != cudaSuccess)                                                           \
            return fail(c, BCT_ECUDA, "%s failed: %s", #call, cudaGetErrorString(_e)); \
    } while (0)

template <typename T>
int dalloc(bct_ctx *c, T **p, int64_t n)
{
    size_t bytes = (size_t)std::max<int64_t>(n, 1) * sizeof(T);
    cudaError_t e = cudaMalloc((void **)p, bytes);
    if (e != cudaSuccess)
        return fail(c, BCT_ENOMEM, "cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
    c->allocs.push_back(*p);
    return 0;
}

#define DALLOC(p, n)                            \
    do {                                        \
        int _r = dalloc(c, &(p), (int64_t)(n)); \
        if (_r) return _r;                      \
    } while (0)

void free_tmp(bct_ctx *c, void *p)
{
    if (!p) return;
    cudaFree(p);
    c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), p), c->allocs.end());
}

int set_mask(uint64_t *mask, int i) { mask[i >> 6] |= 1ull << (i & 63); return 0; }
bool has_bit(const uint64_t *mask, int i) { return ((mask[i >> 6] >> (i & 63)) & 1ull) != 0; }

// Dynamic shared memory the epoch kernel's phase buffers may use: the SM's
// per-CTA opt-in limit less the kernel's static arrays and the per-task
// record (PrepDims for this context's m and a bound on super tiles), and at
// most SMEM_BUDGET (the shapes were tuned under it).
size_t smem_budget(const bct_ctx *c, int sc)
{
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
    const size_t stat = bct::epoch_static_smem(c->dtype);
    PrepDims d{c->m / 2 + 1, sc, c->m, 0};
    const int64_t room = (int64_t)optin - (int64_t)stat - d.bytes() - 16;
    return (size_t)std::max<int64_t>(0, std::min<int64_t>(room, (int64_t)SMEM_BUDGET));
}

// Voxel placement of a panel: device positions grouped into super tiles of
// <= ST_VOXELS voxels and the phase-1 tile order (16 per tile).  A strip of
// h x w voxels (local column c = ix*w + iy) is cut into iy ranges; inside a
// super tile positions run over (ix, iy).  mdiv = w makes the reference
// order (c ascending) = (ix, tile, iy).  Any other column block keeps its
// order in chunks (mdiv = n_cols).
struct Placement {
    std::vector<int32_t> c2d, d2c, st_ptr, corder;
    int32_t mdiv = 1;
    int32_t swz_shift = 7;   // log2 of the super tiles' row length (swz_idx)
    int32_t st_w = 0;        // strip placement: super tile row length (0: generic)
};

Placement place_voxels(int64_t n_cols, int64_t h, int64_t w, int th, int tw, int dtype)
{
    const int ST_VOXELS = st_voxels(dtype);
    Placement pl;
    pl.c2d.resize(n_cols);
    pl.d2c.resize(n_cols);
    if (h > 0 && w > 0 && h * w == n_cols && h <= ST_VOXELS / 4) {
        int64_t sw = std::max<int64_t>(4, (ST_VOXELS / h) & ~3ll);
        pl.st_w = (int32_t)sw;
        pl.swz_shift = 4;
        while (pl.swz_shift < 15 && (2ll << pl.swz_shift) <= sw) ++pl.swz_shift;
        int32_t d = 0;
        for (int64_t y0 = 0; y0 < w; y0 += sw) {
            pl.st_ptr.push_back(d);
            int64_t y1 = std::min(w, y0 + sw);
            for (int64_t ix = 0; ix < h; ++ix)
                for (int64_t iy = y0; iy < y1; ++iy) {
                    int32_t c = (int32_t)(ix * w + iy);
                    pl.c2d[c] = d;
                    pl.d2c[d] = c;
                    ++d;
                }
        }
        pl.st_ptr.push_back(d);
        // th x tw voxel tiles for phase 1 (consecutive groups of th*tw in corder)
        for (int64_t tx = 0; tx < h; tx += th)
            for (int64_t ty = 0; ty < w; ty += tw)
                for (int64_t a = tx; a < std::min(h, tx + th); ++a)
                    for (int64_t b = ty; b < std::min(w, ty + tw); ++b)
                        pl.corder.push_back(pl.c2d[a * w + b]);
        pl.mdiv = (int32_t)w;
    } else {
        for (int64_t c = 0; c < n_cols; ++c) {
            pl.c2d[c] = pl.d2c[c] = (int32_t)c;
            pl.corder.push_back((int32_t)c);
        }
        for (int64_t d = 0; d < n_cols; d += ST_VOXELS) pl.st_ptr.push_back((int32_t)d);
        pl.st_ptr.push_back((int32_t)n_cols);
        pl.mdiv = (int32_t)std::max<int64_t>(n_cols, 1);
    }
    return pl;
}

// Lays out panel lp from its compact forward CSR on the device
// (vals64/cols/indptr temporaries; l2g persistent), rbp on the host.
int build_panel(bct_ctx *c, int lp, int32_t n_rows, int64_t nnz, const double *vals64,
                const int32_t *cols, const int32_t *indptr, int32_t *l2g,
                const std::vector<int32_t> &rbp, int64_t h, int64_t w)
{
    PanelDev &P = c->h_panels[lp];
    const int j = c->pb + lp;
    const int32_t n_cols = (int32_t)(c->col_ptr[j + 1] - c->col_ptr[j]);
    if (nnz >= (1ll << 31) || n_cols >= (1ll << 30))
        return fail(c, BCT_EINVAL, "panel %d: %lld entries / %d voxels exceed 32-bit panel offsets",
                    j, (long long)nnz, n_cols);
    int32_t *d_rbp = nullptr, *d_d2c = nullptr;
    DALLOC(d_rbp, c->m + 1);
    DALLOC(d_d2c, n_cols);
    CK(cudaMemcpy(d_rbp, rbp.data(), 4 * (c->m + 1), cudaMemcpyHostToDevice));
    // phase-1 tiles, in order of preference: 16x16 voxels with one band
    // buffer (long per-warp streams, a quarter of the band staging per column
    // of 8x8), else 8x8 / 4x8 with double-buffered bands.  BCT_TILE=HxW
    // forces a shape (profiling).
    struct Shape { int th, tw, nbuf; };
    std::vector<Shape> shapes = {{16, 16, 1}, {8, 8, 2}, {4, 8, 2}, {4, 8, 1}};
    // FP32 contexts: the batched path stages FP32 bands, two of which fit in
    // one FP64 band's space, so a shape only has to hold one FP64 band (the
    // per-task path then runs single-buffered).  Config 5 (1440 views) gets
    // 8x8 tiles instead of 4x8: phase A 11.8 -> 8.9 ms per epoch.
    if (c->dtype != 0) shapes = {{16, 16, 1}, {8, 8, 1}, {4, 8, 1}};
    if (const char *e = getenv("BCT_TILE")) {
        int a = 0, b2 = 0;
        if (sscanf(e, "%dx%d", &a, &b2) == 2 && a > 0 && b2 > 0 && (a * b2) % 32 == 0 &&
            a * b2 <= 256)
            shapes = getenv("BCT_TILE_NBUF1") ? std::vector<Shape>{{a, b2, 1}, {4, 8, 1}}
                                              : std::vector<Shape>{{a, b2, 2}, {a, b2, 1}, {4, 8, 1}};
    }
    // record bound: super tiles of any placement hold >= ST_VOXELS/4 voxels
    c->sc_bound = std::max<int32_t>(c->sc_bound, (int32_t)((4ll * n_cols) / st_voxels(c->dtype) + 2));
    const size_t budget = smem_budget(c, c->sc_bound);
    Placement pl;
    for (size_t si = 0; si < shapes.size(); ++si) {
        const int th = shapes[si].th, tw = shapes[si].tw;
        pl = place_voxels(n_cols, h, w, th, tw, c->dtype);
        std::string err;
        std::vector<void *> kept;
        PanelDev Q = P;
        Q.swz_shift = pl.swz_shift;
        // strip panels: no cap on a (row, super tile) run, so no run is cut
        // and every segment step-codes (phase B); generic panels cap at 64
        Q.seg_cap = pl.st_w > 0 ? 1 << 20 : 0;
        Q.st_h = pl.st_w > 0 ? (int32_t)h : 0;   // strip placement: step-coded phase B
        if (bct::layout_panel_v2(c->dtype, c->m, n_rows, n_cols, nnz, vals64, cols, indptr, l2g,
                                 d_rbp, pl.c2d, pl.st_ptr, pl.corder, th * tw, Q, kept, err,
                                 c->stream))
            return fail(c, BCT_ENOMEM, "panel %d layout: %s", j, err.c_str());
        if ((size_t)shapes[si].nbuf * Q.band_max * 8 + bct::PHASE1_RED_BYTES <= budget ||
            si + 1 == shapes.size()) {
            P = Q;
            c->allocs.insert(c->allocs.end(), kept.begin(), kept.end());
            if (getenv("BCT_VERBOSE"))
                fprintf(stderr, "panel %d: tile %dx%d nnz %lld fwd_cap %lld csc_cap %lld band_max %d "
                        "n_seg %d n_slices %d\n", j, th, tw, (long long)nnz,
                        (long long)Q.fwd_cap, (long long)Q.csc_cap, Q.band_max,
                        Q.n_seg, Q.n_slices);
            break;
        }
        for (void *q : kept) cudaFree(q);
    }
    if (P.n_st > c->sc_bound)
        return fail(c, BCT_EINVAL, "panel %d: %d super tiles exceed the record bound %d", j,
                    P.n_st, c->sc_bound);
    CK(cudaMemcpy(d_d2c, pl.d2c.data(), 4 * n_cols, cudaMemcpyHostToDevice));
    P.rbp = d_rbp;
    P.l2g = l2g;
    P.d2c = d_d2c;
    P.n_rows = n_rows;
    P.n_cols = n_cols;
    P.nnz = (int32_t)nnz;
    P.j = j;
    P.mdiv = pl.mdiv;
    c->h_d2c[lp] = pl.d2c;
    c->h_rbp[lp] = rbp;
    c->h_stbs[lp].resize((size_t)P.n_st * (c->m + 1));
    CK(cudaMemcpy(c->h_stbs[lp].data(), P.stbs, 4 * c->h_stbs[lp].size(), cudaMemcpyDeviceToHost));
    c->nnz += nnz;
    c->max_rows = std::max<int64_t>(c->max_rows, n_rows);
    c->max_cols = std::max<int64_t>(c->max_cols, n_cols);
    c->max_seg = std::max<int64_t>(c->max_seg, (int64_t)P.n_slices * 32);   // partial slots
    c->band_cap = std::max(c->band_cap, (P.band_max + 3) & ~3);   // 16-byte aligned FP32 buffers
    // staged super tile: (g, x) as float2 in FP32 mode, double2 in FP64 mode (swizzled)
    c->smem = std::max<size_t>(c->smem, (size_t)((P.st_max + 15) & ~15) *
                                            (c->dtype == 0 || getenv("BCT_F32_ACC64") ? 16 : 8));
    return 0;
}

int ensure_task_cap(bct_ctx *c, int64_t n);

// Common tail of context creation: offsets, row-block tables, inverse map, state.
int finalize(bct_ctx *c)
{
    int64_t ro = 0, xo = 0;
    for (int lp = 0; lp < c->np; ++lp) {
        c->h_panels[lp].row_off = ro;
        c->h_panels[lp].x_off = xo;
        ro += c->h_panels[lp].n_rows;
        xo += c->h_panels[lp].n_cols;
    }
    if (ro >= (1ll << 31)) return fail(c, BCT_EINVAL, "z store exceeds 2^31 rows");
    c->z_len = ro;
    c->x_len = xo;
    {   // device position -> global voxel id (state transfers permute on the device)
        std::vector<int32_t> gv(std::max<int64_t>(xo, 1));
        for (int lp = 0; lp < c->np; ++lp) {
            const PanelDev &P = c->h_panels[lp];
            const int64_t cb = c->col_ptr[c->pb + lp];
            for (int64_t d = 0; d < P.n_cols; ++d)
                gv[P.x_off + d] = (int32_t)c->col_vox[cb + c->h_d2c[lp][d]];
        }
        DALLOC(c->d_gvox, std::max<int64_t>(xo, 1));
        DALLOC(c->d_xstage, std::max<int64_t>(c->n_vox, 1));
        CK(cudaMemcpy(c->d_gvox, gv.data(), 4 * std::max<int64_t>(xo, 1), cudaMemcpyHostToDevice));
    }
    // row blocks
    std::vector<int32_t> rbp32(c->rb_ptr.begin(), c->rb_ptr.end());
    std::vector<int32_t> rows32(c->rb_rows.begin(), c->rb_rows.end());
    std::vector<int32_t> of_row(c->n_meas, -1);
    for (int i = 0; i < c->m; ++i)
        for (int64_t q = c->rb_ptr[i]; q < c->rb_ptr[i + 1]; ++q) of_row[c->rb_rows[q]] = i;
    DALLOC(c->d_rb_ptr, c->m + 1);
    DALLOC(c->d_rb_rows, rows32.size());
    DALLOC(c->rb_of_row, c->n_meas);
    CK(cudaMemcpy(c->d_rb_ptr, rbp32.data(), 4 * rbp32.size(), cudaMemcpyHostToDevice));
    if (!rows32.empty())
        CK(cudaMemcpy(c->d_rb_rows, rows32.data(), 4 * rows32.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->rb_of_row, of_row.data(), 4 * of_row.size(), cudaMemcpyHostToDevice));
    DALLOC(c->d_panels, c->np);
    CK(cudaMemcpy(c->d_panels, c->h_panels.data(), sizeof(PanelDev) * c->np,
                  cudaMemcpyHostToDevice));

    // inverse row map over owned panels, panel-ascending
    DALLOC(c->inv_ptr, c->n_meas + 1);
    DALLOC(c->inv_z, c->z_len);
    int32_t *cnt = nullptr, *fill = nullptr;
    DALLOC(cnt, c->n_meas + 1);
    DALLOC(fill, c->n_meas);
    CK(cudaMemsetAsync(cnt, 0, 4 * (c->n_meas + 1), c->stream));
    CK(cudaMemsetAsync(fill, 0, 4 * c->n_meas, c->stream));
    for (int lp = 0; lp < c->np; ++lp)
        CK(bct::inv_count(c->h_panels[lp].l2g, c->h_panels[lp].n_rows, cnt, c->stream));
    size_t sb = bct::scan_temp_bytes(c->n_meas + 1);
    char *cub = nullptr;
    DALLOC(cub, (int64_t)sb);
    CK(bct::exclusive_scan_i32(cnt, c->inv_ptr, c->n_meas + 1, cub, sb, c->stream));
    for (int lp = 0; lp < c->np; ++lp) {
        const PanelDev &P = c->h_panels[lp];
        CK(bct::inv_fill(P.l2g, P.n_rows, P.row_off, c->inv_ptr, fill, c->inv_z, c->stream));
    }
    {
        // interleaved copy for the epoch tail (groups of 32 measurements)
        const int64_t ng = (c->n_meas + 31) / 32;
        size_t sb2 = bct::scan_temp_bytes(ng + 1);
        char *cub2 = nullptr;
        DALLOC(cub2, (int64_t)sb2);
        int32_t *glen = nullptr;
        DALLOC(glen, ng + 1);
        DALLOC(c->invt_off, ng + 1);
        CK(cudaMemsetAsync(glen, 0, 4 * (ng + 1), c->stream));
        CK(bct::invt_len(c->inv_ptr, c->n_meas, glen, c->stream));
        CK(bct::exclusive_scan_i32(glen, c->invt_off, ng + 1, cub2, sb2, c->stream));
        int32_t tot = 0;
        CK(cudaMemcpyAsync(&tot, c->invt_off + ng, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        DALLOC(c->invt, std::max<int32_t>(tot, 1));
        CK(bct::invt_fill(c->inv_ptr, c->inv_z, c->n_meas, c->invt_off, c->invt, c->stream));
        free_tmp(c, glen);
        free_tmp(c, cub2);
    }
    CK(cudaStreamSynchronize(c->stream));
    free_tmp(c, cnt);
    free_tmp(c, fill);
    free_tmp(c, cub);

    // state and scratch
    DALLOC(c->y, c->n_meas);
    DALLOC(c->r, c->n_meas + 2);   // + 16-byte bulk-copy overhang (epoch.cu band staging)
    if (c->dtype == BCT_F32) {
        DALLOC(c->r32, c->n_meas + 4);
        CK(cudaMemsetAsync(c->r32, 0, 4 * (c->n_meas + 4), c->stream));
    }
    DALLOC(c->vec, c->n_meas + 2);
    DALLOC(c->exchange, c->n_meas + 2);
    DALLOC(c->z, c->z_len);
    DALLOC(c->zl_on, std::max(c->np, 1));
    DALLOC(c->zl_st, std::max(c->np, 1));
    DALLOC(c->zl_mu, std::max(c->np, 1));
    CK(cudaMemsetAsync(c->zl_on, 0, 4 * std::max(c->np, 1), c->stream));
    DALLOC(c->x, c->x_len);
    DALLOC(c->xhat, c->x_len);
    DALLOC(c->x_true, c->x_len);
    DALLOC(c->counts, c->np);
    DALLOC(c->gx, 4 * c->max_cols);
    DALLOC(c->t_ax, 2 * c->max_rows);
    DALLOC(c->seg_part, 2 * bct::TASK_PARTS_MAX * c->max_seg + 2);   // partials per lane (epoch.cu)
    // two band buffers when they fit, else one (staging then serializes)
    // phase-1 bands (double-buffered when they fit) + the tile reduction area
    // per-task records: runs of a mask, super tiles, the visit's row blocks
    int sc = 1;
    for (int lp = 0; lp < c->np; ++lp) sc = std::max(sc, c->h_panels[lp].n_st);
    c->pd = PrepDims{c->m / 2 + 1, sc, c->m, 0};
    c->mw = mask_words(c->m);
    const size_t budget = smem_budget(c, sc);
    c->band_dbuf = (2 * (size_t)c->band_cap * 8 + bct::PHASE1_RED_BYTES <= budget &&
                    !getenv("BCT_TILE_NBUF1")) ? 1 : 0;
    c->smem = std::max<size_t>(c->smem, (size_t)c->band_cap * 8 * (c->band_dbuf ? 2 : 1) +
                                            bct::PHASE1_RED_BYTES);
    c->smem = std::max<size_t>(c->smem, 1024 * 12 + 64);
    c->prep_off = (int32_t)((c->smem + 15) & ~(size_t)15);
    c->smem_total = (size_t)c->prep_off + (size_t)c->pd.bytes();
    {
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
        if (c->smem_total + bct::epoch_static_smem(c->dtype) > (size_t)optin)
            return fail(c, BCT_EINVAL, "shared-memory need %zu B exceeds the SM (band %d slots, "
                        "m %d)", c->smem_total, c->band_cap, c->m);
    }
    c->grid = bct::epoch_grid_size(c->dtype, c->device, c->smem_total, &c->block);
    DALLOC(c->part, 8 * (int64_t)c->grid + 8);
    {
        // per-task path, full-panel tasks: CTA b streams the slices whose first
        // entry lies in [F*b/G, F*(b+1)/G) of the panel's F stored entries (a
        // static split, tabled here instead of searched per task)
        const int G = c->grid;
        // (config 2: 256 entries per slice 0.265 -> 0.2625 ms per epoch kernel; 128 and 384
        // no better than 0 -- the gain is partly where the cuts fall)
        const int64_t SC = getenv("BCT_TASK_SLICE_COST") ? atoll(getenv("BCT_TASK_SLICE_COST")) : 256;
        std::vector<int32_t> split((size_t)std::max(c->np, 1) * (G + 1), 0);
        std::vector<int32_t> ss;
        for (int lp = 0; lp < c->np; ++lp) {
            const PanelDev &P = c->h_panels[lp];
            ss.resize((size_t)P.n_slices + 1);
            CK(cudaMemcpy(ss.data(), P.slice_start, 4 * ss.size(), cudaMemcpyDeviceToHost));
            // cost of a slice prefix: its stored entries + SC per slice (a
            // slice's fixed latency: metadata, its first load round trip)
            std::vector<int64_t> cost(ss.size());
            for (size_t q = 0; q < ss.size(); ++q) cost[q] = (int64_t)ss[q] + SC * (int64_t)q;
            const int64_t F = cost[P.n_slices];
            for (int b = 0; b <= G; ++b) {
                const int64_t key = F * b / G;
                split[(size_t)lp * (G + 1) + b] =
                    b == G ? P.n_slices
                           : (int32_t)(std::lower_bound(cost.begin(), cost.begin() + P.n_slices, key) -
                                       cost.begin());
            }
        }
        DALLOC(c->cta_split, split.size());
        CK(cudaMemcpy(c->cta_split, split.data(), 4 * split.size(), cudaMemcpyHostToDevice));
    }
    DALLOC(c->guard_ref, 1);
    DALLOC(c->bar, 1);
    DALLOC(c->ticket, 1);
    DALLOC(c->audit2, 2);
    CK(cudaMemsetAsync(c->y, 0, 8 * c->n_meas, c->stream));
    CK(cudaMemsetAsync(c->r, 0, 8 * (c->n_meas + 2), c->stream));
    CK(cudaMemsetAsync(c->z, 0, 8 * std::max<int64_t>(c->z_len, 1), c->stream));
    CK(cudaMemsetAsync(c->x, 0, 8 * std::max<int64_t>(c->x_len, 1), c->stream));
    CK(cudaMemsetAsync(c->xhat, 0, 8 * std::max<int64_t>(c->x_len, 1), c->stream));
    CK(cudaMemsetAsync(c->counts, 0, 4 * std::max(c->np, 1), c->stream));
    CK(cudaMemsetAsync(c->bar, 0, 4, c->stream));
    CK(cudaMemsetAsync(c->ticket, 0, 4, c->stream));
    for (int s = 0; s < RING; ++s) {
        CK(cudaEventCreateWithFlags(&c->slots[s].done, cudaEventDisableTiming));
        CK(cudaEventCreate(&c->slots[s].t0));
        CK(cudaEventCreate(&c->slots[s].t1));
    }
    CK(cudaStreamSynchronize(c->stream));
    return ensure_task_cap(c, 1);
}

// Byte layout of an epoch's upload block for nt tasks (16-byte aligned parts).
struct UpLayout {
    size_t tasks, masks, prep, total;
};
static size_t a16(size_t v) { return (v + 15) & ~(size_t)15; }
static UpLayout up_layout(const bct_ctx *c, int64_t nt, bool with_prep)
{
    UpLayout L;
    L.tasks = a16(sizeof(EpochHeader));
    L.masks = a16(L.tasks + sizeof(TaskDev) * (size_t)nt);
    L.prep = a16(L.masks + 8 * (size_t)c->mw * (1 + 2 * (size_t)nt));
    L.total = L.prep + (with_prep ? (size_t)c->pd.bytes() * (size_t)nt : 0);
    return L;
}
constexpr size_t RES_HEAD = bct::RES_HEAD_BYTES;   // EpochOut at the start of the result block
static_assert(sizeof(EpochOut) <= RES_HEAD, "result block head");

int ensure_task_cap(bct_ctx *c, int64_t n)
{
    if (n <= c->task_cap) return 0;
    int64_t cap = std::max<int64_t>(n, 2 * c->task_cap);
    // drain pending epochs before reallocating buffers they use
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaStreamSynchronize(c->cstream));
    const size_t up = up_layout(c, cap, true).total;
    for (int b = 0; b < 2; ++b) {
        if (c->d_upb[b]) cudaFree(c->d_upb[b]);
        if (c->h_upb[b]) cudaFreeHost(c->h_upb[b]);
        CK(cudaMalloc((void **)&c->d_upb[b], up));
        CK(cudaHostAlloc((void **)&c->h_upb[b], up, cudaHostAllocDefault));
    }
    c->d_up = c->d_upb[c->up_i];
    c->h_up = c->h_upb[c->up_i];
    c->up_cap = up;
    // the result block; the last epoch's EpochOut carries over (the
    // divergence guard of the next epoch reads it)
    char *res = nullptr;
    const size_t rb = RES_HEAD + 12 * (size_t)cap;
    CK(cudaMalloc((void **)&res, rb));
    CK(cudaMemset(res, 0, rb));
    if (c->d_res) {
        CK(cudaMemcpy(res, c->d_res, sizeof(EpochOut), cudaMemcpyDeviceToDevice));
        cudaFree(c->d_res);
    }
    c->d_res = res;
    c->out = reinterpret_cast<EpochOut *>(res);
    for (int s = 0; s < RING; ++s) {
        if (c->slots[s].h_res) cudaFreeHost(c->slots[s].h_res);
        CK(cudaHostAlloc((void **)&c->slots[s].h_res, rb, cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer((void **)&c->slots[s].d_hres, c->slots[s].h_res, 0));
    }
    c->task_cap = cap;
    return 0;
}

int check_common_desc(bct_ctx *c, int m, int n_panels, int pb, int pe, int dtype)
{
    if (m < 1 || m > BCT_MAX_M) return fail(c, BCT_EINVAL, "m=%d outside [1, %d]", m, BCT_MAX_M);
    if (n_panels < 1) return fail(c, BCT_EINVAL, "n_panels must be >= 1");
    if (pb < 0 || pe > n_panels || pb >= pe)
        return fail(c, BCT_EINVAL, "owned panel range [%d, %d) invalid", pb, pe);
    if (dtype != BCT_F64 && dtype != BCT_F32) return fail(c, BCT_EINVAL, "dtype %d", dtype);
    return 0;
}

void destroy(bct_ctx *c)
{
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    bct::baseline_free(c->bm);
    for (void *p : c->allocs) cudaFree(p);
    for (int i = 0; i < 2; ++i) {
        if (c->h_pin[i]) cudaFreeHost(c->h_pin[i]);
        if (c->pin_ev[i]) cudaEventDestroy(c->pin_ev[i]);
    }
    if (c->d_res) cudaFree(c->d_res);
    if (c->timeline) cudaFree(c->timeline);
    for (double *q : {c->gx_batch, c->seg_batch, c->tax_batch, c->part_task})
        if (q) cudaFree(q);
    if (c->zt) cudaFree(c->zt);
    if (c->cstream) cudaStreamSynchronize(c->cstream);
    for (int b = 0; b < 2; ++b) {
        if (c->d_upb[b]) cudaFree(c->d_upb[b]);
        if (c->h_upb[b]) cudaFreeHost(c->h_upb[b]);
        if (c->staged_b[b]) cudaEventDestroy(c->staged_b[b]);
        if (c->free_b[b]) cudaEventDestroy(c->free_b[b]);
    }
    for (int s = 0; s < RING; ++s) {
        Slot &S = c->slots[s];
        if (S.done) cudaEventDestroy(S.done);
        if (S.t0) cudaEventDestroy(S.t0);
        if (S.t1) cudaEventDestroy(S.t1);
        if (S.h_res) cudaFreeHost(S.h_res);
    }
    if (c->cstream) cudaStreamDestroy(c->cstream);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

int init_ctx(bct_ctx *c, int device, int np)
{
    c->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
        CK(cudaEventCreateWithFlags(&c->staged_b[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->free_b[b], cudaEventDisableTiming));
    }
    int coop = 0;
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
    if (!coop) return fail(c, BCT_ECUDA, "device %d lacks cooperative launch", device);
    c->h_panels.assign(np, PanelDev{});
    c->h_d2c.resize(np);
    c->h_rbp.resize(np);
    c->h_stbs.resize(np);
    return 0;
}

}  // namespace

extern "C" {

const char *bct_last_error(const bct_ctx *ctx)
{
    return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

int bct_version(void) { return 2; }

int bct_create(const bct_system_desc *d, const bct_panel *panels, bct_ctx **out)
{
    if (!d || !panels || !out) return fail(nullptr, BCT_EINVAL, "null argument");
    DeviceGuard device_guard_(d->device);
    *out = nullptr;
    int r = check_common_desc(nullptr, d->m, d->n_panels, d->panel_begin, d->panel_end, d->dtype);
    if (r) return r;
    bct_ctx *c = new bct_ctx();
    auto bail = [&](int code) {
        g_create_err = c->err;
        destroy(c);
        return code;
    };
    if ((r = init_ctx(c, d->device, d->panel_end - d->panel_begin))) return bail(r);
    c->dtype = d->dtype;
    c->m = d->m;
    c->n_panels = d->n_panels;
    c->pb = d->panel_begin;
    c->pe = d->panel_end;
    c->np = c->pe - c->pb;
    c->n_meas = d->n_meas;
    c->n_vox = d->n_vox;
    if (c->n_meas >= (1ll << 31) || c->n_meas < 1 || c->n_vox < 1)
        return bail(fail(c, BCT_EINVAL, "bad sizes n_meas=%lld n_vox=%lld",
                         (long long)c->n_meas, (long long)c->n_vox));
    c->rb_ptr.assign(d->row_block_ptr, d->row_block_ptr + c->m + 1);
    c->rb_rows.assign(d->row_block_rows, d->row_block_rows + c->rb_ptr[c->m]);
    c->col_ptr.assign(d->col_block_ptr, d->col_block_ptr + c->n_panels + 1);
    c->col_vox.assign(d->col_block_vox, d->col_block_vox + c->col_ptr[c->n_panels]);
    c->table_values.assign(d->table_values, d->table_values + (int64_t)c->m * c->n_panels);
    c->table_totals.assign(d->table_totals, d->table_totals + c->n_panels);
    for (int64_t g : c->rb_rows)
        if (g < 0 || g >= c->n_meas) return bail(fail(c, BCT_EINVAL, "row block id out of range"));
    for (int64_t v : c->col_vox)
        if (v < 0 || v >= c->n_vox) return bail(fail(c, BCT_EINVAL, "voxel id out of range"));
    int64_t max_nnz = 1, max_rows = 1;
    for (int lp = 0; lp < c->np; ++lp) {
        const bct_panel &p = panels[lp];
        int j = c->pb + lp;
        int64_t ncols = c->col_ptr[j + 1] - c->col_ptr[j];
        if (p.n_rows < 0 || p.nnz < 0 || p.indptr[p.n_rows] != p.nnz || p.rbp[c->m] != p.n_rows ||
            p.rbp[0] != 0)
            return bail(fail(c, BCT_EINVAL, "panel %d: inconsistent indptr/rbp", j));
        if (p.nnz >= (1ll << 30) || ncols >= (1ll << 24))
            return bail(fail(c, BCT_EINVAL, "panel %d too large", j));
        for (int64_t q = 0; q < p.nnz; ++q)
            if (p.cols[q] < 0 || p.cols[q] >= ncols)
                return bail(fail(c, BCT_EINVAL, "panel %d: column id out of range", j));
        for (int64_t q = 0; q < p.n_rows; ++q)
            if (p.l2g[q] < 0 || p.l2g[q] >= c->n_meas)
                return bail(fail(c, BCT_EINVAL, "panel %d: l2g out of range", j));
        max_nnz = std::max(max_nnz, p.nnz);
        max_rows = std::max(max_rows, p.n_rows);
    }
    double *vals64 = nullptr;
    int32_t *cols = nullptr, *indptr = nullptr;
    {
        bct_ctx *cc = c;
        if (dalloc(cc, &vals64, max_nnz) || dalloc(cc, &cols, max_nnz) ||
            dalloc(cc, &indptr, max_rows + 1))
            return bail(BCT_ENOMEM);
    }
    for (int lp = 0; lp < c->np; ++lp) {
        const bct_panel &p = panels[lp];
        std::vector<int32_t> ip(p.indptr, p.indptr + p.n_rows + 1);
        std::vector<int32_t> rb(p.rbp, p.rbp + c->m + 1);
        std::vector<int32_t> lg(p.l2g, p.l2g + p.n_rows);
        int32_t *l2g = nullptr;
        if (dalloc(c, &l2g, p.n_rows)) return bail(BCT_ENOMEM);
        if (cudaMemcpy(vals64, p.data, 8 * p.nnz, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(cols, p.cols, 4 * p.nnz, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(indptr, ip.data(), 4 * ip.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
            (p.n_rows > 0 &&
             cudaMemcpy(l2g, lg.data(), 4 * lg.size(), cudaMemcpyHostToDevice) != cudaSuccess))
            return bail(fail(c, BCT_ECUDA, "panel upload failed"));
        if ((r = build_panel(c, lp, (int32_t)p.n_rows, p.nnz, vals64, cols, indptr, l2g, rb, 0, 0)))
            return bail(r);
    }
    free_tmp(c, vals64);
    free_tmp(c, cols);
    free_tmp(c, indptr);
    if ((r = finalize(c))) return bail(r);
    *out = c;
    return 0;
}

int bct_create_parallel_beam(const bct_pb_desc *d, bct_ctx **out)
{
    if (!d || !out || !d->cos_views || !d->sin_views)
        return fail(nullptr, BCT_EINVAL, "null argument");
    DeviceGuard device_guard_(d->device);
    *out = nullptr;
    int r = check_common_desc(nullptr, d->m, d->nc, d->panel_begin, d->panel_end, d->dtype);
    if (r) return r;
    if (d->n < 1 || d->views < d->m || d->bins < 1 || d->nc > d->n)
        return fail(nullptr, BCT_EINVAL, "bad parallel-beam sizes");
    bct_ctx *c = new bct_ctx();
    auto bail = [&](int code) {
        g_create_err = c->err;
        destroy(c);
        return code;
    };
    if ((r = init_ctx(c, d->device, d->panel_end - d->panel_begin))) return bail(r);
    const int64_t n = d->n, views = d->views, bins = d->bins;
    c->dtype = d->dtype;
    c->m = d->m;
    c->n_panels = d->nc;
    c->pb = d->panel_begin;
    c->pe = d->panel_end;
    c->np = c->pe - c->pb;
    c->n_meas = views * bins;
    c->n_vox = n * n;
    if (c->n_meas >= (1ll << 31)) return bail(fail(c, BCT_EINVAL, "too many measurements"));
    // partition: numpy round(linspace(0, views, m+1)), half-even
    std::vector<int64_t> aedge(c->m + 1), xedge(c->n_panels + 1);
    {
        double step = (double)views / c->m;
        for (int i = 0; i <= c->m; ++i) {
            double v = (i == c->m) ? (double)views : i * step;
            aedge[i] = (int64_t)std::nearbyint(v);
        }
    }
    int64_t base = (n + c->n_panels - 1) / c->n_panels;
    for (int j = 0; j < c->n_panels; ++j) xedge[j] = std::min<int64_t>(j * base, n);
    xedge[c->n_panels] = n;
    for (int j = 0; j < c->n_panels; ++j)
        if (xedge[j] >= xedge[j + 1]) return bail(fail(c, BCT_EINVAL, "empty strip %d", j));
    c->rb_ptr.resize(c->m + 1);
    for (int i = 0; i <= c->m; ++i) c->rb_ptr[i] = aedge[i] * bins;
    c->rb_rows.resize(c->n_meas);
    for (int64_t g = 0; g < c->n_meas; ++g) c->rb_rows[g] = g;
    c->col_ptr.resize(c->n_panels + 1);
    for (int j = 0; j <= c->n_panels; ++j) c->col_ptr[j] = xedge[j] * n;
    c->col_vox.resize(c->n_vox);
    for (int64_t v = 0; v < c->n_vox; ++v) c->col_vox[v] = v;

    double *d_cos = nullptr, *d_sin = nullptr;
    int64_t *d_edges = nullptr;
    int32_t *d_counts = nullptr, *d_flags = nullptr, *d_pos = nullptr;
    DALLOC(d_cos, views);
    DALLOC(d_sin, views);
    DALLOC(d_edges, c->m + 1);
    DALLOC(d_counts, c->n_meas);
    DALLOC(d_flags, c->n_meas);
    DALLOC(d_pos, c->n_meas + 1);
    CK(cudaMemcpy(d_cos, d->cos_views, 8 * views, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_sin, d->sin_views, 8 * views, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_edges, c->rb_ptr.data(), 8 * (c->m + 1), cudaMemcpyHostToDevice));
    size_t sb = bct::scan_temp_bytes(c->n_meas + 1);
    char *cub = nullptr;
    DALLOC(cub, (int64_t)sb);

    // pass 1: every panel (the density table needs all of them), per-ray counts
    std::vector<int32_t> h_counts(c->n_meas);
    c->table_values.assign((int64_t)c->m * c->n_panels, 0.0);
    std::vector<int64_t> rows(c->np), nnzs(c->np);
    std::vector<int32_t *> p_l2g(c->np, nullptr), p_ip(c->np, nullptr);
    int64_t max_nnz = 1;
    for (int j = 0; j < c->n_panels; ++j) {
        CK(bct::pb_trace_counts(n, views, bins, d_cos, d_sin, xedge[j], xedge[j + 1], d_counts,
                                c->stream));
        CK(cudaMemcpyAsync(h_counts.data(), d_counts, 4 * c->n_meas, cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaStreamSynchronize(c->stream));
        int64_t vox_j = (xedge[j + 1] - xedge[j]) * n;
        int64_t tot = 0;
        for (int i = 0; i < c->m; ++i) {
            int64_t s = 0;
            for (int64_t g = c->rb_ptr[i]; g < c->rb_ptr[i + 1]; ++g) s += h_counts[g];
            tot += s;
            c->table_values[(int64_t)i * c->n_panels + j] =
                (double)s / ((double)(c->rb_ptr[i + 1] - c->rb_ptr[i]) * (double)vox_j);
        }
        if (j < c->pb || j >= c->pe) continue;
        int lp = j - c->pb;
        int64_t n_hit = 0;
        int32_t *rowlen = nullptr;
        DALLOC(p_l2g[lp], c->n_meas);
        DALLOC(rowlen, c->n_meas + 1);
        CK(bct::pb_compact(d_counts, c->n_meas, d_flags, d_pos, cub, sb, p_l2g[lp], rowlen, &n_hit,
                           c->stream));
        DALLOC(p_ip[lp], n_hit + 1);
        CK(cudaMemsetAsync(rowlen + n_hit, 0, 4, c->stream));
        CK(bct::exclusive_scan_i32(rowlen, p_ip[lp], n_hit + 1, cub, sb, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        free_tmp(c, rowlen);
        rows[lp] = n_hit;
        nnzs[lp] = tot;
        max_nnz = std::max(max_nnz, tot);
        if (tot >= (1ll << 30)) return bail(fail(c, BCT_EINVAL, "panel %d too large", j));
    }
    c->table_totals.assign(c->n_panels, 0.0);
    // totals = values.sum(axis=0): numpy reduces axis 0 row by row
    for (int i = 0; i < c->m; ++i)
        for (int j = 0; j < c->n_panels; ++j)
            c->table_totals[j] += c->table_values[(int64_t)i * c->n_panels + j];
    free_tmp(c, d_counts);
    free_tmp(c, d_flags);
    free_tmp(c, d_pos);
    double *vals64 = nullptr;
    int32_t *cols = nullptr, *rbp_tmp = nullptr;
    DALLOC(vals64, max_nnz);
    DALLOC(cols, max_nnz);
    DALLOC(rbp_tmp, c->m + 1);
    for (int lp = 0; lp < c->np; ++lp) {
        int j = c->pb + lp;
        CK(bct::pb_fill(n, views, bins, d_cos, d_sin, xedge[j], xedge[j + 1], p_l2g[lp], p_ip[lp],
                        rows[lp], vals64, cols, c->stream));
        CK(bct::pb_rbp(p_l2g[lp], rows[lp], d_edges, c->m, rbp_tmp, c->stream));
        std::vector<int32_t> rb(c->m + 1);
        CK(cudaMemcpyAsync(rb.data(), rbp_tmp, 4 * (c->m + 1), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if ((r = build_panel(c, lp, (int32_t)rows[lp], nnzs[lp], vals64, cols, p_ip[lp], p_l2g[lp],
                             rb, xedge[j + 1] - xedge[j], n)))
            return bail(r);
        free_tmp(c, p_ip[lp]);
    }
    free_tmp(c, vals64);
    free_tmp(c, cols);
    free_tmp(c, rbp_tmp);
    free_tmp(c, cub);
    if ((r = finalize(c))) return bail(r);
    *out = c;
    return 0;
}

int bct_create_scan(const bct_scan_desc *d, bct_ctx **out)
{
    if (!d || !out || !d->poses || !d->row_block_ptr || !d->row_block_rows || !d->box_lo ||
        !d->box_hi || !d->table_values || !d->table_totals)
        return fail(nullptr, BCT_EINVAL, "null argument");
    DeviceGuard device_guard_(d->device);
    *out = nullptr;
    int r = check_common_desc(nullptr, d->m, d->n_panels, d->panel_begin, d->panel_end, d->dtype);
    if (r) return r;
    for (int a = 0; a < 3; ++a)
        if (d->dims[a] < 1 || !(d->voxel_size[a] > 0.0) || !std::isfinite(d->origin[a]))
            return fail(nullptr, BCT_EINVAL, "bad voxel grid");
    if (d->det_nu < 1 || d->det_nv < 1 || d->n_views < 1 || !(d->det_du > 0.0) ||
        !(d->det_dv > 0.0))
        return fail(nullptr, BCT_EINVAL, "bad detector");
    bct_ctx *c = new bct_ctx();
    auto bail = [&](int code) {
        g_create_err = c->err;
        destroy(c);
        return code;
    };
    if ((r = init_ctx(c, d->device, d->panel_end - d->panel_begin))) return bail(r);
    c->dtype = d->dtype;
    c->m = d->m;
    c->n_panels = d->n_panels;
    c->pb = d->panel_begin;
    c->pe = d->panel_end;
    c->np = c->pe - c->pb;
    c->n_meas = d->n_views * d->det_nu * d->det_nv;
    c->n_vox = d->dims[0] * d->dims[1] * d->dims[2];
    if (c->n_meas >= (1ll << 31) || c->n_vox >= (1ll << 40))
        return bail(fail(c, BCT_EINVAL, "scan too large"));
    c->rb_ptr.assign(d->row_block_ptr, d->row_block_ptr + c->m + 1);
    if (c->rb_ptr[0] != 0) return bail(fail(c, BCT_EINVAL, "row_block_ptr[0] != 0"));
    for (int i = 0; i < c->m; ++i)
        if (c->rb_ptr[i + 1] < c->rb_ptr[i]) return bail(fail(c, BCT_EINVAL, "bad row_block_ptr"));
    c->rb_rows.assign(d->row_block_rows, d->row_block_rows + c->rb_ptr[c->m]);
    for (int64_t g : c->rb_rows)
        if (g < 0 || g >= c->n_meas) return bail(fail(c, BCT_EINVAL, "row block id out of range"));
    const int64_t nL = (int64_t)c->rb_rows.size();
    // column blocks: voxel boxes, ids in C order inside the box (geometry.py:366-383)
    std::vector<Box> boxes(c->n_panels);
    c->col_ptr.assign(1, 0);
    for (int j = 0; j < c->n_panels; ++j) {
        Box &B = boxes[j];
        for (int a = 0; a < 3; ++a) {
            B.lo[a] = d->box_lo[3 * j + a];
            B.hi[a] = d->box_hi[3 * j + a];
            if (B.lo[a] < 0 || B.hi[a] > d->dims[a] || B.lo[a] >= B.hi[a])
                return bail(fail(c, BCT_EINVAL, "column block %d: bad voxel box", j));
        }
        const int64_t bx = B.hi[0] - B.lo[0], by = B.hi[1] - B.lo[1], bz = B.hi[2] - B.lo[2];
        if (bx * by * bz >= (1ll << 24)) return bail(fail(c, BCT_EINVAL, "panel %d too large", j));
        for (int64_t ix = B.lo[0]; ix < B.hi[0]; ++ix)
            for (int64_t iy = B.lo[1]; iy < B.hi[1]; ++iy)
                for (int64_t iz = B.lo[2]; iz < B.hi[2]; ++iz)
                    c->col_vox.push_back((ix * d->dims[1] + iy) * d->dims[2] + iz);
        c->col_ptr.push_back((int64_t)c->col_vox.size());
    }
    c->table_values.assign(d->table_values, d->table_values + (int64_t)c->m * c->n_panels);
    c->table_totals.assign(d->table_totals, d->table_totals + c->n_panels);
    // a source strictly inside an owned box has no defined projection
    // (projector.py:278-284)
    for (int j = c->pb; j < c->pe; ++j)
        for (int64_t v = 0; v < d->n_views; ++v) {
            bool inside = true;
            for (int a = 0; a < 3; ++a) {
                const double s = d->poses[12 * v + a];
                const double plo = d->origin[a] + (double)boxes[j].lo[a] * d->voxel_size[a];
                const double phi = d->origin[a] + (double)boxes[j].hi[a] * d->voxel_size[a];
                inside = inside && s > plo && s < phi;
            }
            if (inside)
                return bail(fail(c, BCT_EINVAL, "source of view %lld lies inside column block %d",
                                 (long long)v, j));
        }
    ScanDev S;
    for (int a = 0; a < 3; ++a) {
        S.origin[a] = d->origin[a];
        S.vsize[a] = d->voxel_size[a];
    }
    S.nu = d->det_nu;
    S.nv = d->det_nv;
    S.du = d->det_du;
    S.dv = d->det_dv;
    double *d_poses = nullptr;
    int64_t *d_edges = nullptr;
    int32_t *d_L = nullptr, *d_counts = nullptr, *d_flags = nullptr, *d_pos = nullptr,
            *d_bad = nullptr;
    DALLOC(d_poses, 12 * d->n_views);
    DALLOC(d_edges, c->m + 1);
    DALLOC(d_L, std::max<int64_t>(nL, 1));
    DALLOC(d_counts, std::max<int64_t>(nL, 1));
    DALLOC(d_flags, std::max<int64_t>(nL, 1));
    DALLOC(d_pos, nL + 1);
    DALLOC(d_bad, 1);
    S.poses = d_poses;
    {
        std::vector<int32_t> L(c->rb_rows.begin(), c->rb_rows.end());
        CK(cudaMemcpy(d_poses, d->poses, 8 * 12 * d->n_views, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_edges, c->rb_ptr.data(), 8 * (c->m + 1), cudaMemcpyHostToDevice));
        if (nL > 0) CK(cudaMemcpy(d_L, L.data(), 4 * nL, cudaMemcpyHostToDevice));
        CK(cudaMemset(d_bad, 0, 4));
    }
    size_t sb = bct::scan_temp_bytes(nL + 1);
    char *cub = nullptr;
    DALLOC(cub, (int64_t)sb);
    double *vals64 = nullptr;
    int32_t *cols = nullptr, *rbp_tmp = nullptr;
    DALLOC(rbp_tmp, c->m + 1);
    for (int lp = 0; lp < c->np; ++lp) {
        const int j = c->pb + lp;
        const Box &B = boxes[j];
        // 1. per-ray counts in row-block order; 2. compaction of the hit rows
        CK(bct::scan_trace_counts(S, d_L, nL, B, d_counts, d_bad, c->stream));
        int32_t bad = 0;
        CK(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (bad) return bail(fail(c, BCT_EINVAL, "degenerate ray (source on a pixel centre)"));
        int64_t n_hit = 0;
        int32_t *l2g = nullptr, *rowlen = nullptr, *ip = nullptr;
        DALLOC(l2g, std::max<int64_t>(nL, 1));
        DALLOC(rowlen, nL + 1);
        if (nL > 0)
            CK(bct::pb_compact(d_counts, nL, d_flags, d_pos, cub, sb, l2g, rowlen, &n_hit,
                               c->stream));
        DALLOC(ip, n_hit + 1);
        CK(cudaMemsetAsync(rowlen + n_hit, 0, 4, c->stream));
        CK(bct::exclusive_scan_i32(rowlen, ip, n_hit + 1, cub, sb, c->stream));
        int32_t nnz32 = 0;
        CK(cudaMemcpyAsync(&nnz32, ip + n_hit, 4, cudaMemcpyDeviceToHost, c->stream));
        // 3. rbp over list positions, then positions -> measurement ids
        CK(bct::pb_rbp(l2g, n_hit, d_edges, c->m, rbp_tmp, c->stream));
        std::vector<int32_t> rb(c->m + 1);
        CK(cudaMemcpyAsync(rb.data(), rbp_tmp, 4 * (c->m + 1), cudaMemcpyDeviceToHost, c->stream));
        CK(bct::gather_i32(d_L, l2g, n_hit, l2g, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        free_tmp(c, rowlen);
        const int64_t nnz = nnz32;
        if (nnz >= (1ll << 30)) return bail(fail(c, BCT_EINVAL, "panel %d too large", j));
        // 4. sorted rows (values + local indices)
        DALLOC(vals64, std::max<int64_t>(nnz, 1));
        DALLOC(cols, std::max<int64_t>(nnz, 1));
        CK(bct::scan_fill(S, l2g, ip, n_hit, B, vals64, cols, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        const int64_t bx = B.hi[0] - B.lo[0], byz = (B.hi[1] - B.lo[1]) * (B.hi[2] - B.lo[2]);
        if ((r = build_panel(c, lp, (int32_t)n_hit, nnz, vals64, cols, ip, l2g, rb, bx, byz)))
            return bail(r);
        free_tmp(c, ip);
        free_tmp(c, vals64);
        free_tmp(c, cols);
    }
    free_tmp(c, rbp_tmp);
    free_tmp(c, cub);
    free_tmp(c, d_L);
    free_tmp(c, d_counts);
    free_tmp(c, d_flags);
    free_tmp(c, d_pos);
    free_tmp(c, d_bad);
    free_tmp(c, d_poses);
    free_tmp(c, d_edges);
    if ((r = finalize(c))) return bail(r);
    *out = c;
    return 0;
}

int bct_destroy(bct_ctx *c)
{
    if (!c) return 0;
    DEVICE_GUARD(c);
    destroy(c);
    return 0;
}

int bct_info(const bct_ctx *c, int64_t *o)
{
    if (!c || !o) return BCT_EINVAL;
    DEVICE_GUARD(c);
    o[0] = c->n_meas; o[1] = c->n_vox; o[2] = c->m; o[3] = c->n_panels;
    o[4] = c->pb; o[5] = c->pe; o[6] = c->nnz; o[7] = c->z_len;
    return 0;
}

int bct_panel_info(const bct_ctx *c, int32_t j, int64_t *n_rows, int64_t *nnz, int64_t *n_cols)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (j < c->pb || j >= c->pe) return BCT_EINVAL;
    const PanelDev &P = c->h_panels[j - c->pb];
    if (n_rows) *n_rows = P.n_rows;
    if (nnz) *nnz = P.nnz;
    if (n_cols) *n_cols = P.n_cols;
    return 0;
}

// The panel back in the reference's cached layout (projector.py:474-488):
// rows in local order, entries in ascending local column.
int bct_get_panel(bct_ctx *c, int32_t j, double *data, int32_t *cols, int64_t *indptr,
                  int64_t *rbp, int64_t *l2g)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (j < c->pb || j >= c->pe) return fail(c, BCT_EINVAL, "panel %d not owned", j);
    int lp = j - c->pb;
    const PanelDev &P = c->h_panels[lp];
    CK(cudaStreamSynchronize(c->stream));
    if (rbp)
        for (int i = 0; i <= c->m; ++i) rbp[i] = c->h_rbp[lp][i];
    if (l2g && P.n_rows > 0) {
        std::vector<int32_t> lg(P.n_rows);
        CK(cudaMemcpy(lg.data(), P.l2g, 4 * P.n_rows, cudaMemcpyDeviceToHost));
        for (int32_t q = 0; q < P.n_rows; ++q) l2g[q] = lg[q];
    }
    if (!data && !cols && !indptr) return 0;   // row maps only
    const int64_t cap = std::max<int64_t>(P.fwd_cap, 1);
    std::vector<double> fv(cap);
    std::vector<uint16_t> fi(cap);
    std::vector<int32_t> sk(P.n_seg + 1), sln(P.n_seg + 1), ssl(P.n_seg + 1), sla(P.n_seg + 1),
        rp(P.n_rows + 1), rs(P.n_seg + 1), stp(P.n_st + 1), sst(P.n_slices + 1),
        lg(std::max(P.n_rows, 1));
    if (c->dtype == BCT_F64) {
        CK(cudaMemcpy(fv.data(), P.fvals, 8 * P.fwd_cap, cudaMemcpyDeviceToHost));
    } else {
        std::vector<float> f(cap);
        CK(cudaMemcpy(f.data(), P.fvals, 4 * P.fwd_cap, cudaMemcpyDeviceToHost));
        for (int64_t q = 0; q < P.fwd_cap; ++q) fv[q] = f[q];
    }
    CK(cudaMemcpy(fi.data(), P.fidx, 2 * P.fwd_cap, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sk.data(), P.seg_key, 4 * (P.n_seg + 1), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sln.data(), P.seg_len, 4 * (P.n_seg + 1), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ssl.data(), P.seg_slice, 4 * (P.n_seg + 1), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sla.data(), P.seg_lane, 4 * (P.n_seg + 1), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rp.data(), P.rseg_ptr, 4 * (P.n_rows + 1), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rs.data(), P.rseg, 4 * (P.n_seg + 1), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(stp.data(), P.st_ptr, 4 * (P.n_st + 1), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sst.data(), P.slice_start, 4 * (P.n_slices + 1), cudaMemcpyDeviceToHost));
    if (P.n_rows > 0) CK(cudaMemcpy(lg.data(), P.l2g, 4 * P.n_rows, cudaMemcpyDeviceToHost));
    const std::vector<int32_t> &d2c = c->h_d2c[lp];
    int64_t o = 0;
    std::vector<std::pair<int32_t, double>> row;
    for (int32_t lr = 0; lr < P.n_rows; ++lr) {
        row.clear();
        for (int q = rp[lr]; q < rp[lr + 1]; ++q) {
            int s = rs[q];
            int basev = stp[sk[s] / P.n_rows];
            for (int e = 0; e < sln[s]; ++e) {
                int64_t pos = sst[ssl[s]] + ((int64_t)(e >> 2) * 32 + sla[s]) * 4 + (e & 3);
                row.push_back({d2c[basev + swz_idx(fi[pos], P.swz_shift)], fv[pos]});
            }
        }
        std::sort(row.begin(), row.end(),
                  [](const std::pair<int32_t, double> &a, const std::pair<int32_t, double> &b) {
                      return a.first < b.first;
                  });
        if (indptr) indptr[lr] = o;
        for (auto &e : row) {
            if (data) data[o] = e.second;
            if (cols) cols[o] = e.first;
            ++o;
        }
    }
    if (indptr) indptr[P.n_rows] = o;
    return 0;
}

int bct_get_table(bct_ctx *c, double *values, double *totals)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (values) std::copy(c->table_values.begin(), c->table_values.end(), values);
    if (totals) std::copy(c->table_totals.begin(), c->table_totals.end(), totals);
    return 0;
}

int bct_get_stream(bct_ctx *c, void **s)
{
    if (!c || !s) return BCT_EINVAL;
    DEVICE_GUARD(c);
    *s = (void *)c->stream;
    return 0;
}

// ---- state I/O (global order <-> panel-major device order) -----------------

__global__ void vox_gather_k(const double *stage, const int32_t *gvox, int64_t n, double *dst)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = stage[gvox[i]];
}

__global__ void vox_scatter_k(const double *src, const int32_t *gvox, int64_t n, double *stage)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) stage[gvox[i]] = src[i];
}

// r = y (the residual of x = 0, z = 0: y - 0.0 is y exactly) and its FP32 copy
__global__ void init_r_k(const double *y, int64_t n, double *r, float *r32)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = y[i];
    r[i] = v;
    if (r32) r32[i] = (float)v;
}

// Image transfers in global voxel order; the permutation runs on the device.
// A context owning every panel moves the whole image in one copy; a shard
// moves only its own voxels on the host side (global order untouched elsewhere).
// Host <-> device copies of state vectors through two pinned chunks: the
// host memcpy of chunk i+1 overlaps the DMA of chunk i (pageable copies run
// at a few GB/s on these hosts).
constexpr size_t PIN_CHUNK = 2u << 20;

static int pin_init(bct_ctx *c)
{
    if (c->h_pin[0]) return 0;
    for (int i = 0; i < 2; ++i) {
        if (cudaMallocHost(&c->h_pin[i], PIN_CHUNK) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->pin_ev[i], cudaEventDisableTiming) != cudaSuccess)
            return fail(c, BCT_ENOMEM, "pinned staging allocation failed");
    }
    return 0;
}

// Page-locked caller buffers (cudaHostAlloc / cudaHostRegister, e.g. a
// pinned torch tensor's numpy view) are copied directly at full DMA rate.
static bool is_pinned(const void *p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

static int h2d_staged(bct_ctx *c, void *dst, const void *src, size_t bytes)
{
    if (bytes > 0 && is_pinned(src)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
        return 0;
    }
    if (int r = pin_init(c)) return r;
    size_t off = 0;
    for (int i = 0; off < bytes; ++i, off += PIN_CHUNK) {
        const int k = i & 1;
        const size_t n = std::min(PIN_CHUNK, bytes - off);
        CK(cudaEventSynchronize(c->pin_ev[k]));   // the DMA that last used chunk k
        memcpy(c->h_pin[k], static_cast<const char *>(src) + off, n);
        CK(cudaMemcpyAsync(static_cast<char *>(dst) + off, c->h_pin[k], n,
                           cudaMemcpyHostToDevice, c->stream));
        CK(cudaEventRecord(c->pin_ev[k], c->stream));
    }
    return 0;
}

static int d2h_staged(bct_ctx *c, void *dst, const void *src, size_t bytes)
{
    if (bytes > 0 && is_pinned(dst)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return 0;
    }
    if (int r = pin_init(c)) return r;
    const size_t nch = (bytes + PIN_CHUNK - 1) / PIN_CHUNK;
    auto issue = [&](size_t i) -> cudaError_t {
        const size_t off = i * PIN_CHUNK, n = std::min(PIN_CHUNK, bytes - off);
        cudaError_t e = cudaMemcpyAsync(c->h_pin[i & 1], static_cast<const char *>(src) + off, n,
                                        cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess) e = cudaEventRecord(c->pin_ev[i & 1], c->stream);
        return e;
    };
    if (nch > 0) CK(issue(0));
    for (size_t i = 0; i < nch; ++i) {
        if (i + 1 < nch) CK(issue(i + 1));
        CK(cudaEventSynchronize(c->pin_ev[i & 1]));
        const size_t off = i * PIN_CHUNK, n = std::min(PIN_CHUNK, bytes - off);
        memcpy(static_cast<char *>(dst) + off, c->h_pin[i & 1], n);
    }
    return 0;
}

static int xvec_to_dev(bct_ctx *c, const double *xg, double *dst)
{
    const unsigned nb = (unsigned)((c->x_len + 255) / 256);
    if (c->np == c->n_panels) {
        if (int r = h2d_staged(c, c->d_xstage, xg, 8 * c->n_vox)) return r;
        if (c->x_len > 0)
            vox_gather_k<<<nb, 256, 0, c->stream>>>(c->d_xstage, c->d_gvox, c->x_len, dst);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(c->stream));
        return 0;
    }
    std::vector<double> buf(std::max<int64_t>(c->x_len, 1));
    for (int lp = 0; lp < c->np; ++lp) {
        const PanelDev &P = c->h_panels[lp];
        const int64_t cb = c->col_ptr[c->pb + lp];
        const std::vector<int32_t> &d2c = c->h_d2c[lp];
        for (int64_t d = 0; d < P.n_cols; ++d) buf[P.x_off + d] = xg[c->col_vox[cb + d2c[d]]];
    }
    CK(cudaMemcpyAsync(dst, buf.data(), 8 * c->x_len, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

static int xvec_from_dev(bct_ctx *c, const double *src, double *xg)
{
    if (c->np == c->n_panels && c->x_len == c->n_vox) {
        const unsigned nb = (unsigned)((c->x_len + 255) / 256);
        if (c->x_len > 0)
            vox_scatter_k<<<nb, 256, 0, c->stream>>>(src, c->d_gvox, c->x_len, c->d_xstage);
        CK(cudaGetLastError());
        return d2h_staged(c, xg, c->d_xstage, 8 * c->n_vox);
    }
    std::vector<double> buf(std::max<int64_t>(c->x_len, 1));
    CK(cudaMemcpyAsync(buf.data(), src, 8 * c->x_len, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int lp = 0; lp < c->np; ++lp) {
        const PanelDev &P = c->h_panels[lp];
        const int64_t cb = c->col_ptr[c->pb + lp];
        const std::vector<int32_t> &d2c = c->h_d2c[lp];
        for (int64_t d = 0; d < P.n_cols; ++d) xg[c->col_vox[cb + d2c[d]]] = buf[P.x_off + d];
    }
    return 0;
}

int bct_set_y(bct_ctx *c, const double *y)
{
    if (!c || !y) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (int r = h2d_staged(c, c->y, y, 8 * c->n_meas)) return r;
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int bct_set_x(bct_ctx *c, const double *x)
{
    if (!c || !x) return BCT_EINVAL;
    DEVICE_GUARD(c);
    return xvec_to_dev(c, x, c->x);
}
int bct_get_x(bct_ctx *c, double *x)
{
    if (!c || !x) return BCT_EINVAL;
    DEVICE_GUARD(c);
    return xvec_from_dev(c, c->x, x);
}
int bct_get_xhat(bct_ctx *c, double *x)
{
    if (!c || !x) return BCT_EINVAL;
    DEVICE_GUARD(c);
    return xvec_from_dev(c, c->xhat, x);
}

int bct_set_x_true(bct_ctx *c, const double *xt)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (!xt) {
        c->has_x_true = false;
        return 0;
    }
    int r = xvec_to_dev(c, xt, c->x_true);
    if (!r) c->has_x_true = true;
    return r;
}

int bct_set_r(bct_ctx *c, const double *r)
{
    if (!c || !r) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (int e = h2d_staged(c, c->r, r, 8 * c->n_meas)) return e;
    CK(cudaStreamSynchronize(c->stream));
    c->r32_valid = false;
    return 0;
}

int bct_get_r(bct_ctx *c, double *r)
{
    if (!c || !r) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (int e = d2h_staged(c, r, c->r, 8 * c->n_meas)) return e;
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

// Panels whose z is in (t, ax) form get it written out (enqueued on the
// context's stream) before anything but a fused batched epoch uses z.
static int materialize_z(bct_ctx *c)
{
    if (!c->z_lazy) return 0;
    CK(bct::z_materialize(c->dtype, c->d_panels, c->np, c->zt, c->zl_mu, c->zl_st, c->zl_on,
                          c->z, c->stream));
    c->z_lazy = false;
    return 0;
}

int bct_set_z(bct_ctx *c, int32_t j, const double *zj)
{
    if (!c || !zj) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (int r = materialize_z(c)) return r;
    if (j < c->pb || j >= c->pe) return fail(c, BCT_EINVAL, "panel %d not owned", j);
    const PanelDev &P = c->h_panels[j - c->pb];
    CK(cudaMemcpyAsync(c->z + P.row_off, zj, 8 * P.n_rows, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int bct_get_z(bct_ctx *c, int32_t j, double *zj)
{
    if (!c || !zj) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (int r = materialize_z(c)) return r;
    if (j < c->pb || j >= c->pe) return fail(c, BCT_EINVAL, "panel %d not owned", j);
    const PanelDev &P = c->h_panels[j - c->pb];
    CK(cudaMemcpyAsync(zj, c->z + P.row_off, 8 * P.n_rows, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int bct_reset_accumulators(bct_ctx *c)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    CK(cudaMemsetAsync(c->xhat, 0, 8 * std::max<int64_t>(c->x_len, 1), c->stream));
    CK(cudaMemsetAsync(c->counts, 0, 4 * std::max(c->np, 1), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int bct_clear_state(bct_ctx *c)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (int r = materialize_z(c)) return r;
    CK(cudaMemsetAsync(c->x, 0, 8 * std::max<int64_t>(c->x_len, 1), c->stream));
    CK(cudaMemsetAsync(c->z, 0, 8 * std::max<int64_t>(c->z_len, 1), c->stream));
    CK(cudaMemsetAsync(c->xhat, 0, 8 * std::max<int64_t>(c->x_len, 1), c->stream));
    CK(cudaMemsetAsync(c->counts, 0, 4 * std::max(c->np, 1), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int bct_get_counts(bct_ctx *c, int64_t *counts)
{
    if (!c || !counts) return BCT_EINVAL;
    DEVICE_GUARD(c);
    std::vector<int32_t> h(std::max(c->np, 1));
    CK(cudaMemcpyAsync(h.data(), c->counts, 4 * c->np, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int j = 0; j < c->n_panels; ++j)
        counts[j] = (j >= c->pb && j < c->pe) ? h[j - c->pb] : 0;
    return 0;
}

int bct_commit_epoch(bct_ctx *c)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    CK(bct::commit(c->d_panels, c->np, c->counts, c->x, c->xhat, c->stream));
    CK(cudaMemsetAsync(c->counts, 0, 4 * std::max(c->np, 1), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int bct_fill_z_from_image(bct_ctx *c)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (int r = materialize_z(c)) return r;
    CK(bct::fill_z(c->dtype, c->d_panels, c->np, c->z_len, c->x, c->z, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

int bct_projection_sum(bct_ctx *c, double *out)
{
    if (!c || !out) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (int r = materialize_z(c)) return r;
    CK(bct::zsum(c->inv_ptr, c->inv_z, c->n_meas, c->z, c->vec, c->stream));
    CK(cudaMemcpyAsync(out, c->vec, 8 * c->n_meas, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}

// r = y - sum_j z^j over every measurement (SolverState.initialize warm start)
int bct_begin_solve(bct_ctx *c, const double *y, const double *x_true)
{
    if (!c || !y) return BCT_EINVAL;
    DEVICE_GUARD(c);
    // z is zeroed: a (t, ax) form left by earlier batched epochs is dropped
    CK(cudaMemsetAsync(c->zl_on, 0, 4 * std::max(c->np, 1), c->stream));
    c->z_lazy = false;
    if (int r = h2d_staged(c, c->y, y, 8 * c->n_meas)) return r;
    CK(cudaMemsetAsync(c->x, 0, 8 * std::max<int64_t>(c->x_len, 1), c->stream));
    CK(cudaMemsetAsync(c->z, 0, 8 * std::max<int64_t>(c->z_len, 1), c->stream));
    CK(cudaMemsetAsync(c->xhat, 0, 8 * std::max<int64_t>(c->x_len, 1), c->stream));
    CK(cudaMemsetAsync(c->counts, 0, 4 * std::max(c->np, 1), c->stream));
    if (c->n_meas > 0)
        init_r_k<<<(unsigned)((c->n_meas + 255) / 256), 256, 0, c->stream>>>(c->y, c->n_meas, c->r,
                                                                           c->r32);
    CK(cudaGetLastError());
    c->r32_valid = c->r32 != nullptr;
    if (!x_true) {
        c->has_x_true = false;
        return 0;
    }
    if (c->np == c->n_panels) {   // one copy + the device permutation, no host wait
        if (int r = h2d_staged(c, c->d_xstage, x_true, 8 * c->n_vox)) return r;
        if (c->x_len > 0)
            vox_gather_k<<<(unsigned)((c->x_len + 255) / 256), 256, 0, c->stream>>>(
                c->d_xstage, c->d_gvox, c->x_len, c->x_true);
        CK(cudaGetLastError());
        c->has_x_true = true;
        return 0;
    }
    int r = xvec_to_dev(c, x_true, c->x_true);
    if (!r) c->has_x_true = true;
    return r;
}

int bct_reset_residual(bct_ctx *c)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (int r = materialize_z(c)) return r;
    CK(bct::zsum(c->inv_ptr, c->inv_z, c->n_meas, c->z, c->vec, c->stream));
    CK(bct::sub(c->y, c->vec, c->n_meas, c->r, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->r32_valid = false;
    return 0;
}

int bct_forward(bct_ctx *c, const double *x, double *y_out)
{
    if (!c || !x || !y_out) return BCT_EINVAL;
    DEVICE_GUARD(c);
    double *dx = nullptr;
    CK(cudaMalloc((void **)&dx, 8 * std::max<int64_t>(c->x_len, 1)));
    int r = xvec_to_dev(c, x, dx);
    if (!r) {
        cudaError_t e = bct::forward(c->dtype, c->d_panels, c->np, c->inv_ptr, c->inv_z, c->n_meas,
                                     dx, c->vec, c->stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(y_out, c->vec, 8 * c->n_meas, cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) r = fail(c, BCT_ECUDA, "forward: %s", cudaGetErrorString(e));
    }
    cudaFree(dx);
    return r;
}

int bct_audit(bct_ctx *c, double *drift)
{
    if (!c || !drift) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (int r = materialize_z(c)) return r;
    CK(bct::zsum(c->inv_ptr, c->inv_z, c->n_meas, c->z, c->vec, c->stream));
    CK(cudaMemsetAsync(c->audit2, 0, 16, c->stream));
    CK(bct::audit(c->y, c->r, c->vec, c->n_meas, c->audit2, c->stream));
    unsigned long long h[2];
    CK(cudaMemcpyAsync(h, c->audit2, 16, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    double d, a;
    memcpy(&d, &h[0], 8);
    memcpy(&a, &h[1], 8);
    if (a == 0.0) a = 1.0;
    *drift = d / a;
    return 0;
}

// ---- epochs ---------------------------------------------------------------

static int launch_staged(bct_ctx *c, int64_t n_tasks, int64_t n_visits, const UpLayout &L,
                         const std::function<int(Slot &)> &before_epoch = nullptr)
{
    int s = c->head;
    Slot &S = c->slots[s];
    if (S.pending) {
        // ring full: retire the oldest result implicitly
        CK(cudaEventSynchronize(S.done));
        S.pending = false;
        c->tail = (c->tail + 1) % RING;
    }
    {
        // upload on the copy stream (it overlaps the previous epoch); buffer
        // b was last read by the epoch before the previous one (free_b[b],
        // recorded when the previous epoch was launched)
        const int b = c->up_i;
        CK(cudaStreamWaitEvent(c->cstream, c->free_b[b], 0));
        CK(cudaMemcpyAsync(c->d_up, c->h_up, L.total, cudaMemcpyHostToDevice, c->cstream));
        CK(cudaEventRecord(c->staged_b[b], c->cstream));
        // all work queued so far (the previous epoch and its all-reduce /
        // finish) is the last reader of the other buffer
        CK(cudaEventRecord(c->free_b[b ^ 1], c->stream));
        CK(cudaStreamWaitEvent(c->stream, c->staged_b[b], 0));
    }
    c->cur_masks = reinterpret_cast<uint64_t *>(c->d_up + L.masks);
    c->cur_tasks = reinterpret_cast<TaskDev *>(c->d_up + L.tasks);
    c->mus = reinterpret_cast<double *>(c->d_res + RES_HEAD);
    c->statuses = reinterpret_cast<int32_t *>(c->d_res + RES_HEAD + 8 * (size_t)n_tasks);
    S.plan_user = nullptr;
    S.n_plan = 0;
    if (before_epoch) {
        int r = before_epoch(S);
        if (r) return r;
    }
    EpochParams p;
    memset(&p, 0, sizeof p);
    p.panels = c->d_panels;
    p.n_panels_owned = c->np; p.m = c->m; p.n_meas = c->n_meas; p.z_len = c->z_len;
    p.x_len = c->x_len; p.inv_ptr = c->inv_ptr; p.inv_z = c->inv_z;
    p.invt = c->invt; p.invt_off = c->invt_off; p.rb_ptr = c->d_rb_ptr;
    p.rb_rows = c->d_rb_rows; p.rb_of_row = c->rb_of_row; p.y = c->y; p.r = c->r; p.r32 = c->r32; p.z = c->z;
    p.x = c->x; p.xhat = c->xhat; p.counts = c->counts;
    p.x_true = c->has_x_true ? c->x_true : nullptr;
    p.hdr = reinterpret_cast<const EpochHeader *>(c->d_up);
    p.tasks = reinterpret_cast<const TaskDev *>(c->d_up + L.tasks);
    p.gx = c->gx; p.gx_stride = 2 * c->max_cols;
    p.t_ax = c->t_ax; p.seg_part = c->seg_part; p.part = c->part; p.mus = c->mus;
    p.band_cap = c->band_cap; p.band_dbuf = c->band_dbuf;
    p.gx_batch = c->gx_batch; p.seg_batch = c->seg_batch; p.tax_batch = c->tax_batch;
    p.zt = c->zt; p.zl_on = c->zl_on; p.zl_st = c->zl_st; p.zl_mu = c->zl_mu;
    p.part_task = c->part_task;
    p.statuses = c->statuses; p.out = c->out; p.res_host = S.d_hres;
    p.exchange = c->exchange; p.bar = c->bar; p.ticket = c->ticket;
    p.cta_split = c->cta_split;
    p.guard_ref = c->guard_ref;
    p.prep = c->d_up + L.prep;
    p.masks = c->cur_masks;
    p.mw = c->mw;
    p.prep_smem_off = c->prep_off;
    p.prep_dims = c->pd;
    p.timeline = nullptr;
    if (getenv("BCT_TIMELINE") && n_tasks > 0) {
        if (c->timeline_tasks < n_tasks) {
            if (c->timeline) cudaFree(c->timeline);
            CK(cudaMalloc((void **)&c->timeline, 8 * 16 * (size_t)n_tasks * c->grid));
            c->timeline_tasks = n_tasks;
        }
        p.timeline = c->timeline;
        p.tl_tasks = c->timeline_tasks;
    }
    CK(cudaEventRecord(S.t0, c->stream));
    cudaError_t e;
    bct::launch_epoch(p, c->dtype, c->grid, c->block, c->smem_total, c->stream, &e);
    if (e != cudaSuccess) return fail(c, BCT_ECUDA, "epoch launch: %s", cudaGetErrorString(e));
    CK(cudaEventRecord(S.t1, c->stream));
    // the last block wrote the result into the slot's mapped block (no copy
    // on the stream); a sharded epoch's norms follow from bct_finish_sharded
    CK(cudaEventRecord(S.done, c->stream));
    S.n_tasks = n_tasks;
    S.n_visits = n_visits;
    S.pending = true;
    c->head = (c->head + 1) % RING;
    return 0;
}

static int plan_and_launch(bct_ctx *c, int32_t mode, int32_t flags, std::vector<TaskDev> &tasks,
                           std::vector<uint64_t> &tmasks, const std::vector<uint64_t> &emask,
                           const std::function<int(Slot &)> &hook, bool host_masks);

int bct_run_epoch(bct_ctx *c, int32_t mode, int64_t n_tasks, const int32_t *task_j,
                  const int32_t *task_visit, const int64_t *task_gptr, const int64_t *sel,
                  const double *betas, int32_t flags)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (mode != BCT_SERIAL_FAITHFUL && mode != BCT_PARALLEL)
        return fail(c, BCT_EINVAL, "mode %d", mode);
    if (n_tasks < 0 || (n_tasks > 0 && (!task_j || !task_visit || !task_gptr || !sel || !betas)))
        return fail(c, BCT_EINVAL, "null plan arrays");
    const bool sharded = (flags & BCT_SHARDED) != 0;
    if (sharded && mode != BCT_PARALLEL)
        return fail(c, BCT_EINVAL, "sharded execution requires parallel mode");
    // validate and pack before touching the device (a failed batch leaves no trace)
    const int mw = c->mw;
    std::vector<TaskDev> tasks;
    std::vector<uint64_t> tmasks;        // mw words per kept task
    std::vector<uint64_t> emask(mw, 0);  // union of every drawn block (all ranks' tasks)
    std::vector<uint64_t> mk(mw);
    tasks.reserve(n_tasks);
    for (int64_t k = 0; k < n_tasks; ++k) {
        int j = task_j[k];
        if (j < 0 || j >= c->n_panels)
            return fail(c, BCT_ESCHEDULE, "task %lld: volume block %d out of range",
                        (long long)k, j);
        if (task_gptr[k + 1] < task_gptr[k])
            return fail(c, BCT_ESCHEDULE, "task %lld: negative group size", (long long)k);
        std::fill(mk.begin(), mk.end(), 0ull);
        for (int64_t q = task_gptr[k]; q < task_gptr[k + 1]; ++q) {
            int64_t i = sel[q];
            if (i < 0 || i >= c->m)
                return fail(c, BCT_ESCHEDULE, "task %lld: measurement block %lld out of range",
                            (long long)k, (long long)i);
            if (has_bit(mk.data(), (int)i))
                return fail(c, BCT_ESCHEDULE, "task %lld: repeated measurement block %lld",
                            (long long)k, (long long)i);
            set_mask(mk.data(), (int)i);
        }
        for (int w = 0; w < mw; ++w) emask[w] |= mk[w];
        if (j < c->pb || j >= c->pe) {
            if (!sharded)
                return fail(c, BCT_ESCHEDULE, "task %lld: volume block %d not owned", (long long)k,
                            j);
            continue;  // another rank's column block
        }
        if (!std::isfinite(betas[k]))
            return fail(c, BCT_ESCHEDULE, "task %lld: non-finite beta", (long long)k);
        TaskDev T;
        memset(&T, 0, sizeof T);
        T.lp = j - c->pb;
        T.j = j;
        T.visit = task_visit[k];
        T.beta = betas[k];
        if (task_gptr[k + 1] - task_gptr[k] == c->m) T.flags |= TASK_FULL;
        tasks.push_back(T);
        tmasks.insert(tmasks.end(), mk.begin(), mk.end());
    }
    return plan_and_launch(c, mode, flags, tasks, tmasks, emask, nullptr, true);
}

// Host restatement of epoch.cu build_runs / prep_task: the per-task path's
// set-up of one task (its TaskDev, panel, mask runs and the visit's drawn
// rows), built with the plan so the kernel copies it instead of walking a
// chain of dependent device loads per task.
static void host_prep(const bct_ctx *c, const TaskDev &T, const uint64_t *mask,
                      const uint64_t *vmask, char *rec)
{
    PrepView R(rec, c->pd);
    PrepHdr &H = *R.h;
    H.T = T;
    H.P = c->h_panels[T.lp];
    const std::vector<int32_t> &rbp = c->h_rbp[T.lp];
    const std::vector<int32_t> &stbs = c->h_stbs[T.lp];
    const int m = c->m;
    int n = 0, acc = 0;
    for (int i = 0; i < m;) {
        if (!has_bit(mask, i)) { ++i; continue; }
        const int s = i;
        while (i < m && has_bit(mask, i)) ++i;
        R.i0[n] = s;
        R.i1[n] = i;
        R.rows0[n] = rbp[s];
        R.pre[n] = acc;
        acc += rbp[i] - rbp[s];
        ++n;
    }
    R.pre[n] = acc;
    H.n_runs = n;
    int uacc = 0;
    for (int st = 0; st < H.P.n_st; ++st) {
        R.st_pre[st] = uacc;
        const int32_t *sb = stbs.data() + (size_t)st * (m + 1);
        for (int q = 0; q < n; ++q) uacc += sb[R.i1[q]] - sb[R.i0[q]];
    }
    R.st_pre[H.P.n_st] = uacc;
    H.nst = H.P.n_st;
    H.full = (n == 1 && R.i0[0] == 0 && R.i1[0] == m);
    int nv = 0;
    acc = 0;
    for (int i = 0; i < m; ++i) {
        if (!has_bit(vmask, i)) continue;
        R.vb[nv] = i;
        R.vpre[nv] = acc;
        acc += (int)(c->rb_ptr[i + 1] - c->rb_ptr[i]);
        ++nv;
    }
    R.vpre[nv] = acc;
    H.nvb = nv;
}

// Visit flags/masks, batched-path prefixes and scratch, staging and launch of
// a validated task list (shared by bct_run_epoch and bct_sample_epoch; the
// hook runs on the stream between the plan upload and the epoch kernel).
// tmasks: each task's row-block set (mw words; zeros when the device sampler
// fills them), emask: the epoch's drawn blocks (zeros: the sampler ORs them).
static int plan_and_launch(bct_ctx *c, int32_t mode, int32_t flags, std::vector<TaskDev> &tasks,
                           std::vector<uint64_t> &tmasks, const std::vector<uint64_t> &emask,
                           const std::function<int(Slot &)> &hook, bool host_masks)
{
    const int mw = c->mw;
    const int64_t nt = (int64_t)tasks.size();
    // visit boundaries and masks
    std::vector<uint64_t> vmasks((size_t)nt * mw, 0ull);
    int64_t n_visits = 0;
    for (int64_t a = 0; a < nt;) {
        int64_t b = a;
        while (b < nt && tasks[b].visit == tasks[a].visit && tasks[b].j == tasks[a].j) ++b;
        for (int64_t q = a; q < b; ++q)
            for (int w = 0; w < mw; ++w) vmasks[(size_t)a * mw + w] |= tmasks[(size_t)q * mw + w];
        for (int64_t q = a; q < b; ++q) {
            if (q > a)
                std::copy(vmasks.begin() + (size_t)a * mw, vmasks.begin() + (size_t)(a + 1) * mw,
                          vmasks.begin() + (size_t)q * mw);
            tasks[q].flags |= (q == a ? TASK_FIRST_OF_VISIT : 0) | (q == b - 1 ? TASK_LAST_OF_VISIT : 0);
        }
        ++n_visits;
        a = b;
    }
    int r = ensure_task_cap(c, std::max<int64_t>(nt, 1));
    if (r) return r;
    // epoch-batched path: parallel epoch whose tasks are all full panels
    bool batched = mode == BCT_PARALLEL && nt > 0 && nt <= bct::MAX_BATCH_TASKS && !getenv("BCT_NO_BATCH");
    for (int64_t k = 0; batched && k < nt; ++k)
        if (!(tasks[k].flags & TASK_FULL)) batched = false;
    // phase D writes each task's z and each panel's x_hat without ordering
    // between tasks: two full-panel tasks of one column block in an epoch (a
    // scripted plan: a repeated visit, or a visit with two full groups) would
    // race where the reference keeps plan order (executor.py:200-213,
    // 247-248), so such plans run on the per-task path
    if (batched) {
        std::vector<char> seen(c->np, 0);
        for (int64_t k = 0; k < nt && batched; ++k) {
            if (seen[tasks[k].lp]) batched = false;
            seen[tasks[k].lp] = 1;
        }
    }
    int64_t tot_tiles = 0, tot_slices = 0, tot_rows = 0, tot_vox = 0, gxo = 0, sgo = 0, txo = 0;
    int64_t tot_ent = 0;
    if (batched) {
        for (int64_t k = 0; k < nt; ++k) {
            TaskDev &T = tasks[k];
            const PanelDev &P = c->h_panels[T.lp];
            T.tile_pre = (int32_t)tot_tiles;
            T.slice_pre = (int32_t)tot_slices;
            T.row_pre = (int32_t)tot_rows;
            T.vox_pre = (int32_t)tot_vox;
            T.gx_off = gxo;
            T.seg_off = sgo;
            T.tax_off = txo;
            T.ent_pre = tot_ent;
            tot_ent += P.fwd_cap;
            tot_tiles += P.n_tiles;
            tot_slices += P.n_slices;
            tot_rows += P.n_rows;
            if (T.flags & TASK_FIRST_OF_VISIT) tot_vox += P.n_cols;
            gxo += P.n_cols;
            sgo += (int64_t)P.n_slices * 32;
            txo += P.n_rows;
        }
        if (tot_slices >= (1ll << 31) || tot_rows >= (1ll << 31) || gxo >= (1ll << 31) ||
            tot_tiles >= (1ll << 31) || tot_vox >= (1ll << 31))
            batched = false;
    }
    // phase D folded into the tail: per owned panel its z / x offsets, its
    // task, z form and (g, x) offset in shared memory (epoch.cu tail)
    const bool fuse = batched && !getenv("BCT_NO_FUSE_TAIL") &&
                      (size_t)(c->np + 1) * bct::FT_PANEL_BYTES + (size_t)nt * 16 + 64 <= c->smem;
    if (batched) {
        // the device may still read the old scratch: drain before growing it
        auto grow = [&](double **ptr, int64_t *have, int64_t need) -> int {
            if (need <= *have) return 0;
            CK(cudaStreamSynchronize(c->stream));
            if (*ptr) cudaFree(*ptr);
            CK(cudaMalloc((void **)ptr, 8 * std::max<int64_t>(need, 1)));
            *have = need;
            return 0;
        };
        if ((r = grow(&c->gx_batch, &c->gx_batch_n, 2 * gxo))) return r;
        if ((r = grow(&c->seg_batch, &c->seg_batch_n, 2 * sgo))) return r;
        if (!fuse && (r = grow(&c->tax_batch, &c->tax_batch_n, 2 * txo))) return r;
        if ((r = grow(&c->part_task, &c->part_task_n, 33 * nt * (int64_t)c->grid + nt))) return r;
    }
    // switch upload buffers; this one's copy (two epochs ago) must be done
    c->up_i ^= 1;
    c->d_up = c->d_upb[c->up_i];
    c->h_up = c->h_upb[c->up_i];
    CK(cudaEventSynchronize(c->staged_b[c->up_i]));
    const bool host_prep_on = !batched && host_masks && nt > 0;
    const UpLayout L = up_layout(c, nt, host_prep_on);
    EpochHeader *hh = reinterpret_cast<EpochHeader *>(c->h_up);
    memset(hh, 0, sizeof(EpochHeader));
    hh->n_tasks = (int32_t)nt;
    hh->mode = mode;
    hh->flags = flags;
    c->cur_flags = flags;
    hh->batched = batched ? 1 : 0;
    hh->n_tiles_total = (int32_t)tot_tiles;
    hh->n_slices_total = (int32_t)tot_slices;
    hh->n_rows_total = (int32_t)tot_rows;
    hh->n_vox_total = (int32_t)tot_vox;
    hh->n_ent_total = tot_ent;
    hh->guard_factor = c->guard_factor;
    hh->r32_valid = c->r32_valid ? 1 : 0;
    hh->fuse_tail = fuse ? 1 : 0;
    if (hh->fuse_tail && !c->zt) {
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaMalloc(&c->zt, bct::zt_pair_bytes(c->dtype) * std::max<int64_t>(c->z_len, 1)));
    }
    // any other epoch reads the stored z
    if (!hh->fuse_tail) {
        if ((r = materialize_z(c))) return r;
    }
    // a batched FP32 epoch refreshes the copy before phase A
    if (batched && c->dtype == BCT_F32) c->r32_valid = true;
    if (nt) memcpy(c->h_up + L.tasks, tasks.data(), sizeof(TaskDev) * nt);
    // masks: the epoch's, then per task its group and its visit's union
    uint64_t *hm = reinterpret_cast<uint64_t *>(c->h_up + L.masks);
    std::copy(emask.begin(), emask.end(), hm);
    for (int64_t k = 0; k < nt; ++k) {
        std::copy(tmasks.begin() + (size_t)k * mw, tmasks.begin() + (size_t)(k + 1) * mw,
                  hm + task_mask_off(k, mw));
        std::copy(vmasks.begin() + (size_t)k * mw, vmasks.begin() + (size_t)(k + 1) * mw,
                  hm + visit_mask_off(k, mw));
    }
    // per-task path with host-known masks: every task's set-up built here
    hh->host_prep = host_prep_on ? 1 : 0;
    if (host_prep_on)
        for (int64_t k = 0; k < nt; ++k)
            host_prep(c, tasks[k], tmasks.data() + (size_t)k * mw, vmasks.data() + (size_t)k * mw,
                      c->h_up + L.prep + c->pd.bytes() * k);
    r = launch_staged(c, nt, n_visits, L, hook);
    if (r == 0 && hh->fuse_tail) c->z_lazy = true;
    return r;
}

int bct_set_divergence_factor(bct_ctx *c, double factor)
{
    if (!c || !(factor > 0.0)) return BCT_EINVAL;
    c->guard_factor = factor;
    return 0;
}

int bct_wait_epoch(bct_ctx *c, bct_epoch_result *o, double *mus, int32_t *statuses)
{
    if (!c || !o) return BCT_EINVAL;
    DEVICE_GUARD(c);
    Slot &S = c->slots[c->tail];
    if (!S.pending) return fail(c, BCT_EINVAL, "no pending epoch");
    // poll (the epoch is usually a fraction of a millisecond away): a
    // blocking wait parks the thread and pays the OS wake-up on every epoch
    for (int spin = 0; spin < (1 << 22); ++spin) {
        const cudaError_t q = cudaEventQuery(S.done);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) return fail(c, BCT_ECUDA, "epoch: %s", cudaGetErrorString(q));
    }
    CK(cudaEventSynchronize(S.done));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, BCT_ECUDA, "epoch: %s", cudaGetErrorString(e));
    const EpochOut *ho = reinterpret_cast<const EpochOut *>(S.h_res);
    o->n_tasks = S.n_tasks;
    o->n_visits = S.n_visits;
    o->n_degenerate = ho->n_degenerate;
    o->resid_sq = ho->resid_sq;
    o->x_sq = ho->x_sq;
    o->err_sq = ho->err_sq;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, S.t0, S.t1);
    o->kernel_ms = ms;
    if (mus) memcpy(mus, S.h_res + RES_HEAD, 8 * S.n_tasks);
    if (statuses) memcpy(statuses, S.h_res + RES_HEAD + 8 * S.n_tasks, 4 * S.n_tasks);
    if (S.plan_user)
        for (int64_t q = 0; q < S.n_plan; ++q) S.plan_user[q] = S.h_plan[q];
    S.plan_user = nullptr;
    S.pending = false;
    c->tail = (c->tail + 1) % RING;
    return 0;
}

// Profiling: phase timestamps of the last epoch (BCT_TIMELINE=1), [2][task][8][grid]
// (the second half: per-task sub-phase marks); out holds 16 * n_tasks * grid.
int bct_debug_timeline(bct_ctx *c, long long *out, int64_t n_tasks, int32_t *grid)
{
    if (!c || !grid) return BCT_EINVAL;
    DEVICE_GUARD(c);
    *grid = c->grid;
    if (!c->timeline || !out) return 0;
    CK(cudaStreamSynchronize(c->stream));
    const size_t nt = (size_t)std::min(n_tasks, c->timeline_tasks), half = 8 * nt * c->grid;
    CK(cudaMemcpy(out, c->timeline, 8 * half, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out + half, c->timeline + 8 * (size_t)c->timeline_tasks * c->grid, 8 * half,
                  cudaMemcpyDeviceToHost));
    return 0;
}

int bct_exchange_buffer(bct_ctx *c, double **dev_ptr, int64_t *len)
{
    if (!c || !dev_ptr || !len) return BCT_EINVAL;
    DEVICE_GUARD(c);
    *dev_ptr = c->exchange;
    *len = c->n_meas + 2;
    return 0;
}

int bct_finish_sharded(bct_ctx *c, int32_t flags, double *resid_sq)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    // the drawn blocks of the last epoch, as the device saw them (host plan or sampler)
    const uint64_t *dmask = c->cur_masks;   // epoch mask first (EpochParams::masks)
    if (!dmask) return fail(c, BCT_EINVAL, "no sharded epoch submitted");
    const int nb = 8 * c->grid;   // c->part holds 8 * grid + 8 partials
    // flags: the epoch's BCT_GUARD / BCT_GUARD_REF (a skipped epoch skips its finish)
    Slot &S = c->slots[(c->head + RING - 1) % RING];
    FinishGuard guard{&c->out->x_sq, c->guard_ref, c->guard_factor, (flags & BCT_GUARD) ? 1 : 0,
                      (flags & BCT_GUARD_REF) ? 1 : 0,
                      S.pending ? reinterpret_cast<EpochOut *>(S.d_hres) : nullptr};
    CK(bct::sharded_finish(c->y, c->exchange, c->n_meas, c->rb_of_row, dmask, c->m, c->r, c->r32,
                           c->part, nb, c->exchange + c->n_meas, c->out, c->ticket, guard,
                           c->stream));
    // the epoch's mapped result block (slot of the last submitted epoch) now
    // carries the global norms (written by the finish's last block)
    if (S.pending) CK(cudaEventRecord(S.done, c->stream));
    if (resid_sq) {   // synchronous form
        double s = 0.0;
        CK(cudaMemcpyAsync(&s, &c->out->resid_sq, 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        *resid_sq = s;
    }
    return 0;
}

int bct_sample_epoch(bct_ctx *c, int32_t mode, int32_t n_visits, const int32_t *visit_j,
                     const double *exp_variates, int64_t n_variates, const int32_t *draws,
                     int32_t group_size, double b, int32_t strategy, double theta,
                     int32_t flags, int64_t *plan_ids_out)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (mode != BCT_SERIAL_FAITHFUL && mode != BCT_PARALLEL)
        return fail(c, BCT_EINVAL, "mode %d", mode);
    if (strategy < BCT_IMPORTANCE || strategy > BCT_MIXED)
        return fail(c, BCT_EINVAL, "strategy %d", strategy);
    if (group_size < 1) return fail(c, BCT_EINVAL, "group_size %d", group_size);
    if (n_visits < 0 || (n_visits > 0 && (!visit_j || !draws)) ||
        (n_variates > 0 && !exp_variates))
        return fail(c, BCT_EINVAL, "null sampler arrays");
    const bool sharded = (flags & BCT_SHARDED) != 0;
    if (sharded && mode != BCT_PARALLEL)
        return fail(c, BCT_EINVAL, "sharded execution requires parallel mode");
    // structure of the plan from the host table (sampling.py:140-152): scope,
    // variate offsets, task skeletons; the ids/masks/betas come from the device
    std::vector<bct::SampleVisit> vis(n_visits);
    std::vector<TaskDev> tasks;
    std::vector<uint64_t> emask(c->mw, 0ull);    // ORed by the sampler on the device
    std::vector<uint64_t> tmasks;                // written by the sampler
    int64_t var_off = 0, id_off = 0;
    for (int32_t v = 0; v < n_visits; ++v) {
        const int j = visit_j[v];
        if (j < 0 || j >= c->n_panels)
            return fail(c, BCT_ESCHEDULE, "visit %d: volume block %d out of range", v, j);
        int scope = 0;
        for (int i = 0; i < c->m; ++i) scope += c->table_values[(int64_t)i * c->n_panels + j] > 0.0;
        if (draws[v] < 0 || draws[v] > scope)
            return fail(c, BCT_ESCHEDULE, "cannot draw %d blocks from %d in scope", draws[v], scope);
        if (draws[v] > 0 && !(c->table_totals[j] > 0.0))
            return fail(c, BCT_ESCHEDULE, "volume block %d has no selectable measurement blocks",
                        j);
        bct::SampleVisit &V = vis[v];
        V.j = j;
        V.draws = draws[v];
        V.var_off = (int32_t)var_off;
        V.id_off = (int32_t)id_off;
        V.task_base = -1;
        var_off += scope;
        id_off += draws[v];
        const bool owned = j >= c->pb && j < c->pe;
        if (!owned && !sharded)
            return fail(c, BCT_ESCHEDULE, "visit %d: volume block %d not owned", v, j);
        if (!owned) continue;
        const int ng = (draws[v] + group_size - 1) / group_size;
        V.task_base = (int32_t)tasks.size();
        for (int t = 0; t < ng; ++t) {
            TaskDev T;
            memset(&T, 0, sizeof T);
            T.lp = j - c->pb;
            T.j = j;
            T.visit = v;
            // full group <=> it holds every row block (masks are filled on the device)
            if (std::min(group_size, draws[v] - t * group_size) == c->m) T.flags |= TASK_FULL;
            tasks.push_back(T);
            tmasks.resize(tmasks.size() + c->mw, 0ull);
        }
    }
    if (var_off != n_variates)
        return fail(c, BCT_ESCHEDULE, "%lld variates for %lld in-scope blocks",
                    (long long)n_variates, (long long)var_off);
    // device inputs (grow-only; drained before reallocation)
    auto grow = [&](auto **ptr, int64_t *have, int64_t need, size_t elt) -> int {
        if (need <= *have) return 0;
        CK(cudaStreamSynchronize(c->stream));
        if (*ptr) cudaFree(*ptr);
        CK(cudaMalloc((void **)ptr, elt * std::max<int64_t>(need, 1)));
        *have = need;
        return 0;
    };
    int r;
    if (!c->d_values) {
        CK(cudaMalloc((void **)&c->d_values, 8 * std::max<size_t>(c->table_values.size(), 1)));
        CK(cudaMalloc((void **)&c->d_totals, 8 * std::max<size_t>(c->table_totals.size(), 1)));
        CK(cudaMemcpy(c->d_values, c->table_values.data(), 8 * c->table_values.size(),
                      cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->d_totals, c->table_totals.data(), 8 * c->table_totals.size(),
                      cudaMemcpyHostToDevice));
    }
    if ((r = grow(&c->d_exp, &c->d_exp_n, n_variates, 8))) return r;
    if ((r = grow(&c->d_visits, &c->d_visits_n, n_visits, sizeof(bct::SampleVisit)))) return r;
    if ((r = grow(&c->d_plan, &c->d_plan_n, id_off, 4))) return r;
    // variates and visits are copied synchronously: the caller's buffers are
    // free on return, and the previous epoch may still read nothing of these
    auto hook = [&](Slot &S) -> int {
        if (n_variates > 0)
            CK(cudaMemcpyAsync(c->d_exp, exp_variates, 8 * n_variates, cudaMemcpyHostToDevice,
                               c->stream));
        if (n_visits > 0)
            CK(cudaMemcpyAsync(c->d_visits, vis.data(), sizeof(bct::SampleVisit) * n_visits,
                               cudaMemcpyHostToDevice, c->stream));
        bct::SamplerParams sp;
        sp.values = c->d_values;
        sp.totals = c->d_totals;
        sp.n_panels = c->n_panels;
        sp.m = c->m;
        sp.visits = c->d_visits;
        sp.exp = c->d_exp;
        sp.strategy = strategy;
        sp.theta = theta;
        sp.group_size = group_size;
        sp.b = b;
        sp.tasks = c->cur_tasks;   // this epoch's upload block (launch_staged)
        sp.masks = c->cur_masks;
        sp.mw = c->mw;
        sp.plan_ids = c->d_plan;
        cudaError_t e;
        bct::launch_sampler(sp, n_visits, c->stream, &e);
        if (e != cudaSuccess) return fail(c, BCT_ECUDA, "sampler launch: %s", cudaGetErrorString(e));
        if (plan_ids_out && id_off > 0) {
            if (S.plan_cap < id_off) {
                if (S.h_plan) cudaFreeHost(S.h_plan);
                CK(cudaHostAlloc((void **)&S.h_plan, 4 * id_off, cudaHostAllocDefault));
                S.plan_cap = id_off;
            }
            CK(cudaMemcpyAsync(S.h_plan, c->d_plan, 4 * id_off, cudaMemcpyDeviceToHost,
                               c->stream));
            S.plan_user = plan_ids_out;
            S.n_plan = id_off;
        }
        return 0;
    };
    return plan_and_launch(c, mode, flags, tasks, tmasks, emask, hook, false);
}

}  // extern "C"

// ---- whole-system baselines (solvers.py:283-379; baseline.cu) -------------

int bct_baseline_init(bct_ctx *c, int32_t kind, int32_t m_rule)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (kind != BCT_ROW_ACTION && kind != BCT_COLUMN_ACTION)
        return fail(c, BCT_EINVAL, "baseline kind %d", kind);
    if (m_rule < BCT_M_IDENTITY || m_rule > BCT_M_NORM_INVERSE)
        return fail(c, BCT_EINVAL, "m_rule %d", m_rule);
    if (c->pb != 0 || c->pe != c->n_panels)
        return fail(c, BCT_EINVAL, "baselines need every volume block on this context");
    CK(cudaStreamSynchronize(c->stream));
    if (!c->bm_built) {
        CK(bct::baseline_build(c->dtype, c->h_panels.data(), c->np, c->d_gvox, c->n_meas, c->n_vox,
                               c->bm, c->stream));
        DALLOC(c->bl_diag, std::max(c->n_meas, c->n_vox));
        DALLOC(c->bl_x, c->n_vox);
        DALLOC(c->bl_r, c->n_meas);
        DALLOC(c->bl_tmp, std::max(c->n_meas, c->n_vox));
        DALLOC(c->bl_part, 4 * 148);
        DALLOC(c->bl_out, 4);
        std::vector<int32_t> cb(c->n_vox, -1);
        for (int j = 0; j < c->n_panels; ++j)
            for (int64_t q = c->col_ptr[j]; q < c->col_ptr[j + 1]; ++q) cb[c->col_vox[q]] = j;
        DALLOC(c->bl_cb_of_vox, c->n_vox);
        DALLOC(c->bl_col_vox, std::max<int64_t>((int64_t)c->col_vox.size(), 1));
        CK(cudaMemcpy(c->bl_cb_of_vox, cb.data(), 4 * c->n_vox, cudaMemcpyHostToDevice));
        if (!c->col_vox.empty())
            CK(cudaMemcpy(c->bl_col_vox, c->col_vox.data(), 8 * c->col_vox.size(),
                          cudaMemcpyHostToDevice));
        c->bm_built = true;
    }
    CK(bct::baseline_scale(c->bm, kind, m_rule, c->bl_diag, c->stream));
    CK(cudaMemsetAsync(c->bl_x, 0, 8 * c->n_vox, c->stream));
    CK(cudaMemcpyAsync(c->bl_r, c->y, 8 * c->n_meas, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemsetAsync(c->bl_tmp, 0, 8 * std::max(c->n_meas, c->n_vox), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->bl_kind = kind;
    return 0;
}

int bct_baseline_epoch(bct_ctx *c, double omega, double *norms4)
{
    if (!c) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (c->bl_kind < 0) return fail(c, BCT_EINVAL, "bct_baseline_init first");
    if (!(omega > 0.0) || !std::isfinite(omega)) return fail(c, BCT_EINVAL, "omega %g", omega);
    // a block whose ids form one range [lo, hi) is passed as that range (the
    // kernels then find its entries by binary search), else lo = -1
    auto id_range = [](const int64_t *ids, int64_t n, int32_t &lo, int32_t &hi) {
        lo = -1;
        hi = -1;
        if (n <= 0) return;
        const int64_t a = *std::min_element(ids, ids + n), b = *std::max_element(ids, ids + n);
        if (b - a + 1 == n && b < INT32_MAX) {   // ids are distinct
            lo = (int32_t)a;
            hi = (int32_t)(b + 1);
        }
    };
    if (c->bl_kind == BCT_ROW_ACTION) {
        for (int i = 0; i < c->m; ++i) {   // row blocks in partition order
            int32_t lo, hi;
            id_range(c->rb_rows.data() + c->rb_ptr[i], c->rb_ptr[i + 1] - c->rb_ptr[i], lo, hi);
            CK(bct::baseline_row_block(c->bm, c->d_rb_rows + c->rb_ptr[i],
                                       c->rb_ptr[i + 1] - c->rb_ptr[i], i, lo, hi, c->rb_of_row,
                                       omega, c->y, c->bl_diag, c->bl_tmp, c->bl_x, c->stream));
        }
    } else {
        for (int j = 0; j < c->n_panels; ++j) {   // volume blocks in partition order
            int32_t lo, hi;
            id_range(c->col_vox.data() + c->col_ptr[j], c->col_ptr[j + 1] - c->col_ptr[j], lo, hi);
            CK(bct::baseline_col_block(c->bm, c->bl_col_vox + c->col_ptr[j],
                                       c->col_ptr[j + 1] - c->col_ptr[j], j, lo, hi,
                                       c->bl_cb_of_vox, omega, c->bl_diag, c->bl_tmp, c->bl_x,
                                       c->bl_r, c->stream));
        }
    }
    CK(bct::baseline_norms(c->bm, c->y, c->bl_r, c->bl_x, c->has_x_true ? c->x_true : nullptr,
                           c->d_gvox, c->x_len, c->bl_kind == BCT_COLUMN_ACTION, c->bl_part,
                           c->bl_out, c->stream));
    double o[4];
    CK(cudaMemcpyAsync(o, c->bl_out, sizeof o, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (!c->has_x_true) o[2] = o[3] = NAN;
    if (norms4) memcpy(norms4, o, sizeof o);
    return 0;
}

int bct_baseline_get_x(bct_ctx *c, double *x)
{
    if (!c || !x) return BCT_EINVAL;
    DEVICE_GUARD(c);
    if (c->bl_kind < 0) return fail(c, BCT_EINVAL, "bct_baseline_init first");
    CK(cudaStreamSynchronize(c->stream));
    if (int e = d2h_staged(c, x, c->bl_x, 8 * c->n_vox)) return e;
    CK(cudaStreamSynchronize(c->stream));
    return 0;
}
