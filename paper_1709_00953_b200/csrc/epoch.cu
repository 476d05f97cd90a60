// epoch.cu -- the persistent epoch kernel and the small state kernels.
//
// One cooperative launch runs a whole epoch of the plan (executor.py:225-253):
// for every task k (a basic iteration of _run_tasks, executor.py:42-102)
//
//   phase 1  g = (A_I^J)^T r_I       warp per voxel column over the panel CSC,
//                                    segments of the task's row blocks only;
//                                    writes (g, x_J) interleaved; gg partials
//   -- grid barrier --               gg = fixed-order sum of block partials
//   phase 2  t = A_I g, ax = A_I x_J warp per local row (dual SpMV, one pass
//                                    over the forward CSR); denom partials
//   -- grid barrier --               denom, mu = beta*gg/denom, status 0/1/2
//   phase 3  xhat_J += x_J + mu g    (x_new rounded exactly like the reference)
//            z_I    = ax + mu t      written straight into the z store
//                                    (commit_task, projector.py:723-740)
//            serial_faithful: refresh of the visit's drawn rows
//            r = y - sum_j z^j in ascending j (executor.py:215-223)
//   -- grid barrier only between serial visits --
//
// then an epoch tail: parallel-mode refresh over the union of drawn rows,
// projection-sum metrics, optional _commit_epoch (solvers.py:180-185) and a
// last-block reduction of the norms.  All reductions are fixed-order, so the
// results are deterministic for a given grid size.
#include <cstdio>
#include <cuda_runtime.h>

#include "internal.h"

namespace {

#ifndef BCT_BLOCK
#define BCT_BLOCK 512
#endif
#ifndef BCT_MINB
#define BCT_MINB 2
#endif
#ifndef BCT_UNROLL
#define BCT_UNROLL 2
#endif
#ifndef BCT_P2_LANES
#define BCT_P2_LANES 8
#endif
constexpr int BLOCK = BCT_BLOCK;
constexpr int WARPS = BLOCK / 32;
constexpr int P2L = BCT_P2_LANES;          // lanes per row in phase 2
constexpr int P2R = 32 / P2L;              // rows per warp in flight
constexpr int UNR = BCT_UNROLL;
constexpr int MAX_RUNS = BCT_MAX_M / 2 + 1;

__device__ __forceinline__ void grid_sync(unsigned int *bar)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int nb = gridDim.x;
        unsigned int inc = (blockIdx.x == 0) ? (0x80000000u - (nb - 1)) : 1u;
        __threadfence();
        unsigned int old = atomicAdd(bar, inc);
        volatile unsigned int *vb = bar;
        while (((old ^ *vb) & 0x80000000u) == 0) {
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ long long gtimer()
{
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// optional per-block phase timestamps: [task][6][block] (profiling only)
#define TL_MARK(k, ph)                                                               \
    do {                                                                             \
        if (p.timeline && threadIdx.x == 0)                                          \
            p.timeline[((int64_t)(k) * 6 + (ph)) * gridDim.x + blockIdx.x] = gtimer(); \
    } while (0)

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ bool mask_has(const uint64_t *mask, int i)
{
    return (mask[i >> 6] >> (i & 63)) & 1ull;
}

// Sum of part[0..n) in a fixed order, identical in every block.
__device__ double fixed_sum(const double *part, int n, double *sh)
{
    double v = 0.0;
    for (int k = threadIdx.x; k < n; k += BLOCK) v += part[k];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) s += sh[w];
    __syncthreads();
    return s;
}

// Per-block sum of one value held by every warp's lane 0, in warp order.
__device__ double block_sum_lane0(double v, double *sh)
{
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int w = 0; w < WARPS; ++w) s += sh[w];
    }
    __syncthreads();
    return s;
}

// Per-block sum of a per-thread value, fixed order.
__device__ double block_sum_all(double v, double *sh)
{
    v = warp_sum(v);
    return block_sum_lane0(v, sh);
}

struct Runs {
    int n;
    int i0[MAX_RUNS];
    int i1[MAX_RUNS];
    int rows0[MAX_RUNS];     // first local row of the run
    int pre[MAX_RUNS + 1];   // prefix of run row counts
    int u0[MAX_RUNS];        // first row unit of the run
    int upre[MAX_RUNS + 1];  // prefix of run unit counts
};

// Contiguous runs of set bits of a row-block mask, with their local row ranges.
__device__ void build_runs(const uint64_t *mask, int m, const int32_t *rbp, const int32_t *ubp,
                           Runs &R)
{
    __syncthreads();  // R of the previous task may still be in use
    if (threadIdx.x == 0) {
        int n = 0, acc = 0, uacc = 0;
        int i = 0;
        while (i < m) {
            if (!mask_has(mask, i)) { ++i; continue; }
            int s = i;
            while (i < m && mask_has(mask, i)) ++i;
            R.i0[n] = s;
            R.i1[n] = i;
            R.rows0[n] = rbp[s];
            R.pre[n] = acc;
            acc += rbp[i] - rbp[s];
            R.u0[n] = ubp[s];
            R.upre[n] = uacc;
            uacc += ubp[i] - ubp[s];
            ++n;
        }
        R.pre[n] = acc;
        R.upre[n] = uacc;
        R.n = n;
    }
    __syncthreads();
}

__device__ __forceinline__ int run_unit(const Runs &R, int f)
{
    int k = 0;
    while (f >= R.upre[k + 1]) ++k;
    return R.u0[k] + (f - R.upre[k]);
}

__device__ __forceinline__ int run_row(const Runs &R, int f)
{
    int k = 0;
    while (f >= R.pre[k + 1]) ++k;
    return R.rows0[k] + (f - R.pre[k]);
}

template <typename V>
__device__ __forceinline__ double ldv(const V *p) { return (double)__ldg(p); }

// 4 consecutive values / indices from a 16-byte aligned position
__device__ __forceinline__ void ld4v(const float *p, double v[4])
{
    float4 a = __ldg(reinterpret_cast<const float4 *>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void ld4v(const double *p, double v[4])
{
    double2 a = __ldg(reinterpret_cast<const double2 *>(p));
    double2 b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void ld4i(const int32_t *p, int k[4])
{
    int4 a = __ldg(reinterpret_cast<const int4 *>(p));
    k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w;
}

__device__ __forceinline__ double z_value(double t, double ax, double mu, int status)
{
    return status == 0 ? fma(mu, t, ax) : ax;
}

template <typename V>
__global__ void __launch_bounds__(BLOCK, BCT_MINB) epoch_kernel(EpochParams p)
{
    __shared__ Runs R;
    __shared__ double sh[WARPS];
    __shared__ TaskDev sT;
    __shared__ PanelDev sP;

    const V *vals = static_cast<const V *>(p.vals);
    const V *tvals = static_cast<const V *>(p.tvals);
    const int lane = threadIdx.x & 31;
    const int gwarp = blockIdx.x * WARPS + (threadIdx.x >> 5);
    const int nwarps = gridDim.x * WARPS;
    const int gtid = blockIdx.x * BLOCK + threadIdx.x;
    const int nthreads = gridDim.x * BLOCK;
    const int m = p.m;
    const EpochHeader hdr = *p.hdr;
    const int n_tasks = hdr.n_tasks;
    const bool serial = hdr.mode == 0;
    const bool sharded = (hdr.flags & 4) != 0;
    double *part_gg = p.part;
    double *part_den = p.part + gridDim.x;
    double *part_m = p.part + 2 * gridDim.x;

    for (int k = 0; k < n_tasks; ++k) {
        __syncthreads();  // sT/sP/R of the previous task may still be in use
        if (threadIdx.x == 0) {
            sT = p.tasks[k];
            sP = p.panels[sT.lp];
        }
        __syncthreads();
        const TaskDev &T = sT;
        const PanelDev &P = sP;
        const int32_t *rbp = p.rbp + (int64_t)T.lp * (m + 1);
        build_runs(T.mask, m, rbp, p.ubp + (int64_t)T.lp * (m + 1), R);
        TL_MARK(k, 0);
        double2 *gx = reinterpret_cast<double2 *>(p.gx + (k & 1) * p.gx_stride);
        const double *xj = p.x + P.x_off;

        // ---- phase 1: g = A_I^T r_I over the panel CSC -------------------
        // warp per voxel column, columns taken in 4x4-tile order (corder) so
        // a CTA's warps gather overlapping r rows; 128-bit loads of 4 entries
        double wsum = 0.0;
        {
            const V *tv = tvals + P.csc_off;
            const int32_t *tr = p.trows + P.csc_off;
            const int32_t *co = p.corder + P.x_off;
            const double *rr = p.r;
            for (int q = gwarp; q < P.n_cols; q += nwarps) {
                const int c = __ldg(co + q);
                const int32_t *cp = p.cptr + P.cptr_off + (int64_t)c * (m + 1);
                double acc = 0.0;
                for (int k2 = 0; k2 < R.n; ++k2) {
                    const int s = __ldg(cp + R.i0[k2]), e = __ldg(cp + R.i1[k2]);
#pragma unroll UNR
                    for (int i = (s & ~3) + 4 * lane; i < e; i += 128) {
                        int rows[4];
                        double v[4];
                        ld4i(tr + i, rows);
                        ld4v(tv + i, v);
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (i + u >= s && i + u < e) acc = fma(v[u], rr[rows[u]], acc);
                    }
                }
                acc = warp_sum(acc);
                if (lane == 0) {
                    gx[c] = make_double2(acc, xj[c]);
                    wsum = fma(acc, acc, wsum);
                }
            }
        }
        TL_MARK(k, 1);
        double bsum = block_sum_lane0(wsum, sh);
        if (threadIdx.x == 0) part_gg[blockIdx.x] = bsum;
        grid_sync(p.bar);
        double gg = fixed_sum(part_gg, gridDim.x, sh);
        TL_MARK(k, 2);

        // ---- phase 2: dual SpMV t = A_I g, ax = A_I x_J -----------------
        // The task's rows come in units of whole rows (~512 padded entries);
        // a warp streams a unit 128 entries per step (one 4-entry vector per
        // lane, 16-byte loads; rows are 4-aligned so a vector never straddles
        // two rows).  Row boundaries come from the row-start bitmap; each step
        // does a segmented warp reduction, the row left open at lane 31 keeps
        // per-lane partials until it closes.  Fixed unit -> warp assignment
        // and fixed reduction order: deterministic.
        wsum = 0.0;
        const int n_task_rows = R.pre[R.n];
        {
            const V *fv = vals + P.fwd_off;
            const int32_t *fc = p.cols + P.fwd_off;
            const int32_t *rp = p.rptr + P.row_off + T.lp;
            const uint32_t *vb = p.vbits + P.fwd_off / 128;
            const int32_t *ur = p.urow + P.unit_off;
            const int32_t *ue = p.uend + P.unit_off;
            double2 *tax = reinterpret_cast<double2 *>(p.t_ax);
            const int n_units = R.upre[R.n];
            const unsigned le_mask = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
            for (int fu = gwarp; fu < n_units; fu += nwarps) {
                const int u = run_unit(R, fu);
                const int r0 = __ldg(ur + u), r1 = __ldg(ue + u);
                const int E0 = __ldg(rp + r0), E1 = __ldg(rp + r1);
                int open = r0 - 1;                 // row left open by the previous step
                double pt = 0.0, pax = 0.0;        // per-lane partials of the open row
                for (int b = E0 & ~127; b < E1; b += 128) {
                    const int i = b + 4 * lane;
                    double t = 0.0, ax = 0.0;
                    if (i >= E0 && i < E1) {
                        int cc[4];
                        double v[4];
                        ld4i(fc + i, cc);
                        ld4v(fv + i, v);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const double2 a = gx[cc[q]];
                            t = fma(v[q], a.x, t);
                            ax = fma(v[q], a.y, ax);
                        }
                    }
                    // bit l: vector (b/4 + l) starts a row; keep the unit's vectors
                    uint32_t word = __ldg(vb + (b >> 7));
                    const int nv = (E1 - b) >> 2;
                    if (nv < 32) word &= (1u << nv) - 1u;
                    if (b < E0) word &= ~((1u << ((E0 - b) >> 2)) - 1u);
                    if (word == 0u) {              // the whole step continues the open row
                        pt += t;
                        pax += ax;
                        continue;
                    }
                    const int rel = __popc(word & le_mask);   // 0: continues the open row
                    if (rel == 0) {
                        pt += t;
                        pax += ax;
                        t = 0.0;
                        ax = 0.0;
                    }
                    // the open row closes in this step
                    const double ot = warp_sum(pt), oax = warp_sum(pax);
                    if (lane == 0 && open >= r0) {
                        tax[open] = make_double2(ot, oax);
                        wsum = fma(ot, ot, wsum);
                    }
                    // segmented inclusive scan over lanes keyed by rel
                    const double t0 = t, ax0 = ax;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const double tt = __shfl_up_sync(0xffffffffu, t, o);
                        const double aa = __shfl_up_sync(0xffffffffu, ax, o);
                        const int rr = __shfl_up_sync(0xffffffffu, rel, o);
                        if (lane >= o && rr == rel) {
                            t += tt;
                            ax += aa;
                        }
                    }
                    const int rel31 = __popc(word);
                    // rows fully inside the step end where the next vector starts a row
                    if (rel > 0 && rel < rel31 && lane < 31 && ((word >> (lane + 1)) & 1u)) {
                        tax[open + rel] = make_double2(t, ax);
                        wsum = fma(t, t, wsum);
                    }
                    // the last segment stays open: keep its raw per-lane values
                    const bool last = rel == rel31;
                    pt = last ? t0 : 0.0;
                    pax = last ? ax0 : 0.0;
                    open += rel31;
                }
                // flush the row still open at the unit end
                const double ot = warp_sum(pt), oax = warp_sum(pax);
                if (lane == 0) {
                    tax[open] = make_double2(ot, oax);
                    wsum = fma(ot, ot, wsum);
                }
            }
        }
        TL_MARK(k, 3);
        bsum = block_sum_all(wsum, sh);
        if (threadIdx.x == 0) part_den[blockIdx.x] = bsum;
        grid_sync(p.bar);
        double denom = fixed_sum(part_den, gridDim.x, sh);
        TL_MARK(k, 4);

        // ---- phase 3: step, x accumulation, z store, serial refresh -----
        double mu = 0.0;
        int status = 0;
        if (gg == 0.0) {
            status = 1;
        } else if (denom < 1e-30) {
            status = 2;
        } else {
            mu = T.beta * gg / denom;
        }
        if (gtid == 0) {
            p.mus[k] = mu;
            p.statuses[k] = status;
            p.counts[T.lp] += 1;
        }
        {
            double *xh = p.xhat + P.x_off;
            for (int c = gtid; c < P.n_cols; c += nthreads) {
                double2 a = gx[c];
                double xn = status == 0 ? __dadd_rn(a.y, __dmul_rn(mu, a.x)) : a.y;
                xh[c] += xn;
            }
        }
        {
            const double2 *tax = reinterpret_cast<const double2 *>(p.t_ax);
            double *zj = p.z + P.row_off;
            for (int f = gtid; f < n_task_rows; f += nthreads) {
                int lr = run_row(R, f);
                double2 q = tax[lr];
                zj[lr] = z_value(q.x, q.y, mu, status);
            }
        }
        const bool last_of_visit = (T.flags & TASK_LAST_OF_VISIT) != 0;
        if (serial && last_of_visit) {
            // refresh every row of the visit's drawn blocks (executor.py:215-223)
            const double2 *tax = reinterpret_cast<const double2 *>(p.t_ax);
            const int64_t zlo = P.row_off, zhi = P.row_off + P.n_rows;
            for (int i = 0; i < m; ++i) {
                if (!mask_has(T.visit_mask, i)) continue;
                const bool cur = mask_has(T.mask, i);
                int b0 = p.rb_ptr[i], b1 = p.rb_ptr[i + 1];
                for (int q = b0 + gtid; q < b1; q += nthreads) {
                    int g = p.rb_rows[q];
                    double acc = 0.0;
                    for (int e = p.inv_ptr[g]; e < p.inv_ptr[g + 1]; ++e) {
                        int off = p.inv_z[e];
                        double v;
                        if (cur && off >= zlo && off < zhi) {
                            double2 qq = tax[off - zlo];
                            v = z_value(qq.x, qq.y, mu, status);
                        } else {
                            v = p.z[off];
                        }
                        acc += v;
                    }
                    p.r[g] = p.y[g] - acc;
                }
            }
            if (k + 1 < n_tasks) grid_sync(p.bar);
        }
        TL_MARK(k, 5);
        {
        }
    }

    // ---- epoch tail ------------------------------------------------------
    grid_sync(p.bar);
    const bool do_metrics = (hdr.flags & 2) != 0;
    const bool do_commit = (hdr.flags & 1) != 0;
    double rsq = 0.0, xsq = 0.0, esq = 0.0;
    if (!serial || do_metrics || sharded) {
        for (int g = gtid; g < p.n_meas; g += nthreads) {
            double acc = 0.0;
            for (int e = p.inv_ptr[g]; e < p.inv_ptr[g + 1]; ++e) acc += p.z[p.inv_z[e]];
            if (sharded) {
                p.exchange[g] = acc;
            } else {
                double d = p.y[g] - acc;
                int rb = p.rb_of_row[g];
                if (!serial && rb >= 0 && mask_has(hdr.epoch_mask, rb)) p.r[g] = d;
                rsq = fma(d, d, rsq);
            }
        }
    }
    for (int lp = 0; lp < p.n_panels_owned; ++lp) {
        const PanelDev P = p.panels[lp];
        const int cnt = p.counts[lp];
        double *xs = p.x + P.x_off;
        double *xh = p.xhat + P.x_off;
        const double *xt = p.x_true ? p.x_true + P.x_off : nullptr;
        for (int c = gtid; c < P.n_cols; c += nthreads) {
            double xv = xs[c];
            if (do_commit && cnt > 0) {
                xv = xh[c] / (double)cnt;
                xs[c] = xv;
                xh[c] = 0.0;
            }
            xsq = fma(xv, xv, xsq);
            if (xt) {
                double d = xt[c] - xv;
                esq = fma(d, d, esq);
            }
        }
    }
    double b0 = block_sum_all(rsq, sh);
    double b1 = block_sum_all(xsq, sh);
    double b2 = block_sum_all(esq, sh);
    __shared__ bool is_last;
    if (threadIdx.x == 0) {
        part_m[3 * blockIdx.x + 0] = b0;
        part_m[3 * blockIdx.x + 1] = b1;
        part_m[3 * blockIdx.x + 2] = b2;
        __threadfence();
        unsigned int t = atomicAdd(p.ticket, 1u);
        is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (is_last) {
        __threadfence();
        if (threadIdx.x == 0) {
            double a0 = 0.0, a1 = 0.0, a2 = 0.0;
            for (unsigned int b = 0; b < gridDim.x; ++b) {
                a0 += ((volatile double *)part_m)[3 * b + 0];
                a1 += ((volatile double *)part_m)[3 * b + 1];
                a2 += ((volatile double *)part_m)[3 * b + 2];
            }
            int ndeg = 0;
            for (int k = 0; k < n_tasks; ++k) ndeg += p.statuses[k] != 0;
            p.out->resid_sq = a0;
            p.out->x_sq = a1;
            p.out->err_sq = p.x_true ? a2 : __longlong_as_double(0x7ff8000000000000ll);
            p.out->n_degenerate = ndeg;
            if (sharded) {
                p.exchange[p.n_meas] = a1;
                p.exchange[p.n_meas + 1] = a2;
            }
            if (do_commit)
                for (int lp = 0; lp < p.n_panels_owned; ++lp) p.counts[lp] = 0;
            *p.ticket = 0;
        }
    }
}

}  // namespace

namespace bct {

std::string cuda_err(cudaError_t e) { return std::string(cudaGetErrorString(e)); }

int epoch_grid_size(int dtype, int device, int *block)
{
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (dtype == 0)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, epoch_kernel<double>, BLOCK, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, epoch_kernel<float>, BLOCK, 0);
    if (per < 1) per = 1;
    if (per > BCT_MINB) per = BCT_MINB;
    *block = BLOCK;
    return sms * per;
}

void launch_epoch(const EpochParams &p, int dtype, int grid, int block, cudaStream_t s,
                  cudaError_t *err)
{
    EpochParams local = p;
    void *args[] = {&local};
    if (dtype == 0)
        *err = cudaLaunchCooperativeKernel((const void *)epoch_kernel<double>, grid, block,
                                           args, 0, s);
    else
        *err = cudaLaunchCooperativeKernel((const void *)epoch_kernel<float>, grid, block,
                                           args, 0, s);
}

}  // namespace bct
