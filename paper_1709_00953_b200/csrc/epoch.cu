// epoch.cu -- the persistent epoch kernel.
//
// One cooperative launch (one 1024-thread CTA per SM) runs a whole epoch of
// the plan (executor.py:225-253): every task is one basic iteration of
// _run_tasks (executor.py:42-102), then the z commits, the refresh, the
// optional _commit_epoch (solvers.py:180-185) and the metric norms.  All
// reductions have a fixed order: a run is bitwise reproducible for a grid.
//
// Batched path (parallel epochs whose tasks are all full panels; the BASELINE
// configs 3-5): every phase runs over the tasks of the whole epoch at once,
// four grid barriers per epoch.
//   A  g = A_J^T r per 16x16-voxel tile: the tile's band of r staged in
//      shared memory (cp.async 16-byte granules, 8-lane groups per range;
//      FP32 copy of r in FP32 mode, double-buffered), the lane-interleaved
//      CSC streamed by 4 warps per 32-column slice in groups of 4 vector
//      rows, column partials reduced in a fixed order; (g, x) pairs + gg
//   B  per SELL slice of a super tile (its (g, x) staged, swizzled): one
//      (row, super tile) segment per lane -> (t, ax) partial, SELL order;
//      strip panels decode voxel indices from 2-bit step codes
//   C  per row: t, ax = its segments' partials in tile order; denom partials
//   D  mu, status per task; xhat += x_new per visit; z = ax + mu t
//   tail: r = y - sum_j z^j on the drawn rows (ascending j, interleaved
//      inverse map), commit, norms
// FP32 mode computes the streamed inner products in FP32: phase A's lane sums
// over an FP32 copy of r, phase B's segment partials over (g, x) staged as
// float2, and the batched path stores segment partials and row (t, ax) as
// FP32 pairs (so z = ax + mu t and the denominator use FP32-rounded t, ax).
// Every sum across lanes, warps, segments and tasks, mu, x, xhat, z, r and the
// norms are FP64.  FP64 mode is FP64 throughout.  (Measured cost against the
// FP64 reference: tests/test_parity_configs.py.)
// Per-task path (serial_faithful and partial groups): the same phase-1 and
// phase-2 code per task, three grid barriers per task, and in serial mode the
// refresh of the visit's drawn rows after its last task (executor.py:215-223).
#include <cstdio>
#include <mutex>
#include <cuda_runtime.h>
#include <type_traits>

#include "internal.h"

namespace {

// Measurement variant: FP32 values with FP64 inner
// products -- FP64 bands and (g, x) staging, FP64 lane and segment partials
// (build with -DBCT_F32_ACC64=1 and run with BCT_F32_ACC64=1 set, which gives
// FP32 contexts 8192-voxel super tiles so the double2 staging fits)
#ifndef BCT_F32_ACC64
#define BCT_F32_ACC64 0
#endif
// narrow (FP32) streamed arithmetic for value type V
template <typename V>
__host__ __device__ constexpr bool narrow_math() { return sizeof(V) == 4 && !BCT_F32_ACC64; }
// Checked build (-DBCT_CHECK=1, tools/checked_build.sh): bounds of every
// gather and scattered store of the epoch kernel, trapping on a violation
// (compute-sanitizer is not available on the GPU pool).
#ifndef BCT_CHECK
#define BCT_CHECK 0
#endif

#define BCT_ASSERT(cond)                                                              \
    do {                                                                              \
        if (BCT_CHECK && !(cond)) {                                                   \
            printf("bct check failed %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
            __trap();                                                                 \
        }                                                                             \
    } while (0)
#ifndef BCT_EXP
#define BCT_EXP 0   // profiling variants (5: no band copies, 6: no phase-1 stream, 7: no gathers)
#endif
#ifndef BCT_P1_UNROLL
#define BCT_P1_UNROLL 1
#endif
#ifndef BCT_P2_UNROLL
#define BCT_P2_UNROLL 4
#endif
#ifndef BCT_FENCED_BARRIER
#define BCT_FENCED_BARRIER 0
#endif
constexpr int P1U = BCT_P1_UNROLL;
// per-task phase 2a: a SELL slice of nvec lane-vectors is split into
// parts_of(nvec) work units (one per ~PART_VECS vectors, at most TS_MAX), so
// a CTA's longest slice is not one warp's long latency chain; the partials of
// a lane sit at spart[(slice * TS_MAX + part) * 32 + lane]
constexpr int TS_MAX = bct::TASK_PARTS_MAX;
#ifndef BCT_PART_VECS
#define BCT_PART_VECS 4
#endif
constexpr int PART_VECS = BCT_PART_VECS;
constexpr int UCAP = 256;           // slices per prefix round (shared memory)
constexpr int TS_PARTIAL = 4;       // partial tasks (a few short slices): fixed parts
__host__ __device__ __forceinline__ int parts_of(int nvec, bool full)
{
    return full ? min(TS_MAX, max(1, (nvec + PART_VECS - 1) / PART_VECS)) : TS_PARTIAL;
}
constexpr int P2U = BCT_P2_UNROLL;
constexpr int BLOCK = 1024;         // one CTA per SM
constexpr int WARPS = BLOCK / 32;

__device__ __forceinline__ long long gtimer()
{
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// optional per-block phase timestamps: [task][8][block] (profiling only)
#ifndef BCT_NO_TL_BATCH
#define BCT_NO_TL_BATCH 0
#endif
#define TL_MARK(k, ph)                                                                \
    do {                                                                              \
        if (p.timeline && threadIdx.x == 0)                                           \
            p.timeline[((int64_t)(k) * 8 + (ph)) * gridDim.x + blockIdx.x] = gtimer(); \
    } while (0)

// per-task sub-phase marks: second half of the timeline, [task][8][block]
// (p.tl_tasks = tasks the buffer holds)
#define TL_MARK2(k, ph)                                                               \
    do {                                                                              \
        if (p.timeline && threadIdx.x == 0)                                           \
            p.timeline[(((int64_t)p.tl_tasks + (k)) * 8 + (ph)) * gridDim.x + blockIdx.x] = \
                gtimer();                                                             \
    } while (0)

__device__ __forceinline__ void grid_sync(unsigned int *bar)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int nb = gridDim.x;
        unsigned int inc = (blockIdx.x == 0) ? (0x80000000u - (nb - 1)) : 1u;
#if BCT_FENCED_BARRIER
        __threadfence();
        unsigned int old = atomicAdd(bar, inc);
        volatile unsigned int *vb = bar;
        while (((old ^ *vb) & 0x80000000u) == 0) {
        }
        __threadfence();
#else
        // release-add / acquire-poll at gpu scope: the CTA's writes (ordered
        // before this thread by __syncthreads, release is cumulative) are
        // visible to every CTA that observes the flip, without full fences
        unsigned int old, cur;
        asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(bar), "r"(inc)
                     : "memory");
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];\n" : "=r"(cur) : "l"(bar) : "memory");
        } while (((old ^ cur) & 0x80000000u) == 0);
#endif
    }
    __syncthreads();
}

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

// Sums of pa[0..n) and pb[0..n) in a fixed order, identical in every block.
__device__ void fixed_sum2(const double *pa, const double *pb, int n, double *sh, double &a,
                           double &b)
{
    __shared__ double sh2[WARPS];
    double va = 0.0, vb = 0.0;
    for (int k = threadIdx.x; k < n; k += BLOCK) {
        va += pa[k];
        vb += pb[k];
    }
    va = warp_sum(va);
    vb = warp_sum(vb);
    if ((threadIdx.x & 31) == 0) {
        sh[threadIdx.x >> 5] = va;
        sh2[threadIdx.x >> 5] = vb;
    }
    __syncthreads();
    double sa = 0.0, sb = 0.0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
        sa += sh[w];
        sb += sh2[w];
    }
    __syncthreads();
    a = sa;
    b = sb;
}

// Per-block sum of a per-thread value, fixed order.
__device__ double block_sum_all(double v, double *sh)
{
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < WARPS; ++w) s += sh[w];
    __syncthreads();
    return s;
}

// Contiguous runs of set bits of a row-block mask, with their local row ranges
// and the task's units per super tile (one thread; restated on the host,
// api.cu host_prep, when the masks are known)
__device__ void build_runs(const uint64_t *mask, int m, const PanelDev &P, PrepView &R)
{
    int n = 0, acc = 0;
    int i = 0;
    while (i < m) {
        if (!mask_has(mask, i)) { ++i; continue; }
        int s = i;
        while (i < m && mask_has(mask, i)) ++i;
        R.i0[n] = s;
        R.i1[n] = i;
        R.rows0[n] = P.rbp[s];
        R.pre[n] = acc;
        acc += P.rbp[i] - P.rbp[s];
        ++n;
    }
    R.pre[n] = acc;
    R.h->n_runs = n;
    int uacc = 0;
    for (int st = 0; st < P.n_st; ++st) {
        R.st_pre[st] = uacc;
        const int32_t *sb = P.stbs + st * (m + 1);
        for (int q = 0; q < n; ++q) uacc += sb[R.i1[q]] - sb[R.i0[q]];
    }
    R.st_pre[P.n_st] = uacc;
    R.h->nst = P.n_st;
    R.h->full = (n == 1 && R.i0[0] == 0 && R.i1[0] == m);
}

__device__ void prep_task(const EpochParams &p, int k, PrepView &out)
{
    const TaskDev &T = p.tasks[k];
    const PanelDev &P = p.panels[T.lp];
    out.h->T = T;
    out.h->P = P;
    build_runs(p.masks + task_mask_off(k, p.mw), p.m, P, out);
    const uint64_t *vm = p.masks + visit_mask_off(k, p.mw);
    int nv = 0, acc = 0;
    for (int i = 0; i < p.m; ++i) {
        if (!mask_has(vm, i)) continue;
        out.vb[nv] = i;
        out.vpre[nv] = acc;
        acc += p.rb_ptr[i + 1] - p.rb_ptr[i];
        ++nv;
    }
    out.vpre[nv] = acc;
    out.h->nvb = nv;
}


__device__ __forceinline__ int run_row(const PrepView &R, int f)
{
    int k = 0;
    while (f >= R.pre[k + 1]) ++k;
    return R.rows0[k] + (f - R.pre[k]);
}

// flattened task slice f of super tile st -> slice id
__device__ __forceinline__ int task_slice(const PrepView &R, const PanelDev &P, int m, int f, int st)
{
    int off = f - R.st_pre[st];
    const int32_t *sb = P.stbs + st * (m + 1);
    for (int k = 0;; ++k) {
        int c = sb[R.i1[k]] - sb[R.i0[k]];
        if (off < c) return sb[R.i0[k]] + off;
        off -= c;
    }
}

// streamed panel data is read once per task: keep it from evicting the
// residual / gradient vectors that must stay in L2
#ifndef BCT_STREAM_HINT
#define BCT_STREAM_HINT 0        // measured: costs phase 1 ~10% on f32 panels
#endif
#ifndef BCT_B_HINT
#define BCT_B_HINT 1
#endif
#ifndef BCT_A_DEPHASE
#define BCT_A_DEPHASE 1          // phase A: CTAs' tile boundaries offset by (b % 8)/8 tile
#endif
#ifndef BCT_B_PREFETCH
#define BCT_B_PREFETCH 4         // phase B prefetches slice f+4 into L2 (0: off; 8: 0.3% slower at config 4)
#endif
#ifndef BCT_B_PF_CODES
#define BCT_B_PF_CODES 1         // the phase-B prefetch also covers the slice's step codes (0: 0.4% slower)
#endif
#ifndef BCT_B_SLICE_COST
#define BCT_B_SLICE_COST 120     // phase-B balance: entries-equivalent cost of one slice
#endif
#ifndef BCT_ROW_ORDER
#define BCT_ROW_ORDER 1          // batched phase B stores segment partials in row order (P.rq)
#endif
#ifndef BCT_A_PF_VALUES_ONLY
#define BCT_A_PF_VALUES_ONLY 0
#endif
#ifndef BCT_A_PF_LEN
#define BCT_A_PF_LEN 16          // vector rows per phase-A prefetch request set
#endif
#ifndef BCT_A_PF_SCALE
#define BCT_A_PF_SCALE 1         // phase-A prefetch distance / length scaled to the rows per iteration
                                 // (config 5, 16 warps per slice: 16.25 -> 15.70 ms; config 4 unchanged)
#endif
#ifndef BCT_A_PREFETCH
#define BCT_A_PREFETCH 8         // phase A prefetches its slice 8 vector rows ahead into L2 (0: off)
#endif
#ifndef BCT_P1_G
#define BCT_P1_G 4               // phase-A FP32 loop: vector rows per load group
#endif
#ifndef BCT_FC_TAIL_GROUP
#define BCT_FC_TAIL_GROUP 0      // 1: phase-B coded tail (< BCT_FC_G vectors) as one predicated group
#endif
#ifndef BCT_FC_G
#define BCT_FC_G 8               // phase-B coded loop: vectors per load group (4 or 8)
#endif
#ifndef BCT_NO_FCODE_K
#define BCT_NO_FCODE_K 0         // 1: phase B ignores the step codes (profiling)
#endif
#ifndef BCT_REFRESH_RF
#define BCT_REFRESH_RF 4         // per-task serial refresh: z slots of a row loaded in groups of 4 (1: 2% slower, 8: 0.1%)
#endif
#ifndef BCT_B_ROT
#define BCT_B_ROT 1              // batched phase B: a share's last (partial) row-block group visited first
#endif
#ifndef BCT_REFRESH_ALL
#define BCT_REFRESH_ALL 1        // per-task serial refresh of every row: interleaved inverse map
#endif
#ifndef BCT_TAIL_U
#define BCT_TAIL_U 6             // epoch tail: z slots of a measurement loaded in predicated groups of 6 (4, 8: slower; 12 spills)
#endif
#ifndef BCT_STREAM_HINT_F64
#define BCT_STREAM_HINT_F64 1    // f64 values (serial configs): the hint helps
#endif
__device__ __forceinline__ uint64_t evict_first_policy()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ float4 ld_stream(const float4 *p)
{
#if BCT_STREAM_HINT
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(evict_first_policy()));
    return v;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ double2 ld_stream(const double2 *p)
{
#if BCT_STREAM_HINT || BCT_STREAM_HINT_F64
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(evict_first_policy()));
    return v;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ uint4 ld_stream(const uint4 *p)
{
#if BCT_STREAM_HINT
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(evict_first_policy()));
    return v;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ uint2 ld_stream(const uint2 *p)
{
#if BCT_STREAM_HINT
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(evict_first_policy()));
    return v;
#else
    return __ldg(p);
#endif
}

__device__ __forceinline__ void ld8v(const float *p, double v[8])
{
    float4 a = ld_stream(reinterpret_cast<const float4 *>(p));
    float4 b = ld_stream(reinterpret_cast<const float4 *>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void ld8v(const double *p, double v[8])
{
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        double2 a = ld_stream(reinterpret_cast<const double2 *>(p) + q);
        v[2 * q] = a.x;
        v[2 * q + 1] = a.y;
    }
}
__device__ __forceinline__ void ld8u16(const uint16_t *p, int k[8])
{
    uint4 a = ld_stream(reinterpret_cast<const uint4 *>(p));
    k[0] = a.x & 0xffff; k[1] = a.x >> 16; k[2] = a.y & 0xffff; k[3] = a.y >> 16;
    k[4] = a.z & 0xffff; k[5] = a.z >> 16; k[6] = a.w & 0xffff; k[7] = a.w >> 16;
}
// phase-2 streams (SELL values / indices): L2 evict-first measured a small
// gain here (it costs phase 1, whose loads use the plain path)
__device__ __forceinline__ void ld4v(const float *p, double v[4])
{
#if BCT_B_HINT == 2
    float4 a;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(p), "l"(evict_first_policy()));
#elif BCT_B_HINT
    float4 a;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(p), "l"(evict_first_policy()));
#else
    float4 a = ld_stream(reinterpret_cast<const float4 *>(p));
#endif
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void ld4v(const double *p, double v[4])
{
    double2 a = ld_stream(reinterpret_cast<const double2 *>(p));
    double2 b = ld_stream(reinterpret_cast<const double2 *>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void ld4u16(const uint16_t *p, int k[4])
{
#if BCT_B_HINT == 2
    uint2 a;
    asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(a.x), "=r"(a.y) : "l"(p), "l"(evict_first_policy()));
#elif BCT_B_HINT
    uint2 a;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(a.x), "=r"(a.y) : "l"(p), "l"(evict_first_policy()));
#else
    uint2 a = ld_stream(reinterpret_cast<const uint2 *>(p));
#endif
    k[0] = a.x & 0xffff; k[1] = a.x >> 16; k[2] = a.y & 0xffff; k[3] = a.y >> 16;
}

// Ordered stream load (asm volatile keeps it ahead of the gathers that follow)
__device__ __forceinline__ float4 ldv4_ordered(const float *p)
{
    float4 a;
    asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(p));
    return a;
}
__device__ __forceinline__ uint2 ldu2_ordered(const void *p)
{
    uint2 a;
    asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(a.x), "=r"(a.y) : "l"(p));
    return a;
}
// Band gather through a 32-bit shared-window address (the band pointer is a
// generic pointer by the time it reaches tile_g: without this the compiler
// emits generic 64-bit loads)
__device__ __forceinline__ float lds_f32(uint32_t a)
{
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ double lds_f64(uint32_t a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
// element idx of a shared band of TB (32-bit shared-window base address)
template <typename TB>
__device__ __forceinline__ double lds_band(uint32_t base, int idx)
{
    if constexpr (sizeof(TB) == 8) return lds_f64(base + 8u * (uint32_t)idx);
    else return (double)lds_f32(base + 4u * (uint32_t)idx);
}

// L2 prefetch of a byte range (one bulk request; 16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint32_t ld_code(const uint32_t *p)
{
#if BCT_B_HINT
    uint32_t a;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(a) : "l"(p), "l"(evict_first_policy()));
    return a;
#else
    return __ldg(p);
#endif
}

// One SELL lane's (t, ax) partial over a step-coded segment (layout.cu
// fcode_k): the voxel index of every entry is the previous one moved by
// code 0 / 1 / 2 / 3 -> 0 / s / w / w + s.  All value loads of a 4-vector
// group are issued before the gathers (memory-level parallelism).
__device__ __forceinline__ void coded_decode4(uint32_t byte, int &q, int sy, int wst, int shift,
                                              int cc[4])
{
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int code = (byte >> (2 * e)) & 3;
        q += ((code & 1) ? sy : 0) + (code >> 1) * wst;
        cc[e] = swz_idx(q, shift);
    }
}

// Raw 4-vector of stored values (no conversion): FP32 products in FP32 mode.
__device__ __forceinline__ void ld4raw(const float *p, float v[4])
{
#if BCT_B_HINT
    float4 a;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(p), "l"(evict_first_policy()));
#else
    const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
#endif
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void ld4raw(const double *p, double v[4]) { ld4v(p, v); }

// FP32 mode accumulates a lane's segment in FP32 (north_star: FP32 mode
// matches the reference's residual curve to 1e-4); rows sum the segment
// partials in FP64 (phase C).  FP64 mode is FP64 throughout.
template <typename V, typename GS>
__device__ __forceinline__ double2 coded_segment(const PanelDev &P, const V *fv, int sl, int base,
                                                 int nvec, int lane, int wst, const GS *gs,
                                                 int hdr)
{
    using A = typename std::conditional<narrow_math<V>(), float, double>::type;
    const int sy = (hdr >> 16) & 1 ? -1 : 1;
    const int shift = P.swz_shift;
    int q = hdr & 0xffff;
    const uint32_t *cw = P.fcode + (base >> 4) + 24 * sl + lane;
    A t = A(0), ax = A(0);
    // groups of FG vectors (FG/4 code words): all value loads of a group are
    // issued before its gathers; indices are decoded just in time
    constexpr int FG = BCT_FC_G;
    int kv4 = 0;
    for (; kv4 + FG <= nvec; kv4 += FG) {
        uint32_t word[FG / 4];
#pragma unroll
        for (int w = 0; w < FG / 4; ++w) word[w] = ld_code(cw + ((kv4 >> 2) + w) * 32);
        V v[FG][4];
#pragma unroll
        for (int j = 0; j < FG; ++j) ld4raw(fv + base + (((kv4 + j) * 32 + lane) << 2), v[j]);
#pragma unroll
        for (int j = 0; j < FG; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int code = (word[j >> 2] >> (8 * (j & 3) + 2 * e)) & 3;
                q += ((code & 1) ? sy : 0) + (code >> 1) * wst;
                BCT_ASSERT(q >= 0 && swz_idx(q, shift) < P.st_max);
                const GS a = gs[swz_idx(q, shift)];
                t = fma((A)v[j][e], (A)a.x, t);
                ax = fma((A)v[j][e], (A)a.y, ax);
            }
    }
#if BCT_FC_TAIL_GROUP
    // the last < FG vectors as one predicated group: every load issued
    // before the first gather (one vector at a time exposed the load
    // latency per vector)
    if (kv4 < nvec) {
        const int nr = nvec - kv4;
        uint32_t word[FG / 4];
#pragma unroll
        for (int w = 0; w < FG / 4; ++w)
            word[w] = 4 * w < nr ? ld_code(cw + ((kv4 >> 2) + w) * 32) : 0u;
        V v[FG][4];
#pragma unroll
        for (int j = 0; j < FG; ++j) {
            if (j < nr) {
                ld4raw(fv + base + (((kv4 + j) * 32 + lane) << 2), v[j]);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) v[j][e] = V(0);
            }
        }
#pragma unroll
        for (int j = 0; j < FG; ++j) {
            if (j >= nr) break;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int code = (word[j >> 2] >> (8 * (j & 3) + 2 * e)) & 3;
                q += ((code & 1) ? sy : 0) + (code >> 1) * wst;
                BCT_ASSERT(q >= 0 && swz_idx(q, shift) < P.st_max);
                const GS a = gs[swz_idx(q, shift)];
                t = fma((A)v[j][e], (A)a.x, t);
                ax = fma((A)v[j][e], (A)a.y, ax);
            }
        }
    }
#else
    for (int j = 0; kv4 + j < nvec; ++j) {
        const int kv = kv4 + j;
        const uint32_t word = ld_code(cw + (kv >> 2) * 32);
        V v[4];
        int cc[4];
        ld4raw(fv + base + ((kv * 32 + lane) << 2), v);
        coded_decode4(word >> (8 * (kv & 3)), q, sy, wst, shift, cc);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const GS a = gs[cc[e]];
            t = fma((A)v[e], (A)a.x, t);
            ax = fma((A)v[e], (A)a.y, ax);
        }
    }
#endif
    return make_double2((double)t, (double)ax);
}

__device__ __forceinline__ uint32_t smem_addr(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp_async8(void *sdst, const void *gsrc)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_addr(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async16(void *sdst, const void *gsrc)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(sdst)), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n"); }

// Band staging of one tile (whole CTA).  Range k of the tile is an
// even-aligned span of the residual (layout.cu ranges_k).  Lanes hold the
// metadata of 32 consecutive ranges; each 8-lane group then copies one range
// in 16-byte granules (cp.async), so one instruction moves four whole ranges
// (a handful of cache lines) instead of 32 scattered ones.  (One bulk copy
// per ~100-byte range is TMA request-rate bound: ~35 cycles per request.)
// A partial task (mask != nullptr) writes zeros for the ranges of row blocks
// outside its mask, so phase 1 may stream whole vectors of the tile.
struct BandMeta {
    int2 m[2];
    int keep[2];
    int k0, k1;
};

__device__ __forceinline__ void band_meta_load(const PanelDev &P, int t, BandMeta &bm,
                                               const uint64_t *mask)
{
    const int k0 = __ldg(P.band_ptr + t), k1 = __ldg(P.band_ptr + t + 1);
    bm.k0 = k0;
    bm.k1 = k1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int it = 0; it < 2; ++it) {
        const int q = k0 + warp * 32 + lane + it * BLOCK;
        bm.m[it] = q < k1 ? __ldg(P.band_meta + q) : make_int2(0, 0);
        bm.keep[it] = (mask == nullptr || q >= k1) ? 1 : (int)mask_has(mask, __ldg(P.band_rb + q));
    }
}

// Caller guarantees every read of buf is ordered before this call by a CTA
// barrier; completion: cp.async.wait_group 0 + a CTA barrier.
// GL: lanes per range (8: ranges of 5-8 granules, the 16x16 tiles; 4: the
// short ranges of 8x8 / 4x8 tiles, eight ranges per instruction)
template <typename TB, int GL = 8>
__device__ __forceinline__ void band_issue(const PanelDev &P, const BandMeta &bm, const TB *r,
                                           TB *buf, const uint64_t *mask)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NG = 32 / GL;   // ranges per instruction
    const int sub = lane / GL, sl = lane % GL;
#pragma unroll
    for (int it = 0; it < 2; ++it) {
        const int q0 = bm.k0 + warp * 32 + it * BLOCK;
        if (q0 >= bm.k1) continue;   // warp-uniform
#pragma unroll 2
        for (int jj = 0; jj < GL; ++jj) {
            const int src = jj * NG + sub;
            const int g0 = __shfl_sync(0xffffffffu, bm.m[it].x, src);
            const int pk = __shfl_sync(0xffffffffu, bm.m[it].y, src);
            const int keep = __shfl_sync(0xffffffffu, bm.keep[it], src);
            if (q0 + src < bm.k1 && BCT_EXP != 5) {
                const int pre = (int)((unsigned)pk >> 16), len = pk & 0xffff;
                // 16-byte granules of GE elements from the aligned range start
                constexpr int GE = 16 / sizeof(TB);
                constexpr int AM = bct::BAND_ALIGN - 1;
                const int ng = ((g0 & AM) + len + GE - 1) / GE;
                const TB *rs = r + (g0 & ~AM);
                TB *dst = buf + pre;
                if (keep) {
                    for (int e = sl; e < ng; e += GL) cp_async16(dst + GE * e, rs + GE * e);
                } else {
                    for (int e = sl; e < ng; e += GL)
#pragma unroll
                        for (int u = 0; u < GE; ++u) dst[GE * e + u] = TB(0);
                }
            }
        }
    }
    // ranges beyond 2*BLOCK per tile (not expected): plain loads
    for (int q = bm.k0 + 2 * BLOCK + threadIdx.x; q < bm.k1; q += BLOCK) {
        const int2 mm = __ldg(P.band_meta + q);
        const int pre = (int)((unsigned)mm.y >> 16), len = mm.y & 0xffff;
        const bool keep = mask == nullptr || mask_has(mask, __ldg(P.band_rb + q));
        const int off = mm.x & (bct::BAND_ALIGN - 1);
        for (int e = 0; e < len; ++e) buf[pre + off + e] = keep ? r[mm.x + e] : TB(0);
    }
    cp_async_commit();
}

// batched phase A: four lanes per range on the small tiles (short ranges)
#ifndef BCT_BAND_GL_SMALL
#define BCT_BAND_GL_SMALL 4      // config 5 (8x8): 15.85 -> 15.32 ms per epoch against 8
#endif
#ifndef BCT_BAND_GL_BIG
#define BCT_BAND_GL_BIG 8
#endif
template <typename TB>
__device__ __forceinline__ void band_issue_gl(const PanelDev &P, const BandMeta &bm, const TB *r,
                                              TB *buf)
{
    if (sizeof(TB) == 4 && P.tile_cols <= 64) band_issue<TB, BCT_BAND_GL_SMALL>(P, bm, r, buf, nullptr);
    else band_issue<TB, BCT_BAND_GL_BIG>(P, bm, r, buf, nullptr);
}

// Phase-1 work of one tile: g of its columns in slices [sl0, sl1) of the tile.
// Each 32-column slice is stored lane-interleaved (lane = column, 8 entries
// per 16/32-byte lane vector), so a warp-wide vector row is one coalesced
// 2 KB (FP64) / 1 KB (FP32) access.  The slices of the tile are split over
// the warps (WARPS/ns warps per slice, vector rows interleaved among them);
// per-warp column partials meet in `red` and thread c sums column c's
// partials in a fixed order.  vr (partial tasks): per slice, the vector rows
// that can hold rows of the task (rows outside the mask read zeros).
// Returns this thread's share of gg (threads < 32*ns, one column each).
constexpr int RED_DOUBLES = WARPS * 32;         // partials: (WARPS/ns) x (32*ns)
static_assert(2 * RED_DOUBLES * 8 == bct::PHASE1_RED_BYTES, "reduction areas");

template <typename V, typename TB = double>
__device__ __forceinline__ double tile_g(const PanelDev &P, int t, int sl0, int sl1,
                                         const TB *bt, const double *xj, double2 *gx,
                                         double *red, const int2 *vr)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const V *tv = static_cast<const V *>(P.tvals);
    const int nsl_tile = P.tile_cols >> 5;
    const int sb = t * nsl_tile + sl0;
    // slices of this item (0 when a column part lies past the panel's last slice)
    const int ns = max(0, min(sb + (sl1 - sl0), P.n_cslices) - sb);
    const int wps = WARPS / max(ns, 1);
    const int si = warp / wps, sub = warp - si * wps;
    // the column this thread reduces: prefetch its id and x_J entry
    const int c = threadIdx.x;
    const int qc = sb * 32 + c;
    const bool owner = c < ns * 32 && qc < P.n_cols;
    int d = 0;
    double xv = 0.0;
    if (owner) {
        d = __ldg(P.corder + qc);
        xv = xj[d];
    }
    if (si < ns) {
        const int base = __ldg(P.csl_start + sb + si);
        int lo = 0, hi = (__ldg(P.csl_start + sb + si + 1) - base) >> 8;
        if (vr != nullptr) {
            lo = vr[si].x;
            hi = vr[si].y;
        }
        if (BCT_EXP == 6) hi = lo;   // profiling: staging and structure only
        double acc = 0.0;
        const uint8_t *toff = P.toff;
        if (sizeof(TB) == 4 && sizeof(V) == 4) {
            // FP32 mode, batched path: FP32 products and lane partial sums
            // (north_star: FP32 mode matches the reference curve to 1e-4);
            // the partials meet in FP64 below
            float acc32 = 0.f;
            const uint16_t *tbase = P.tbase;
            const uint16_t *tloc = P.tloc;
            if (toff != nullptr) {
                // groups of R vector rows: every stream load of the group is
                // issued before its gathers
                constexpr int R = BCT_P1_G;
                const uint32_t bts = (uint32_t)__cvta_generic_to_shared(bt);
                int u = lo + sub;
#pragma unroll 1
                for (; u < hi; u += R * wps) {
#if BCT_A_PREFETCH
                    // the slice's vector rows BCT_A_PREFETCH ahead (one group's
                    // worth) into L2: bulk requests hold bytes in flight
                    // without registers
                    // (BCT_A_PF_LEN: a multiple of the R * wps rows one
                    // iteration consumes; longer requests every few iterations)
                    // (tiles of one or two slices: R * wps > BCT_A_PF_LEN rows per
                    // iteration, so the request covers the next iteration's rows)
                    const int pf_len = BCT_A_PF_SCALE ? max(BCT_A_PF_LEN, R * wps) : BCT_A_PF_LEN;
                    const int pf_ahead = BCT_A_PF_SCALE ? max(BCT_A_PREFETCH, R * wps / 2) : BCT_A_PREFETCH;
                    if (sub == 0 && lane == 0 &&
                        ((u - lo) / (R * wps)) % max(1, BCT_A_PF_LEN / (R * wps)) == 0) {
                        const int v0 = u + pf_ahead;
                        const int v1 = min(hi, v0 + pf_len);
                        if (v0 < v1) {
                            const int64_t e0 = base + (int64_t)v0 * 256, n = (int64_t)(v1 - v0) * 256;
                            prefetch_l2(reinterpret_cast<const float *>(tv) + e0, (uint32_t)(4 * n));
#if !BCT_A_PF_VALUES_ONLY
                            prefetch_l2(toff + e0, (uint32_t)n);
                            prefetch_l2(tbase + (e0 >> 3), (uint32_t)(n >> 2));
#endif
                        }
                    }
#endif
                    float4 a[R][2];
                    uint2 o[R];
                    int b0[R];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const bool ok = u + r * wps < hi;
                        const int i = base + (u + r * wps) * 256 + lane * 8;
                        if (ok) {
                            a[r][0] = ldv4_ordered(reinterpret_cast<const float *>(tv) + i);
                            a[r][1] = ldv4_ordered(reinterpret_cast<const float *>(tv) + i + 4);
                            o[r] = ldu2_ordered(toff + i);
                            b0[r] = __ldg(tbase + (i >> 3));
                        } else {
                            a[r][0] = a[r][1] = make_float4(0.f, 0.f, 0.f, 0.f);
                            o[r] = make_uint2(0u, 0u);
                            b0[r] = 0;
                        }
                    }
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const float vf[8] = {a[r][0].x, a[r][0].y, a[r][0].z, a[r][0].w,
                                             a[r][1].x, a[r][1].y, a[r][1].z, a[r][1].w};
                        const uint32_t bb = bts + 4u * (uint32_t)b0[r];
                        BCT_ASSERT(b0[r] >= 0 &&
                                   b0[r] + (int)max(max(max(o[r].x & 0xff, (o[r].x >> 8) & 0xff),
                                                        max((o[r].x >> 16) & 0xff, o[r].x >> 24)),
                                                    max(max(o[r].y & 0xff, (o[r].y >> 8) & 0xff),
                                                        max((o[r].y >> 16) & 0xff, o[r].y >> 24))) <
                                   ((P.band_max + 3) & ~3));
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            acc32 = fmaf(vf[e], lds_f32(bb + 4u * ((o[r].x >> (8 * e)) & 0xff)), acc32);
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            acc32 = fmaf(vf[4 + e], lds_f32(bb + 4u * ((o[r].y >> (8 * e)) & 0xff)), acc32);
                    }
                }
            } else {
#pragma unroll 1
                for (int u = lo + sub; u < hi; u += wps) {
                    const int i = base + u * 256 + lane * 8;
                    const float4 a0 = ld_stream(reinterpret_cast<const float4 *>(tv + i));
                    const float4 a1 = ld_stream(reinterpret_cast<const float4 *>(tv + i) + 1);
                    const float vf[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    int loc[8];
                    ld8u16(tloc + i, loc);
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc32 = fmaf(vf[e], (float)bt[loc[e]], acc32);
                }
            }
            acc = acc32;
        } else if (toff != nullptr) {   // delta form: 8-bit offsets on a 16-bit base
            const uint16_t *tbase = P.tbase;
            const uint32_t bts = (uint32_t)__cvta_generic_to_shared(bt);
#pragma unroll P1U
            for (int u = lo + sub; u < hi; u += wps) {
                const int i = base + u * 256 + lane * 8;
                const uint2 o = ld_stream(reinterpret_cast<const uint2 *>(toff + i));
                const int b0 = __ldg(tbase + (i >> 3));
                double v[8];
                ld8v(tv + i, v);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    BCT_ASSERT(b0 + ((o.x >> (8 * e)) & 0xff) < ((P.band_max + 3) & ~3));
                    acc = fma(v[e], lds_band<TB>(bts, b0 + ((o.x >> (8 * e)) & 0xff)), acc);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    acc = fma(v[4 + e], lds_band<TB>(bts, b0 + ((o.y >> (8 * e)) & 0xff)), acc);
            }
        } else {
            const uint16_t *tloc = P.tloc;
            const uint32_t bts = (uint32_t)__cvta_generic_to_shared(bt);
#pragma unroll P1U
            for (int u = lo + sub; u < hi; u += wps) {
                const int i = base + u * 256 + lane * 8;
                int loc[8];
                double v[8];
                ld8u16(tloc + i, loc);
                ld8v(tv + i, v);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    BCT_ASSERT(loc[e] < ((P.band_max + 3) & ~3));
                    acc = fma(v[e], BCT_EXP == 7 ? (double)loc[e] : lds_band<TB>(bts, loc[e]), acc);
                }
            }
        }
        red[sub * (ns * 32) + si * 32 + lane] = acc;
    }
    cp_async_wait_all();   // (batched path: ring copies / next band of this thread)
    __syncthreads();
    double wsum = 0.0;
    if (owner) {
        double g = 0.0;
        for (int k = 0; k < wps; ++k) g += red[k * (ns * 32) + c];
        gx[d] = make_double2(g, xv);
        wsum = g * g;
    }
    return wsum;
}

// vr of a partial task (see tile_g): warp si < ns computes slice si's range
// over the columns' entries of row blocks [i_first, i_last)
__device__ __forceinline__ void tile_vr(const PanelDev &P, int m, int t, int sl0, int sl1,
                                        int i_first, int i_last, int2 *vr)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sb = t * (P.tile_cols >> 5) + sl0;
    const int ns = min(sb + (sl1 - sl0), P.n_cslices) - sb;
    if (warp < ns) {
        const int q = (sb + warp) * 32 + lane;
        int lo = 1 << 30, hi = 0;
        if (q < P.n_cols) {
            const int32_t *cp = P.cptr + (int64_t)__ldg(P.corder + q) * (m + 1);
            const int s = __ldg(cp + i_first), e = __ldg(cp + i_last);
            if (e > s) {
                lo = s >> 3;
                hi = (e + 7) >> 3;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) vr[warp] = hi > lo ? make_int2(lo, hi) : make_int2(0, 0);
    }
}

// A super tile's (g, x) pairs into shared memory, swizzled (swz_idx), as
// GS (float2 in FP32 mode): each thread issues its loads of a round before
// its stores (a load-store chain per element costs one L2 round trip each).
// L2-coherent loads: the pairs were written earlier in this launch.
template <typename GS>
__device__ __forceinline__ void stage_gx(GS *gs, const double2 *src, int n, int shift)
{
    constexpr int U = 4;
    for (int q0 = threadIdx.x; q0 < n; q0 += U * BLOCK) {
        double2 a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int q = q0 + u * BLOCK;
            a[u] = q < n ? __ldcg(src + q) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int q = q0 + u * BLOCK;
            if (q < n) gs[swz_idx(q, shift)] = GS{(decltype(GS::x))a[u].x, (decltype(GS::x))a[u].y};
        }
    }
}

__device__ __forceinline__ double z_value(double t, double ax, double mu, int status)
{
    return status == 0 ? fma(mu, t, ax) : ax;
}


// ======================================================================
// Epoch-batched path (parallel mode, every task a full panel): all tasks
// read the epoch-start residual and image, so each phase runs over the
// tasks of the whole epoch at once -- one continuous, pipelined stream per
// phase and four grid barriers per epoch instead of three per task.
// ======================================================================

// First i in [0, n] with key <= at(i) (at ascending; at(n) = +inf), found by one
// full warp with 32-way probes: a few dependent loads instead of log2(n).
template <typename At, typename K>
__device__ __forceinline__ int lower_bound_warp(At at, int n, K key)
{
    const int lane = threadIdx.x & 31;
    int lo = 0, hi = n;
    for (;;) {
        const int span = hi - lo;
        const int step = span > 32 ? (span + 31) / 32 : 1;
        const int idx = lo + lane * step;
        const bool ge = idx >= hi || !(at(idx) < key);
        const unsigned m = __ballot_sync(0xffffffffu, ge);
        if (span <= 32) return m ? min(lo + __ffs(m) - 1, hi) : hi;
        if (m == 0) {                        // every probe < key: past the last probe
            lo += 31 * step + 1;
            continue;
        }
        const int f = __ffs(m) - 1;
        if (f == 0) return lo;
        const int nlo = lo + (f - 1) * step + 1;
        hi = min(hi, lo + f * step);
        lo = nlo;
    }
}

__device__ __forceinline__ int task_of(const TaskDev *tasks, int n_tasks, int which, int f)
{
    // last task whose prefix (field `which`) is <= f
    int lo = 0, hi = n_tasks - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) / 2;
        const TaskDev &T = tasks[mid];
        const int v = which == 0 ? T.tile_pre : which == 1 ? T.slice_pre : which == 2 ? T.row_pre
                                                                               : T.vox_pre;
        if (v <= f) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Batched phase-A ring: panel + item of the next tiles, copied by warp 0
// with cp.async (4 slots: a slot is rewritten two tiles after its last read)
struct RingSlot {
    PanelDev P;
    int64_t gx_off;
    int k, t;
    int q0, q1, qd;     // slices [nsl*q0/qd, nsl*q1/qd) of the tile (0, 1, 1: whole tile)
};
#ifndef BCT_A_META_EARLY
#define BCT_A_META_EARLY 0       // batched phase A: tile it+2's band metadata loaded before tile it's
                                 // streams (ring one slot deeper) instead of after them
#endif
constexpr int RING = BCT_A_META_EARLY ? 5 : 4;
static_assert(sizeof(RingSlot) % 8 == 0, "ring slots are copied in 8-byte words");

// fused batched tail (EpochHeader::fuse_tail): tables in the phase buffers
// after the per-task mu / status, per owned panel lp: z and x offsets (one
// past the last panel: z_len, x_len), its task this epoch (-1: none), the
// offset of that task's (g, x) pairs relative to x, and the form of its z:
// st >= 0: z = ax + mu t from the persistent (t, ax) pairs (EpochParams::zt)
// with this mu / status, st = -1: the stored z
struct FuseTables {
    double *mu_t;   // per task (phase D's mu)
    int *st_t;
    int64_t *xoff, *gxo;
    double *mu;
    int32_t *roff, *task, *st;
};

__device__ __forceinline__ FuseTables fuse_tables(double *rs, int n_tasks, int np)
{
    FuseTables t;
    t.mu_t = rs;
    t.st_t = reinterpret_cast<int *>(rs + n_tasks);
    int64_t *q = reinterpret_cast<int64_t *>(rs + n_tasks + (n_tasks + 1) / 2);
    t.xoff = q;
    t.gxo = q + np + 1;
    t.mu = reinterpret_cast<double *>(q + 2 * np + 1);
    int32_t *w = reinterpret_cast<int32_t *>(t.mu + np);
    t.roff = w;
    t.task = w + np + 1;
    t.st = w + 2 * np + 1;
    return t;
}

template <typename V>
__device__ void batched_epoch(const EpochParams &p, const EpochHeader &hdr, double *rs, double *sh,
                              RingSlot *ring, int *s_tpre, int *s_lp)
{
    __shared__ long long s_range_dbg[3];
    __shared__ long long s_stage_dbg;
    if (!BCT_NO_TL_BATCH) TL_MARK(0, 0);
    if (p.timeline && threadIdx.x == 0 && hdr.n_tasks > 3) {   // profiling: the block's SM
        unsigned int smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.timeline[((int64_t)3 * 8 + 0) * gridDim.x + blockIdx.x] = smid;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = gridDim.x, b = blockIdx.x;
    const int n_tasks = hdr.n_tasks;
    const int m = p.m;
    double2 *gxb = reinterpret_cast<double2 *>(p.gx_batch);
    // segment partials and row (t, ax) pairs: FP32 in FP32 mode (the lane
    // partials are FP32 sums already), FP64 in FP64 mode
    using PT = typename std::conditional<narrow_math<V>(), float2, double2>::type;
    PT *segb = reinterpret_cast<PT *>(p.seg_batch);
    PT *taxb = reinterpret_cast<PT *>(p.tax_batch);
    double *pgg = p.part_task;                       // [k][G][WARPS]
    double *pden = p.part_task + (int64_t)n_tasks * G * WARPS;   // [k][G]
    double *ggs = p.part_task + (int64_t)n_tasks * G * (WARPS + 1);   // [k] reduced gg

    // ---- phase A: g = A^T r for every task, tiles round-robin over CTAs ----
    // One CTA barrier per tile: the band of tile it+1 streams in (bulk
    // copies, mbarrier) while tile it is computed; the reduction area is
    // double-buffered by tile parity.  gg partials per (task, CTA, warp).
    // FP32 mode: the bands are staged from an FP32 copy of the epoch-start r
    // (half the staging bytes and single-wavefront gathers)
    using TB = typename std::conditional<narrow_math<V>(), float, double>::type;
    const TB *rband;
    if constexpr (narrow_math<V>()) {
        if (!hdr.r32_valid) {   // r was written outside an epoch since the last copy
            for (int64_t i = (int64_t)b * BLOCK + threadIdx.x; i < p.n_meas; i += (int64_t)G * BLOCK)
                p.r32[i] = (float)p.r[i];
            grid_sync(p.bar);
        }
        rband = p.r32;
    } else {
        rband = p.r;
    }
    for (int k = threadIdx.x; k < n_tasks; k += BLOCK) {
        s_tpre[k] = p.tasks[k].tile_pre;
        s_lp[k] = p.tasks[k].lp;
    }
    if (threadIdx.x == 0) s_tpre[n_tasks] = hdr.n_tiles_total;
    for (int q = threadIdx.x; q < n_tasks * WARPS; q += BLOCK)
        pgg[((int64_t)(q / WARPS) * G + b) * WARPS + q % WARPS] = 0.0;
    __syncthreads();
    {
        // whole tiles in rounds of G; the tiles of the last partial round are
        // cut into up to 8 slice parts so every CTA gets the same share.
        // The CTAs' tile boundaries are de-phased: CTA b starts with the last
        // (8 - f)/8 of its first tile (f = b % 8) and does its first f/8 after
        // its other whole tiles.  In lock step every CTA waits for its next
        // band and restarts its streams at the same moment, leaving HBM idle
        // at each tile start (measured: the first tiles of an epoch ran
        // 36 -> 28 us until the CTAs drifted apart).
        const int bb = b;
        const int full = hdr.n_tiles_total / G, rem = hdr.n_tiles_total - full * G;
        const int nsplit = rem > 0 ? max(1, min(8, G / rem)) : 1;
        const int fph = BCT_A_DEPHASE ? bb % 8 : 0;
        const bool wrap = full >= 2 && fph > 0;
        const int n_whole = full + (wrap ? 1 : 0);   // items before the remainder part
        const int n_items = n_whole + (bb < rem * nsplit ? 1 : 0);
        // FP32 bands: two buffers fit in one FP64 band's space
        const bool dbuf = sizeof(TB) == 4 || p.band_dbuf != 0;
        TB *buf[2] = {reinterpret_cast<TB *>(rs), reinterpret_cast<TB *>(rs) + (dbuf ? p.band_cap : 0)};
        double *red = rs + (int64_t)p.band_cap * (sizeof(TB) == 4 ? 1 : (dbuf ? 2 : 1));
        auto ring_issue = [&](int it) {   // warp 0
            int item, q0 = 0, q1 = 1, qd = 1;
            if (it >= n_whole) {   // the remainder tile's part
                item = full * G + bb / nsplit;
                q0 = bb % nsplit;
                q1 = q0 + 1;
                qd = nsplit;
            } else if (wrap && it == 0) {   // the first tile's last (8 - fph)/8
                item = bb;
                q0 = fph;
                q1 = qd = 8;
            } else if (wrap && it == full) {   // ... and its first fph/8
                item = bb;
                q1 = fph;
                qd = 8;
            } else {
                item = bb + it * G;
            }
            int lo = 0, hi = n_tasks - 1;  // last task with tile_pre <= item
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_tpre[mid] <= item) lo = mid; else hi = mid - 1;
            }
            RingSlot &S = ring[it % RING];
            const uint64_t *src = reinterpret_cast<const uint64_t *>(p.panels + s_lp[lo]);
            uint64_t *dst = reinterpret_cast<uint64_t *>(&S.P);
            for (int w = lane; w < (int)(sizeof(PanelDev) / 8); w += 32) cp_async8(dst + w, src + w);
            if (lane == 0) {
                cp_async8(&S.gx_off, &p.tasks[lo].gx_off);
                S.k = lo;
                S.t = item - s_tpre[lo];
                S.q0 = q0;
                S.q1 = q1;
                S.qd = qd;
            }
            cp_async_commit();
        };
        BandMeta bm;
        if (warp == 0) {
            if (n_items > 0) ring_issue(0);
            if (n_items > 1) ring_issue(1);
            if (BCT_A_META_EARLY && n_items > 2) ring_issue(2);
            cp_async_wait_all();
        }
        __syncthreads();
        if (n_items > 0) {
            band_meta_load(ring[0].P, ring[0].t, bm, nullptr);
            band_issue_gl(ring[0].P, bm, rband, buf[0]);
            if (n_items > 1) band_meta_load(ring[1].P, ring[1].t, bm, nullptr);
        }
        double wacc = 0.0;
        for (int it = 0; it < n_items; ++it) {
            const int cb = dbuf ? (it & 1) : 0;
            if (it == 0 || !dbuf) {   // this band was issued after the last barrier
                cp_async_wait_all();
                __syncthreads();
            }
            if (it == 0 && p.timeline && threadIdx.x == 0 && n_tasks > 1)   // profiling: first band
                p.timeline[((int64_t)1 * 8 + 5) * gridDim.x + blockIdx.x] = gtimer();
            if (it == 1 && p.timeline && threadIdx.x == 0 && n_tasks > 1)   // profiling: first tile done
                p.timeline[((int64_t)1 * 8 + 6) * gridDim.x + blockIdx.x] = gtimer();
            if (it < 8 && p.timeline && threadIdx.x == 0 && n_tasks > 2)    // profiling: tile starts
                p.timeline[((int64_t)2 * 8 + it) * gridDim.x + blockIdx.x] = gtimer();
            const RingSlot &S = ring[it % RING];
            // the other buffer was last read by tile it-1 (before its barrier)
            if (dbuf && it + 1 < n_items)
                band_issue_gl(ring[(it + 1) % RING].P, bm, rband, buf[cb ^ 1]);
            if (BCT_A_META_EARLY) {
                // slot it+3 was last read in iteration it-2 (a barrier ago); slot
                // it+2 completed at the end of the last tile
                if (warp == 0 && it + 3 < n_items) ring_issue(it + 3);
                if (dbuf && it + 2 < n_items)
                    band_meta_load(ring[(it + 2) % RING].P, ring[(it + 2) % RING].t, bm, nullptr);
            } else if (warp == 0 && it + 2 < n_items) {
                ring_issue(it + 2);
            }
            const int nsl = S.P.tile_cols >> 5;
            const double wsum = tile_g<V, TB>(S.P, S.t, S.q0 * nsl / S.qd, S.q1 * nsl / S.qd, buf[cb],
                                          p.x + S.P.x_off, gxb + S.gx_off,
                                          red + (it & 1) * RED_DOUBLES, nullptr);
            wacc += wsum;
            // flush this warp's gg partial when the next item is another task
            // (added: the de-phased first tile's task comes back later)
            const int k = S.k;
            if (it + 1 == n_items || ring[(it + 1) % RING].k != k) {
                const double ws = warp_sum(wacc);
                if (lane == 0) pgg[((int64_t)k * G + b) * WARPS + warp] += ws;
                wacc = 0.0;
            }
            if (!dbuf && it + 1 < n_items)
                band_issue_gl(ring[(it + 1) % RING].P, bm, rband, buf[0]);
            if (it + 2 < n_items && !(BCT_A_META_EARLY && dbuf))
                band_meta_load(ring[(it + 2) % RING].P, ring[(it + 2) % RING].t, bm, nullptr);
        }
    }
    if (!BCT_NO_TL_BATCH) TL_MARK(0, 1);
    grid_sync(p.bar);
    if (!BCT_NO_TL_BATCH) TL_MARK(0, 2);

    // ---- phase B: segment partials of every task (contiguous slice ranges) --
    {
        using GS = typename std::conditional<narrow_math<V>(), float2, double2>::type;
        GS *gs = reinterpret_cast<GS *>(rs);
        // this CTA: the slices whose first entry lies in an equal share of the
        // epoch's stored entries (slices differ in length)
        // cost of a slice prefix = its entries + BCT_B_SLICE_COST per slice
        // (per-slice latency: short slices of rays across the strip cost more
        // per entry than long ones)
        constexpr int64_t SC = BCT_B_SLICE_COST;
        const int64_t cost_total = hdr.n_ent_total + SC * hdr.n_slices_total;
        auto slice_at = [&](int64_t c) -> int {
            if (c >= cost_total) return hdr.n_slices_total;
            const int k = lower_bound_warp([&](int q) {
                return p.tasks[q].ent_pre + SC * p.tasks[q].slice_pre; }, n_tasks, c + 1) - 1;
            const TaskDev &T = p.tasks[k];
            const PanelDev &PP = p.panels[T.lp];
            const int64_t local = c - (T.ent_pre + SC * T.slice_pre);
            return T.slice_pre +
                   lower_bound_warp([&](int q) { return (int64_t)PP.slice_start[q] + SC * q; },
                                    PP.n_slices, local);
        };
        __shared__ int s_range[2];
        __shared__ int s_next;
        if (warp == 0) {
            const int u0 = slice_at(cost_total * b / G);
            const int u1 = slice_at(cost_total * (b + 1) / G);
            if (lane == 0) {
                s_range[0] = u0;
                s_range[1] = u1;
            }
        }
        __syncthreads();
        const int ub = s_range[0], ue = s_range[1];
        int fu = ub;
        int dbg_segs = 0;   // profiling (BCT_TIMELINE): super tiles of this CTA
        long long dbg_stage = 0;   // and their staging time
        while (fu < ue) {
            __syncthreads();
            if (threadIdx.x == 0) {
                const int k = task_of(p.tasks, n_tasks, 1, fu);
                ring[0].k = k;
                ring[0].P = p.panels[p.tasks[k].lp];
                s_next = 0;
            }
            __syncthreads();
            const PanelDev &P = ring[0].P;
            const int k = ring[0].k;
            const TaskDev &T = p.tasks[k];
            const int sl0 = fu - T.slice_pre;          // full panel: flattened = slice id
            // super tile of slice sl0 and the end of its slices
            int st = 0;
            while (__ldg(P.stbs + (st + 1) * (m + 1)) <= sl0 && st + 1 < P.n_st) ++st;
            const int st_end = (st + 1 < P.n_st) ? __ldg(P.stbs + (st + 1) * (m + 1)) : P.n_slices;
            const int ge = min(ue, T.slice_pre + st_end);
            const int v0 = __ldg(P.st_ptr + st), v1 = __ldg(P.st_ptr + st + 1);
            const double2 *gx = gxb + T.gx_off;
            ++dbg_segs;
            const long long tst0 = p.timeline ? gtimer() : 0;
            // Visit order of [fu, ge): the part from the start of its last
            // (super tile, row block) group first, then the rest.  Groups are
            // stored longest slice first, so a share that ends inside a group
            // would otherwise take that group's longest slices last, and the
            // warp holding the last one would finish long after the others.
            __shared__ int s_cut;
            if (threadIdx.x == 0) {
                int cut = fu;
                if (BCT_B_ROT) {
                    const int32_t *g = P.stbs + st * (m + 1);
                    int lo = 0, hi = m;   // last group start < ge
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (T.slice_pre + __ldg(g + mid) < ge) lo = mid; else hi = mid - 1;
                    }
                    cut = max(fu, T.slice_pre + __ldg(g + lo));
                }
                s_cut = cut;
            }
            stage_gx(gs, gx + v0, v1 - v0, P.swz_shift);
            __syncthreads();
            if (p.timeline) dbg_stage += gtimer() - tst0;   // profiling: super-tile staging
            const int n_hi = ge - s_cut, cut = s_cut;
            auto pos = [&](int gq) { return gq < n_hi ? cut + gq : fu + (gq - n_hi); };
            const V *fv = static_cast<const V *>(P.fvals);
            PT *spart = segb + T.seg_off;
            const int wst = P.st_h > 0 ? (v1 - v0) / P.st_h : 1;   // step-coded row length
            // slices are taken one at a time from a shared counter: their
            // lengths vary (up to seg_cap/4 vectors), so a static round robin
            // leaves warps idle at the super tile's barrier
            // The next slice is taken (and its metadata loaded) before the
            // current one is processed: short slices (rays across the strip)
            // would otherwise pay the counter, slice_start and fq0 round trips
            // back to back before their first stream load.
            auto grab = [&]() {   // next visit position (ge: done)
                int g = 0;
                if (lane == 0) g = atomicAdd(&s_next, 1);
                g = __shfl_sync(0xffffffffu, g, 0);
                return g < ge - fu ? pos(g) : ge;
            };
            const bool coded = P.fcode != nullptr && !BCT_NO_FCODE_K;
            int f = grab();
            int base = 0, bend = 0, hdr = 0, dst = 0;
            // a lane's partial goes to its segment's row-order position
            // (P.rq): phase C then reads each row's partials contiguously
            auto dst_of = [&](int slc) {
                return BCT_ROW_ORDER ? __ldg(P.rq + (int64_t)slc * 32 + lane) : slc * 32 + lane;
            };
            if (f < ge) {
                const int sl = f - T.slice_pre;
                base = __ldg(P.slice_start + sl);
                bend = __ldg(P.slice_start + sl + 1);
                if (coded) hdr = __ldg(P.fq0 + (int64_t)sl * 32 + lane);
                dst = dst_of(sl);
            }
            while (f < ge) {
                const int sl = f - T.slice_pre;
                const int fn = grab();
                int nbase = 0, nbend = 0, nhdr = 0, ndst = 0;
                if (fn < ge) {
                    const int sn = fn - T.slice_pre;
                    nbase = __ldg(P.slice_start + sn);
                    nbend = __ldg(P.slice_start + sn + 1);
                    if (coded) nhdr = __ldg(P.fq0 + (int64_t)sn * 32 + lane);
                    ndst = dst_of(sn);
                }
                if (BCT_B_PREFETCH > 0 && lane == 0 && f + BCT_B_PREFETCH < (f >= cut ? ge : cut)) {
                    // the slice another warp takes next round: into L2 now
                    const int sp = sl + BCT_B_PREFETCH;
                    const int e0 = __ldg(P.slice_start + sp), e1 = __ldg(P.slice_start + sp + 1);
                    prefetch_l2(fv + e0, (uint32_t)(e1 - e0) * (uint32_t)sizeof(V));
#if BCT_B_PF_CODES
                    // and its step-code words: (k/4)*32 + lane past
                    // slice_start/16 + 24*slice (128 B per 4 vectors)
                    if (coded && e1 > e0)
                        prefetch_l2(P.fcode + (e0 >> 4) + 24 * sp,
                                    (uint32_t)((((e1 - e0) >> 7) + 3) >> 2) * 128u);
#endif
                }
                const int nvec = (bend - base) >> 7;
                if (coded && !__any_sync(0xffffffffu, (hdr >> 17) & 1)) {
                    // step-coded slice (a lane flagged in fq0 bit 17 keeps its
                    // 16-bit indices: the indexed loop below)
                    const double2 cp = coded_segment<V, GS>(P, fv, sl, base, nvec, lane, wst, gs, hdr);
                    BCT_ASSERT(dst < P.n_slices * 32);
                    if (dst >= 0) spart[dst] = PT{(decltype(PT::x))cp.x, (decltype(PT::x))cp.y};
                } else {
                    // FP32 mode: FP32 lane partials (see coded_segment)
                    using A = typename std::conditional<narrow_math<V>(), float, double>::type;
                    A t = A(0), ax = A(0);
#pragma unroll P2U
                    for (int kv = 0; kv < nvec; ++kv) {
                        const int i = base + ((kv * 32 + lane) << 2);
                        int cc[4];
                        V v[4];
                        ld4u16(P.fidx + i, cc);
                        ld4raw(fv + i, v);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            BCT_ASSERT(cc[q] < P.st_max);
                            const GS a = gs[cc[q]];
                            t = fma((A)v[q], (A)a.x, t);
                            ax = fma((A)v[q], (A)a.y, ax);
                        }
                    }
                    if (dst >= 0) spart[dst] = PT{(decltype(PT::x))t, (decltype(PT::x))ax};
                }
                f = fn;
                base = nbase;
                bend = nbend;
                hdr = nhdr;
                dst = ndst;
            }
            fu = ge;
        }
        if (threadIdx.x == 0) {
            s_range_dbg[0] = ub;
            s_range_dbg[1] = ue;
            s_range_dbg[2] = dbg_segs;
            s_stage_dbg = dbg_stage;
        }
    }
    if (!BCT_NO_TL_BATCH) TL_MARK(0, 3);
    if (p.timeline && n_tasks > 1) {   // profiling: every warp of the block done with B
        __syncthreads();
        if (threadIdx.x == 0) p.timeline[((int64_t)1 * 8 + 4) * gridDim.x + blockIdx.x] = gtimer();
        if (threadIdx.x == 0) __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) p.timeline[((int64_t)1 * 8 + 7) * gridDim.x + blockIdx.x] = gtimer();
    }
    if (p.timeline && threadIdx.x == 0 && n_tasks > 1) {   // profiling: phase-B shares
        p.timeline[((int64_t)1 * 8 + 0) * gridDim.x + blockIdx.x] = s_range_dbg[0];
        p.timeline[((int64_t)1 * 8 + 1) * gridDim.x + blockIdx.x] = s_range_dbg[1];
        p.timeline[((int64_t)1 * 8 + 2) * gridDim.x + blockIdx.x] = s_range_dbg[2];
        p.timeline[((int64_t)1 * 8 + 3) * gridDim.x + blockIdx.x] = s_stage_dbg;
    }
    grid_sync(p.bar);
    if (!BCT_NO_TL_BATCH) TL_MARK(0, 4);

    // ---- phase C: rows of every task (contiguous ranges), denom partials ----
    for (int k = threadIdx.x; k < n_tasks; k += BLOCK) pden[(int64_t)k * G + b] = 0.0;
    // gg of task k from its G*WARPS phase-A partials, one CTA per task (fixed
    // order), so phase D reads one value instead of every CTA summing them all
    for (int k = b; k < n_tasks; k += G) {
        double v = 0.0;
        for (int q = threadIdx.x; q < G * WARPS; q += BLOCK) v += pgg[(int64_t)k * G * WARPS + q];
        v = block_sum_all(v, sh);
        if (threadIdx.x == 0) ggs[k] = v;
    }
    __syncthreads();
    {
        const int nr = hdr.n_rows_total;
        const int rb0 = (int)((int64_t)nr * b / G), rb1 = (int)((int64_t)nr * (b + 1) / G);
        int f0 = rb0;
        while (f0 < rb1) {
            const int k = task_of(p.tasks, n_tasks, 2, f0);
            const TaskDev &T = p.tasks[k];
            const PanelDev &P = p.panels[T.lp];
            const int f1 = min(rb1, T.row_pre + P.n_rows);
            const PT *spart = segb + T.seg_off;
            // fused tail: (t, ax) kept per panel row (the z of the panel from
            // now on), else per-epoch scratch for phase D
            PT *tax = hdr.fuse_tail ? reinterpret_cast<PT *>(p.zt) + P.row_off
                                    : taxb + T.tax_off;
            double wsum = 0.0;
            // CR rows per thread at a time, their (pointer, position, partial)
            // loads issued level by level: CR-fold memory parallelism for a
            // chain of three dependent loads per row
            constexpr int CR = 4;
            for (int fb = f0 + (int)threadIdx.x; fb < f1; fb += CR * BLOCK) {
                int q0[CR], q1[CR];
                double t[CR], ax[CR];
                int nmax = 0;
#pragma unroll
                for (int j = 0; j < CR; ++j) {
                    const int f = fb + j * BLOCK;
                    const int lr = f - T.row_pre;
                    q0[j] = f < f1 ? __ldg(P.rseg_ptr + lr) : 0;
                    q1[j] = f < f1 ? __ldg(P.rseg_ptr + lr + 1) : 0;
                    t[j] = 0.0;
                    ax[j] = 0.0;
                    nmax = max(nmax, q1[j] - q0[j]);
                }
                for (int s = 0; s < nmax; ++s) {
                    int pos[CR];
#pragma unroll
                    for (int j = 0; j < CR; ++j)
                        pos[j] = q0[j] + s < q1[j] ? (BCT_ROW_ORDER ? q0[j] + s : __ldg(P.rpos + q0[j] + s))
                                                   : -1;
#pragma unroll
                    for (int j = 0; j < CR; ++j)
                        if (pos[j] >= 0) {
                            // written in phase B of this launch: L2-coherent load
                            const PT a = __ldcg(spart + pos[j]);   // row-order partials
                            t[j] += (double)a.x;
                            ax[j] += (double)a.y;
                        }
                }
#pragma unroll
                for (int j = 0; j < CR; ++j) {
                    const int f = fb + j * BLOCK;
                    if (f < f1) {
                        const PT tq = PT{(decltype(PT::x))t[j], (decltype(PT::x))ax[j]};
                        tax[f - T.row_pre] = tq;
                        // denom from the stored t (phase D's z uses the same t)
                        wsum = fma((double)tq.x, (double)tq.x, wsum);
                    }
                }
            }
            const double bs = block_sum_all(wsum, sh);
            if (threadIdx.x == 0) pden[(int64_t)k * G + b] += bs;
            f0 = f1;
        }
    }
    if (!BCT_NO_TL_BATCH) TL_MARK(0, 5);
    grid_sync(p.bar);

    // ---- phase D: mu per task, xhat per visit, z per task -----------------
    double *mu_s = rs;                                    // [n_tasks]
    int *st_s = reinterpret_cast<int *>(rs + n_tasks);   // [n_tasks]
    for (int k = warp; k < n_tasks; k += WARPS) {
        double gg = 0.0, den = 0.0;
        for (int q = lane; q < G; q += 32) den += pden[(int64_t)k * G + q];
        gg = ggs[k];
        den = warp_sum(den);
        if (lane != 0) continue;
        double mu = 0.0;
        int status = 0;
        if (gg == 0.0) status = 1;
        else if (den < 1e-30) status = 2;
        else mu = p.tasks[k].beta * gg / den;
        mu_s[k] = mu;
        st_s[k] = status;
        if (b == 0) {
            p.mus[k] = mu;
            p.statuses[k] = status;
        }
    }
    __syncthreads();
    if (hdr.fuse_tail) {
        // phase D is done by the epoch tail (z from (t, ax) where the refresh
        // reads it, x-hat in the commit pass; counts by the last block):
        // per owned panel its offsets and task, after mu / status
        const FuseTables ft = fuse_tables(rs, n_tasks, p.n_panels_owned);
        for (int lp = threadIdx.x; lp <= p.n_panels_owned; lp += BLOCK) {
            const bool in = lp < p.n_panels_owned;
            ft.roff[lp] = in ? (int32_t)p.panels[lp].row_off : (int32_t)p.z_len;
            ft.xoff[lp] = in ? p.panels[lp].x_off : p.x_len;
            if (in) {
                // z form left by earlier epochs (rewritten by the last block)
                const bool lazy = p.zl_on[lp] != 0;
                ft.task[lp] = -1;
                ft.st[lp] = lazy ? p.zl_st[lp] : -1;
                ft.mu[lp] = lazy ? p.zl_mu[lp] : 0.0;
            }
        }
        __syncthreads();
        for (int k = threadIdx.x; k < n_tasks; k += BLOCK) {
            const TaskDev &T = p.tasks[k];
            const PanelDev &P = p.panels[T.lp];
            ft.task[T.lp] = k;   // one task per panel on this path (api.cu)
            ft.st[T.lp] = st_s[k];
            ft.mu[T.lp] = mu_s[k];
            ft.gxo[T.lp] = T.gx_off - P.x_off;
        }
        __syncthreads();
        if (!BCT_NO_TL_BATCH) TL_MARK(0, 6);
        return;
    }
    if (b == 0 && threadIdx.x == 0)
        for (int k = 0; k < n_tasks; ++k) p.counts[p.tasks[k].lp] += 1;
    {
        // xhat: voxels of every visit (its first task), its tasks summed in
        // order; contiguous voxel ranges per CTA, one task lookup per visit
        const int nv = hdr.n_vox_total;
        const int vb0 = (int)((int64_t)nv * b / G), vb1 = (int)((int64_t)nv * (b + 1) / G);
        int v0 = vb0;
        while (v0 < vb1) {
            int k0 = task_of(p.tasks, n_tasks, 3, v0);
            while (k0 > 0 && !(p.tasks[k0].flags & TASK_FIRST_OF_VISIT)) --k0;
            int k1 = k0 + 1;
            while (k1 < n_tasks && !(p.tasks[k1].flags & TASK_FIRST_OF_VISIT)) ++k1;
            const TaskDev &T0 = p.tasks[k0];
            const PanelDev &P = p.panels[T0.lp];
            const int v1 = min(vb1, T0.vox_pre + P.n_cols);
            const double *xs_in = p.x + P.x_off;
            double *xh = p.xhat + P.x_off;
            for (int v = v0 + (int)threadIdx.x; v < v1; v += BLOCK) {
                const int d = v - T0.vox_pre;
                const double xv = xs_in[d];
                double xs = 0.0;
                for (int k = k0; k < k1; ++k) {
                    const double2 a = gxb[p.tasks[k].gx_off + d];
                    xs += st_s[k] == 0 ? __dadd_rn(xv, __dmul_rn(mu_s[k], a.x)) : xv;
                }
                xh[d] += xs;
            }
            v0 = v1;
        }
        // z of every task's rows: contiguous row ranges per CTA (as phase C)
        const int nr = hdr.n_rows_total;
        const int rb0 = (int)((int64_t)nr * b / G), rb1 = (int)((int64_t)nr * (b + 1) / G);
        int f0 = rb0;
        while (f0 < rb1) {
            const int k = task_of(p.tasks, n_tasks, 2, f0);
            const TaskDev &T = p.tasks[k];
            const PanelDev &P = p.panels[T.lp];
            const int f1 = min(rb1, T.row_pre + P.n_rows);
            const PT *tax = taxb + T.tax_off - T.row_pre;
            double *zr = p.z + P.row_off - T.row_pre;
            const double mu = mu_s[k];
            const int st = st_s[k];
            // four rows in flight per thread: loads (L2-coherent: tax was
            // written in phase C of this launch) before the stores
            for (int fb = f0 + (int)threadIdx.x; fb < f1; fb += 4 * BLOCK) {
                PT q[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    q[j] = fb + j * BLOCK < f1 ? __ldcg(tax + fb + j * BLOCK) : PT{0, 0};
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (fb + j * BLOCK < f1)
                        zr[fb + j * BLOCK] = z_value((double)q[j].x, (double)q[j].y, mu, st);
            }
            f0 = f1;
        }
    }
    if (!BCT_NO_TL_BATCH) TL_MARK(0, 6);
}

// Per-task phase 2a: exclusive prefix of the work units (parts_of) of slices
// [c0, c0 + nc) of super tile st into s_upre[0..nc] (whole CTA; complete after
// the caller's next __syncthreads)
__device__ __forceinline__ void unit_prefix(const PanelDev &P, const PrepView &R, int m, int c0,
                                            int nc, int st, bool rfull, int *s_upre)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < nc; i += BLOCK) {
        const int sl = rfull ? c0 + i : task_slice(R, P, m, c0 + i, st);
        s_upre[i] = parts_of((__ldg(P.slice_start + sl + 1) - __ldg(P.slice_start + sl)) >> 7, true);
    }
    __syncthreads();
    if (warp == 0) {   // exclusive prefix, 32 slices per step
        int carry = 0;
        for (int b0 = 0; b0 < nc; b0 += 32) {
            const int v = b0 + lane < nc ? s_upre[b0 + lane] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (b0 + lane < nc) s_upre[b0 + lane] = carry + incl - v;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) s_upre[nc] = carry;
    }
}

template <typename V>
__global__ void __launch_bounds__(BLOCK, 1) epoch_kernel(EpochParams p)
{
    extern __shared__ double4 dyn_smem[];
    __shared__ double sh[WARPS];
    // the current task's record (PrepHdr + arrays) after the phase buffers
    PrepView R(reinterpret_cast<char *>(dyn_smem) + p.prep_smem_off, p.prep_dims);
    __shared__ int2 vr_s[8];
    __shared__ int s_upre[UCAP + 1];   // per-task phase 2a unit prefix

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gtid = blockIdx.x * BLOCK + threadIdx.x;
    const int nthreads = gridDim.x * BLOCK;
    const int m = p.m;
    const EpochHeader hdr = *p.hdr;
    if (hdr.flags & 8) {
        // divergence guard: the previous epoch's |x| (its result is still in
        // p.out; every block reads it before any block can pass a grid
        // barrier, and only the last block of this launch rewrites it)
        const double nx = sqrt(__ldcg(&p.out->x_sq));
        if (!isfinite(nx) || nx > hdr.guard_factor * __ldcg(p.guard_ref)) {
            // skipped: the result block repeats the previous epoch's (as the
            // device block still holds it)
            if (blockIdx.x == 0 && p.res_host)
                for (int q = threadIdx.x; q < (int)(sizeof(EpochOut) / 8); q += BLOCK)
                    reinterpret_cast<double *>(p.res_host)[q] =
                        __ldcg(reinterpret_cast<const double *>(p.out) + q);
            return;
        }
    }
    const int n_tasks = hdr.n_tasks;
    const bool serial = hdr.mode == 0;
    const bool sharded = (hdr.flags & 4) != 0;
    double *part_gg = p.part;
    double *part_den = p.part + gridDim.x;
    double *part_m = p.part + 2 * gridDim.x;
    double *rs = reinterpret_cast<double *>(dyn_smem);   // phase 1 band
    // phase 2 super tile: (g, x) pairs, float2 when values are float (FP32 mode)
    using GS = typename std::conditional<narrow_math<V>(), float2, double2>::type;
    GS *gs = reinterpret_cast<GS *>(dyn_smem);

    __shared__ RingSlot ring[RING];
    __shared__ int s_tpre[bct::MAX_BATCH_TASKS + 1], s_lp[bct::MAX_BATCH_TASKS];
    if (hdr.batched) batched_epoch<V>(p, hdr, rs, sh, ring, s_tpre, s_lp);
    // a task's set-up record into shared memory: built on the host with the
    // plan (api.cu host_prep, one copy) or by one thread (sampled epochs)
    auto load_record = [&](int kk) {
        if (!hdr.host_prep) {
            if (threadIdx.x == 0) prep_task(p, kk, R);
        } else {
            const int64_t rb = p.prep_dims.bytes();
            const float4 *src = reinterpret_cast<const float4 *>(p.prep + rb * kk);
            float4 *dst = reinterpret_cast<float4 *>(R.h);
            for (int q = threadIdx.x; q < (int)(rb / 16); q += BLOCK) dst[q] = __ldcg(src + q);
        }
    };
    bool have_rec = false;   // loaded ahead, before the previous task's last barrier
    // phase-1 work items: whole tiles in rounds of gridDim.x; the tiles left
    // for the last round are split into column parts so every CTA gets the
    // same share
    struct Items {
        int full, S, n;
        __device__ Items(const PanelDev &P)
        {
            const int NSL = P.tile_cols >> 5, G = gridDim.x;
            full = P.n_tiles / G;
            const int rem = P.n_tiles - full * G;
            S = rem > 0 ? max(1, min(NSL, G / rem)) : 1;
            n = full + ((int)blockIdx.x < rem * S ? 1 : 0);
        }
        __device__ int tile(int it) const
        {
            return it < full ? (int)blockIdx.x + it * (int)gridDim.x
                             : full * (int)gridDim.x + (int)blockIdx.x / S;
        }
    };
    for (int k = 0; k < (hdr.batched ? 0 : n_tasks); ++k) {
        if (!have_rec) {
            __syncthreads();  // the previous task's record may still be in use
            load_record(k);
            __syncthreads();
        }
        have_rec = false;
        const TaskDev &T = R.h->T;
        const PanelDev &P = R.h->P;
        const uint64_t *tmask = p.masks + task_mask_off(k, p.mw);
        TL_MARK(k, 0);
        double2 *gx = reinterpret_cast<double2 *>(p.gx + (k & 1) * p.gx_stride);
        const double *xj = p.x + P.x_off;
        const bool rfull = R.h->full != 0;
        const Items items(P);

        // This CTA's phase-2a slices: a full-panel task splits them by stored
        // entries (table built at set-up, api.cu finalize: no per-task search),
        // any other task by slice count.
        // (CTA-uniform values kept in shared memory: registers are scarce)
        __shared__ int s_ub, s_ue, s_pre_nc;
        int ub, ue;
        {
            const int ns = R.st_pre[R.h->nst];
            if (rfull) {
                const int32_t *cs = p.cta_split + (int64_t)T.lp * (gridDim.x + 1) + blockIdx.x;
                ub = __ldg(cs);
                ue = __ldg(cs + 1);
            } else {
                ub = (int)((int64_t)ns * blockIdx.x / gridDim.x);
                ue = (int)((int64_t)ns * (blockIdx.x + 1) / gridDim.x);
            }
        }
        // ---- phase 1: g = A_I^T r_I, tile bands in shared memory ----------
        // Work items are whole tiles in rounds of gridDim.x; the tiles left for
        // the last round are split into column parts so every CTA gets the
        // same share.  The band of the next item is copied (bulk copies) into
        // the second buffer while the current item is computed.
        double wsum = 0.0;
        {
            const int NSL = P.tile_cols >> 5;
            const int full = items.full, S = items.S, n_items = items.n;
            auto item_tile = [&](int it) { return items.tile(it); };
            const bool dbuf = p.band_dbuf != 0;
            double *buf0 = rs, *buf1 = rs + (dbuf ? p.band_cap : 0);
            double *red = rs + (int64_t)p.band_cap * (dbuf ? 2 : 1);
            const uint64_t *bmask = R.h->full ? nullptr : tmask;
            BandMeta bm;
            if (n_items > 0) {
                band_meta_load(P, item_tile(0), bm, bmask);
                band_issue(P, bm, p.r, buf0, bmask);
                if (n_items > 1) band_meta_load(P, item_tile(1), bm, bmask);
            }
            // while the first band is in flight: the unit prefix of this
            // CTA's first phase-2a chunk (plan-only).  (L2 prefetches of the
            // CTA's phase-1 or phase-2a streams here or at the task start, and
            // loading the next task's first band metadata before the refresh
            // barrier, measured slower: config 2 2.1-6% per epoch)
            // unit prefix of the first phase-2a chunk (full tasks; chunk [ub, ub + s_pre_nc))
            {
                int pre_nc = 0;
                if (rfull && ue > ub) {
                    int st = 0;
                    while (ub >= R.st_pre[st + 1]) ++st;
                    pre_nc = min(min(ue, R.st_pre[st + 1]) - ub, UCAP);
                    unit_prefix(P, R, m, ub, pre_nc, st, true, s_upre);
                }
                if (threadIdx.x == 0) {
                    s_ub = ub;
                    s_ue = ue;
                    s_pre_nc = pre_nc;
                }
            }

            int cur = 0;
            for (int it = 0; it < n_items; ++it) {
                cp_async_wait_all();
                __syncthreads();
                if (it == 0) TL_MARK(k, 7);   // profiling: the first band is staged
                const int t = item_tile(it);
                int c0 = 0, c1 = NSL;
                if (it >= full) {
                    const int part = (int)blockIdx.x % S;
                    c0 = part * NSL / S;
                    c1 = (part + 1) * NSL / S;
                }
                double *bt = cur ? buf1 : buf0;
                if (dbuf && it + 1 < n_items) {
                    band_issue(P, bm, p.r, cur ? buf0 : buf1, bmask);
                    if (it + 2 < n_items) band_meta_load(P, item_tile(it + 2), bm, bmask);
                }
                if (bmask != nullptr) {
                    const int nr = R.h->n_runs;
                    tile_vr(P, m, t, c0, c1, nr > 0 ? R.i0[0] : 0, nr > 0 ? R.i1[nr - 1] : 0,
                            vr_s);
                    __syncthreads();
                }
                wsum += tile_g<V>(P, t, c0, c1, bt, xj, gx, red, bmask != nullptr ? vr_s : nullptr);
                if (it == 0) TL_MARK2(k, 0);   // profiling: first item computed

                __syncthreads();
                if (dbuf) {
                    cur ^= 1;
                } else if (it + 1 < n_items) {
                    band_issue(P, bm, p.r, buf0, bmask);
                    if (it + 2 < n_items) band_meta_load(P, item_tile(it + 2), bm, bmask);
                }
            }
        }
        TL_MARK(k, 1);
        // gg is first needed for mu, after the next barrier: reduced there,
        // together with the denominators (one read of the partials off the
        // critical path here).  Partials alternate between two buffers by
        // task: without a barrier between tasks (parallel mode) a fast CTA
        // writes the next task's while a slow one may still read these.
        double *pgg = part_gg + ((k & 1) ? 5 * gridDim.x : 0);
        double bsum = block_sum_all(wsum, sh);
        if (threadIdx.x == 0) pgg[blockIdx.x] = bsum;
        grid_sync(p.bar);
        TL_MARK(k, 2);

        // ---- phase 2a: segment partials of t = A_I g, ax = A_I x_J -------
        // SELL-32 slices, one segment per lane; (g, x) of the slice's super
        // tile staged in shared memory.  A full-panel task splits the slices
        // among CTAs by stored entries, any other task by slice count.
        // A panel whose rows are single segments (one super tile, uncut
        // runs: every strip panel of an FP64 context up to 8192 voxels) has
        // its rows complete in this CTA's slices: the CTA sums their parts
        // itself, and the grid barrier + row pass of phase 2b go away.
        const bool fused = P.n_st == 1 && P.n_seg == P.n_rows;
        {
            const V *fv = static_cast<const V *>(P.fvals);
            double2 *spart = reinterpret_cast<double2 *>(p.seg_part);
            ub = s_ub;
            ue = s_ue;
            const int pre_c0 = ub, pre_nc = s_pre_nc;
            int fu = ub;
            while (fu < ue) {
                int st = 0;
                while (fu >= R.st_pre[st + 1]) ++st;
                const int ge = min(ue, R.st_pre[st + 1]);
                const int v0 = __ldg(P.st_ptr + st), v1 = __ldg(P.st_ptr + st + 1);
                stage_gx(gs, gx + v0, v1 - v0, P.swz_shift);
                // work unit = (slice, part): part q of a slice with np parts
                // takes its vectors kv = q (mod np); the units of up to UCAP
                // slices are numbered through a prefix of their part counts
                // (partial tasks: TS_PARTIAL parts per slice, no prefix)
                if (!rfull) {
                    __syncthreads();
                    for (int u = fu * TS_PARTIAL + warp; u < ge * TS_PARTIAL; u += WARPS) {
                        const int f = u / TS_PARTIAL, part = u - f * TS_PARTIAL;
                        const int sl = task_slice(R, P, m, f, st);
                        const int base = __ldg(P.slice_start + sl);
                        const int nvec = (__ldg(P.slice_start + sl + 1) - base) >> 7;
                        double t = 0.0, ax = 0.0;
#pragma unroll P2U
                        for (int kv = part; kv < nvec; kv += TS_PARTIAL) {
                            const int i = base + ((kv * 32 + lane) << 2);
                            int cc[4];
                            double v[4];
                            ld4u16(P.fidx + i, cc);
                            ld4v(fv + i, v);
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                BCT_ASSERT(cc[q] < P.st_max);
                            const GS a = gs[cc[q]];
                                t = fma(v[q], (double)a.x, t);
                                ax = fma(v[q], (double)a.y, ax);
                            }
                        }
                        spart[((int64_t)sl * TS_MAX + part) * 32 + lane] = make_double2(t, ax);
                    }
                    __syncthreads();
                    fu = ge;
                    continue;
                }
                for (int c0 = fu; c0 < ge; c0 += UCAP) {
                    const int nc = min(ge - c0, UCAP);
                    if (c0 != pre_c0 || nc != pre_nc) unit_prefix(P, R, m, c0, nc, st, rfull, s_upre);
                    __syncthreads();   // (the staged (g, x) too)
                    if (c0 == ub) TL_MARK2(k, 1);   // profiling: super tile staged
                    const int total = s_upre[nc];
                    for (int u = warp; u < total; u += WARPS) {
                        int lo = 0, hi = nc - 1;   // last slice whose units start <= u
                        while (lo < hi) {
                            const int mid = (lo + hi + 1) >> 1;
                            if (s_upre[mid] <= u) lo = mid; else hi = mid - 1;
                        }
                        const int part = u - s_upre[lo], np = s_upre[lo + 1] - s_upre[lo];
                        const int f = c0 + lo;
                        const int sl = rfull ? f : task_slice(R, P, m, f, st);
                        const int base = __ldg(P.slice_start + sl);
                        const int nvec = (__ldg(P.slice_start + sl + 1) - base) >> 7;
                        double t = 0.0, ax = 0.0;
#pragma unroll P2U
                        for (int kv = part; kv < nvec; kv += np) {
                            const int i = base + ((kv * 32 + lane) << 2);
                            int cc[4];
                            double v[4];
                            ld4u16(P.fidx + i, cc);
                            ld4v(fv + i, v);
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                BCT_ASSERT(cc[q] < P.st_max);
                            const GS a = gs[cc[q]];
                                t = fma(v[q], (double)a.x, t);
                                ax = fma(v[q], (double)a.y, ax);
                            }
                        }
                        spart[((int64_t)sl * TS_MAX + part) * 32 + lane] = make_double2(t, ax);
                    }
                    __syncthreads();
                }
                fu = ge;
            }
        }
        TL_MARK(k, 3);
        TL_MARK2(k, 2);
        const int n_task_rows = R.pre[R.h->n_runs];
        wsum = 0.0;
        if (fused) {
            // rows of this CTA's slices (written by this CTA above: the
            // __syncthreads that closed the loop orders them): t, ax = the
            // lane's parts in order; denominators per CTA
            const double2 *spart = reinterpret_cast<const double2 *>(p.seg_part);
            double2 *tax = reinterpret_cast<double2 *>(p.t_ax);
            for (int q = ub * 32 + (int)threadIdx.x; q < ue * 32; q += BLOCK) {
                const int f = q >> 5, ln = q & 31;
                const int sl = rfull ? f : task_slice(R, P, m, f, 0);
                const int seg = __ldg(P.sl_seg + (int64_t)sl * 32 + ln);
                if (seg < 0) continue;
                const int lr = __ldg(P.seg_key + seg);   // one super tile: key = local row
                const double2 *pp = spart + ((int64_t)sl * TS_MAX) * 32 + ln;
                const int np = parts_of((__ldg(P.slice_start + sl + 1) -
                                         __ldg(P.slice_start + sl)) >> 7, rfull);
                double t = 0.0, ax = 0.0;
                for (int part = 0; part < np; ++part) {
                    const double2 a = pp[part * 32];
                    t += a.x;
                    ax += a.y;
                }
                BCT_ASSERT(lr >= 0 && lr < P.n_rows);
                tax[lr] = make_double2(t, ax);
                wsum = fma(t, t, wsum);
            }
        } else {
        grid_sync(p.bar);

        // ---- phase 2b: rows = sum of their segments in tile order ----------
        {
            const double2 *spart = reinterpret_cast<const double2 *>(p.seg_part);
            double2 *tax = reinterpret_cast<double2 *>(p.t_ax);
            for (int f = gtid; f < n_task_rows; f += nthreads) {
                const int lr = run_row(R, f);
                double t = 0.0, ax = 0.0;
                const int q1 = __ldg(P.rseg_ptr + lr + 1);
                for (int q = __ldg(P.rseg_ptr + lr); q < q1; ++q) {
                    const int rp = __ldg(P.rpos + q);   // SELL position: slice*32 + lane
                    const int sq = rp >> 5;
                    const double2 *pp = spart + ((int64_t)sq * TS_MAX) * 32 + (rp & 31);
                    const int np = parts_of((__ldg(P.slice_start + sq + 1) -
                                             __ldg(P.slice_start + sq)) >> 7, R.h->full != 0);
                    double st_ = 0.0, sa_ = 0.0;
                    for (int part = 0; part < np; ++part) {
                        const double2 a = pp[part * 32];
                        st_ += a.x;
                        sa_ += a.y;
                    }
                    t += st_;
                    ax += sa_;
                }
                BCT_ASSERT(lr >= 0 && lr < P.n_rows);
                tax[lr] = make_double2(t, ax);
                wsum = fma(t, t, wsum);
            }
        }
        }
        TL_MARK(k, 4);
        bsum = block_sum_all(wsum, sh);
        if (threadIdx.x == 0) part_den[blockIdx.x] = bsum;
        grid_sync(p.bar);
        double gg, denom;
        fixed_sum2(pgg, part_den, gridDim.x, sh, gg, denom);
        TL_MARK(k, 5);

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
            for (int d = gtid; d < P.n_cols; d += nthreads) {
                double2 a = gx[d];
                double xn = status == 0 ? __dadd_rn(a.y, __dmul_rn(mu, a.x)) : a.y;
                xh[d] += xn;
            }
        }
        TL_MARK2(k, 3);   // profiling: mu, xhat done
        const bool last_of_visit = (T.flags & TASK_LAST_OF_VISIT) != 0;
        const bool refresh = serial && last_of_visit;
        if (!refresh) {   // (the refresh below stores this task's z itself)
            const double2 *tax = reinterpret_cast<const double2 *>(p.t_ax);
            double *zj = p.z + P.row_off;
            for (int f = gtid; f < n_task_rows; f += nthreads) {
                int lr = run_row(R, f);
                double2 q = tax[lr];
                zj[lr] = z_value(q.x, q.y, mu, status);
            }
        }
        if (refresh) {
            // refresh every row of the visit's drawn blocks (executor.py:215-223),
            // one flat pass over their rows; the current task's z is computed
            // here and stored on the way (every one of its rows is refreshed)
            const int *s_vb = R.vb, *s_vpre = R.vpre;
            const int nvb = R.h->nvb, tot = s_vpre[nvb];
            const double2 *tax = reinterpret_cast<const double2 *>(p.t_ax);
            const int64_t zlo = P.row_off, zhi = P.row_off + P.n_rows;
            // every row block drawn and in the task's group (full-panel serial
            // visits): every measurement is refreshed, so walk them in order
            // through the interleaved inverse map (coalesced slot lists, the
            // same ascending-j fold) instead of block -> row -> list lookups
            const bool all_rows = BCT_REFRESH_ALL && R.h->full && nvb == m && tot == p.n_meas;
            if (all_rows) {
                const int64_t n_pad = (p.n_meas + 31) & ~31ll;
                for (int64_t g = gtid; g < n_pad; g += nthreads) {
                    const int64_t G = g >> 5;
                    const int e0 = __ldg(p.invt_off + G), e1 = __ldg(p.invt_off + G + 1);
                    const double yg = g < p.n_meas ? __ldg(p.y + g) : 0.0;
                    double acc = 0.0;
                    constexpr int RF = BCT_REFRESH_RF;
                    for (int e = e0 + (int)(g & 31); e < e1; e += 32 * RF) {
                        int off[RF];
                        double v[RF];
#pragma unroll
                        for (int u = 0; u < RF; ++u)
                            off[u] = e + 32 * u < e1 ? __ldg(p.invt + e + 32 * u) : -1;
#pragma unroll
                        for (int u = 0; u < RF; ++u) {
                            BCT_ASSERT(off[u] < p.z_len);
                            if (off[u] < 0) {
                                v[u] = 0.0;
                            } else if (off[u] >= zlo && off[u] < zhi) {
                                const double2 qq = tax[off[u] - zlo];
                                v[u] = z_value(qq.x, qq.y, mu, status);
                                p.z[off[u]] = v[u];
                            } else {
                                v[u] = __ldcg(p.z + off[u]);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < RF; ++u)
                            if (off[u] >= 0) acc += v[u];
                    }
                    if (g >= p.n_meas) continue;
                    const double rv = yg - acc;
                    p.r[g] = rv;
                    if (p.r32) p.r32[g] = (float)rv;
                }
            }
            for (int f = all_rows ? tot : gtid; f < tot; f += nthreads) {
                int lo = 0, hi = nvb - 1;   // last drawn block with prefix <= f
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_vpre[mid] <= f) lo = mid; else hi = mid - 1;
                }
                const int i = s_vb[lo];
                const bool cur = mask_has(tmask, i);
                const int g = __ldg(p.rb_rows + __ldg(p.rb_ptr + i) + (f - s_vpre[lo]));
                const int e1 = __ldg(p.inv_ptr + g + 1);
                const double yg = __ldg(p.y + g);
                double acc = 0.0;
                // the row's z slots (ascending j) in groups of RF: their
                // offsets, then their values, in flight together
                constexpr int RF = BCT_REFRESH_RF;
                for (int e = __ldg(p.inv_ptr + g); e < e1; e += RF) {
                    int off[RF];
                    double v[RF];
#pragma unroll
                    for (int u = 0; u < RF; ++u) off[u] = e + u < e1 ? __ldg(p.inv_z + e + u) : -1;
#pragma unroll
                    for (int u = 0; u < RF; ++u) {
                        BCT_ASSERT(off[u] < p.z_len);
                        if (off[u] < 0) {
                            v[u] = 0.0;
                        } else if (cur && off[u] >= zlo && off[u] < zhi) {
                            const double2 qq = tax[off[u] - zlo];
                            v[u] = z_value(qq.x, qq.y, mu, status);
                            p.z[off[u]] = v[u];
                        } else {
                            v[u] = __ldcg(p.z + off[u]);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < RF; ++u)
                        if (off[u] >= 0) acc += v[u];
                }
                const double rv = yg - acc;
                p.r[g] = rv;
                if (p.r32) p.r32[g] = (float)rv;
            }
            TL_MARK2(k, 4);   // profiling: refresh done (this block)
            if (k + 1 < n_tasks) {
                // this task's record is no longer read: load the next task's
                // while the other CTAs finish their refresh (it depends on
                // the plan only, not on r)
                __syncthreads();
                load_record(k + 1);
                have_rec = true;
                TL_MARK2(k, 5);
                grid_sync(p.bar);
            }
        }
        TL_MARK(k, 6);
    }

    // ---- epoch tail ------------------------------------------------------
    // fused batched tail: phase D's work is done here, after phase C's barrier
    const bool fuse = hdr.batched && hdr.fuse_tail;
    if (!fuse) grid_sync(p.bar);
    const bool do_metrics = (hdr.flags & 2) != 0;
    const bool do_commit = (hdr.flags & 1) != 0;
    double rsq = 0.0, xsq = 0.0, esq = 0.0;
    using PT = typename std::conditional<narrow_math<V>(), float2, double2>::type;
    const PT *zt = reinterpret_cast<const PT *>(p.zt);
    const FuseTables ft = fuse_tables(rs, n_tasks, p.n_panels_owned);
    int lpc = 0;   // panel of the thread's last z offset (offsets ascend within a row)
    // z values at offsets o[0..N) (-1: none): the stored z, or on the fused
    // path z = ax + mu t from the panel's persistent (t, ax) pairs
    auto zvals = [&](auto &o, auto &v) {
        constexpr int N = sizeof(o) / sizeof(o[0]);
        if (!fuse) {
#pragma unroll
            for (int u = 0; u < N; ++u) v[u] = o[u] >= 0 ? __ldcg(p.z + o[u]) : 0.0;
            return;
        }
        int lq[N];
#pragma unroll
        for (int u = 0; u < N; ++u) {
            lq[u] = -1;
            if (o[u] < 0) continue;
            while (o[u] < ft.roff[lpc]) --lpc;
            while (o[u] >= ft.roff[lpc + 1]) ++lpc;
            lq[u] = lpc;
        }
        PT q[N];
#pragma unroll
        for (int u = 0; u < N; ++u) {
            // (t, ax) written in phase C of this launch: L2-coherent loads
            if (lq[u] >= 0 && ft.st[lq[u]] >= 0) q[u] = __ldcg(zt + o[u]);
            else v[u] = o[u] >= 0 ? __ldcg(p.z + o[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < N; ++u)
            if (lq[u] >= 0 && ft.st[lq[u]] >= 0)
                v[u] = z_value((double)q[u].x, (double)q[u].y, ft.mu[lq[u]], ft.st[lq[u]]);
    };
    if (!serial || do_metrics || sharded) {
        // warps cover 32 consecutive measurements (gtid and nthreads are
        // multiples of 32): the interleaved inverse map is read coalesced
        // (contiguous CTA shares balanced by z slots measured slower: 1.736 ->
        // 1.746 ms at config 4, the strided deal spreads long and short lists)
        const int64_t n_pad = (p.n_meas + 31) & ~31ll;
        for (int64_t g = gtid; g < n_pad; g += nthreads) {
            double acc = 0.0;
            const int64_t G = g >> 5;
            const int e0 = __ldg(p.invt_off + G), e1 = __ldg(p.invt_off + G + 1);
            // the row's y and block, loaded ahead of its slot chain
            const bool live = g < p.n_meas && !sharded;
            const double yg = live ? __ldg(p.y + g) : 0.0;
            const int rbg = live ? __ldg(p.rb_of_row + g) : -1;
            // ascending j (the reference's fold); z was written earlier in this
            // launch: L2-coherent loads, TU in flight (predicated groups: a
            // list's last few slots do not pay one round trip each); -1 pads
            // a list
            constexpr int TU = BCT_TAIL_U;
            for (int e = e0 + (int)(g & 31); e < e1; e += 32 * TU) {
                int o[TU];
                double v[TU];
#pragma unroll
                for (int u = 0; u < TU; ++u) o[u] = e + 32 * u < e1 ? __ldg(p.invt + e + 32 * u) : -1;
                zvals(o, v);
#pragma unroll
                for (int u = 0; u < TU; ++u)
                    if (o[u] >= 0) acc += v[u];
            }
            if (g >= p.n_meas) continue;
            if (sharded) {
                p.exchange[g] = acc;
            } else {
                double d = yg - acc;
                int rb = rbg;
                if (!serial && rb >= 0 && mask_has(p.masks, rb)) {
                    p.r[g] = d;
                    if (p.r32) p.r32[g] = (float)d;
                }
                rsq = fma(d, d, rsq);
            }
        }
    }
    if (hdr.batched) TL_MARK2(0, 0);   // profiling: the tail's measurement pass done
    // commit and image norms over all owned voxels at once (panels are
    // contiguous in x / xhat / x_true); the panel of a voxel by binary search
    {
        const int npo = p.n_panels_owned;
        const double2 *gxb = reinterpret_cast<const double2 *>(p.gx_batch);
        for (int64_t v = gtid; v < p.x_len; v += nthreads) {
            int lo = 0, hi = npo - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if ((fuse ? ft.xoff[mid] : p.panels[mid].x_off) <= v) lo = mid; else hi = mid - 1;
            }
            int cnt = p.counts[lo];
            double xv = p.x[v];
            const int kf = fuse ? ft.task[lo] : -1;
            if (kf >= 0) {
                // phase D's x-hat update of the visit (one task), then commit
                const double2 a = __ldcg(gxb + ft.gxo[lo] + v);
                const double xs =
                    0.0 + (ft.st[lo] == 0 ? __dadd_rn(xv, __dmul_rn(ft.mu[lo], a.x)) : xv);
                const double xh = p.xhat[v] + xs;
                ++cnt;
                if (do_commit) {
                    xv = xh / (double)cnt;
                    p.x[v] = xv;
                    p.xhat[v] = 0.0;
                } else {
                    p.xhat[v] = xh;
                }
            } else if (do_commit && cnt > 0) {
                xv = p.xhat[v] / (double)cnt;
                p.x[v] = xv;
                p.xhat[v] = 0.0;
            }
            xsq = fma(xv, xv, xsq);
            if (p.x_true) {
                const double d = p.x_true[v] - xv;
                esq = fma(d, d, esq);
            }
        }
    }
    if (hdr.batched && !BCT_NO_TL_BATCH) TL_MARK(0, 7);
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
        // the whole last block: the blocks' partials summed by thread
        // (blocks t, t + BLOCK, ...), then the fixed-order block sum; the
        // per-task and per-panel updates one per thread (a one-thread loop of
        // dependent L2 round trips here cost ~20 us per epoch)
        __threadfence();
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        for (unsigned int b = threadIdx.x; b < gridDim.x; b += BLOCK) {
            a0 += __ldcg(part_m + 3 * b + 0);
            a1 += __ldcg(part_m + 3 * b + 1);
            a2 += __ldcg(part_m + 3 * b + 2);
        }
        double nd = 0.0;
        for (int k = threadIdx.x; k < n_tasks; k += BLOCK) nd += __ldcg(p.statuses + k) != 0;
        a0 = block_sum_all(a0, sh);
        a1 = block_sum_all(a1, sh);
        a2 = block_sum_all(a2, sh);
        nd = block_sum_all(nd, sh);
        if (threadIdx.x == 0) {
            p.out->resid_sq = a0;
            p.out->x_sq = a1;
            p.out->err_sq = p.x_true ? a2 : __longlong_as_double(0x7ff8000000000000ll);
            p.out->n_degenerate = (int)nd;
            if (sharded) {
                p.exchange[p.n_meas] = a1;
                p.exchange[p.n_meas + 1] = a2;
            }
            // reference |x| (sharded: the finish writes it from the global norm)
            if ((hdr.flags & 16) && !sharded) *p.guard_ref = fmax(sqrt(a1), 1e-12);
            *p.ticket = 0;
            if (p.res_host) {   // the host's copy (mapped pinned memory)
                EpochOut *ho = reinterpret_cast<EpochOut *>(p.res_host);
                ho->resid_sq = p.out->resid_sq;
                ho->x_sq = a1;
                ho->err_sq = p.out->err_sq;
                ho->n_degenerate = (int)nd;
            }
        }
        if (p.res_host) {   // mu and status per task (written earlier in this launch)
            double *hm = reinterpret_cast<double *>(p.res_host + bct::RES_HEAD_BYTES);
            int32_t *hs = reinterpret_cast<int32_t *>(p.res_host + bct::RES_HEAD_BYTES + 8 * (int64_t)n_tasks);
            for (int k = threadIdx.x; k < n_tasks; k += BLOCK) {
                hm[k] = __ldcg(p.mus + k);
                hs[k] = __ldcg(p.statuses + k);
            }
        }
        if (do_commit)
            for (int lp = threadIdx.x; lp < p.n_panels_owned; lp += BLOCK) p.counts[lp] = 0;
        if (fuse) {
            // phase D's updates (every block has read the old values); one
            // task per panel on this path
            __syncthreads();
            for (int k = threadIdx.x; k < n_tasks; k += BLOCK) {
                const int lp = p.tasks[k].lp;
                if (!do_commit) p.counts[lp] += 1;
                p.zl_on[lp] = 1;
                p.zl_mu[lp] = __ldcg(p.mus + k);
                p.zl_st[lp] = __ldcg(p.statuses + k);
            }
        }
    }
}

// z of every owned panel in (t, ax) form written out (z = ax + mu t, the
// fused tail's value bit for bit) and the panel returned to the stored form;
// blockIdx.y = panel
template <typename V>
__global__ void z_materialize_kernel(const PanelDev *panels, const void *zt_, const double *mu,
                                     const int32_t *st, const int32_t *on, double *z)
{
    using PT = typename std::conditional<narrow_math<V>(), float2, double2>::type;
    const int lp = blockIdx.y;
    if (!on[lp]) return;
    const PT *zt = reinterpret_cast<const PT *>(zt_) + panels[lp].row_off;
    double *zr = z + panels[lp].row_off;
    const double m = mu[lp];
    const int s = st[lp];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < panels[lp].n_rows;
         i += gridDim.x * blockDim.x) {
        const PT q = zt[i];
        zr[i] = z_value((double)q.x, (double)q.y, m, s);
    }
}

}  // namespace

namespace bct {

size_t zt_pair_bytes(int dtype)
{
    return dtype == 0 ? sizeof(double2)
                      : (narrow_math<float>() ? sizeof(float2) : sizeof(double2));
}

cudaError_t z_materialize(int dtype, const PanelDev *panels, int np, const void *zt,
                          const double *mu, const int32_t *st, int32_t *on, double *z,
                          cudaStream_t s)
{
    if (np < 1) return cudaSuccess;
    const dim3 grid(64, np);
    if (dtype == 0)
        z_materialize_kernel<double><<<grid, 256, 0, s>>>(panels, zt, mu, st, on, z);
    else
        z_materialize_kernel<float><<<grid, 256, 0, s>>>(panels, zt, mu, st, on, z);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaMemsetAsync(on, 0, sizeof(int32_t) * np, s);
}

std::string cuda_err(cudaError_t e) { return std::string(cudaGetErrorString(e)); }

// The dynamic shared-memory limit is a per-function, per-device attribute
// shared by every context of the process: raise it (never lower it) to a
// context's need before that context sizes or launches its grid.
static void ensure_smem_attr(int dtype, size_t smem)
{
    static std::mutex mu;
    static size_t set_for[64][2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    size_t &cur = set_for[dev & 63][dtype != 0];
    if (smem <= cur) return;
    cudaFuncSetAttribute(dtype == 0 ? (const void *)epoch_kernel<double>
                                    : (const void *)epoch_kernel<float>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cur = smem;
}

size_t epoch_static_smem(int dtype)
{
    cudaFuncAttributes fa;
    const void *fn = dtype == 0 ? (const void *)epoch_kernel<double> : (const void *)epoch_kernel<float>;
    if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) return 16 * 1024;
    return fa.sharedSizeBytes;
}

int epoch_grid_size(int dtype, int device, size_t smem, int *block)
{
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    ensure_smem_attr(dtype, smem);
    if (dtype == 0)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, epoch_kernel<double>, BLOCK, smem);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, epoch_kernel<float>, BLOCK, smem);
    if (per < 1) per = 1;
    if (per > 1) per = 1;
    *block = BLOCK;
    return sms * per;
}

void launch_epoch(const EpochParams &p, int dtype, int grid, int block, size_t smem,
                  cudaStream_t s, cudaError_t *err)
{
    EpochParams local = p;
    void *args[] = {&local};
    ensure_smem_attr(dtype, smem);
    if (dtype == 0)
        *err = cudaLaunchCooperativeKernel((const void *)epoch_kernel<double>, grid, block, args,
                                           smem, s);
    else
        *err = cudaLaunchCooperativeKernel((const void *)epoch_kernel<float>, grid, block, args,
                                           smem, s);
}

}  // namespace bct
