// sampler.cu -- device-side block selection (bct_sample_epoch).
//
// Replays BlockScheduler.epoch_plan (sampling.py:140-152) from the host's
// numpy variates: the column-block visit order (rng.choice) and the
// exponential stream (rng.exponential, scope_n values per visit, in visit
// order) are drawn on the host, so the RNG stream stays numpy's; the device
// computes everything that follows from them, one CTA per visit:
//
//   weights   raw = table.values[:, j]; importance -> raw; random/mixed ->
//             raw + theta*(max(raw_live) - raw) on raw > 0 (sampling.py:63-77),
//             rounded op by op like numpy (no contraction)
//   race      keys = E / w over the live blocks in id order, stable argsort,
//             first `draws` ids (sampling.py:90-105)
//   groups    chunks of group_size in draw order (sampling.py:108-109)
//   beta      b * sum(values[ids, j]) / totals[j] with numpy's pairwise
//             summation (solvers.py:173-177)
//
// and writes the task masks, visit masks and betas straight into the epoch's
// device task array (the host fills the structural fields), ORs the drawn
// blocks into the epoch mask and stores the drawn ids for the host record.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace {

constexpr int SBLOCK = 256;   // threads per visit; row blocks are strided over them

// numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src) over
// values[ids[q]*stride + j], q in [0, n): sequential below 8 terms, eight
// interleaved partial sums up to 128, halves (multiple of 8) above.
__device__ double np_pairwise(const int *ids, int n, const double *values, int stride, int j)
{
    if (n < 8) {
        double res = 0.0;
        for (int q = 0; q < n; ++q) res = __dadd_rn(res, values[(int64_t)ids[q] * stride + j]);
        return res;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = values[(int64_t)ids[u] * stride + j];
        int q = 8;
        for (; q < n - (n % 8); q += 8)
#pragma unroll
            for (int u = 0; u < 8; ++u) r[u] = __dadd_rn(r[u], values[(int64_t)ids[q + u] * stride + j]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; q < n; ++q) res = __dadd_rn(res, values[(int64_t)ids[q] * stride + j]);
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(np_pairwise(ids, n2, values, stride, j),
                     np_pairwise(ids + n2, n - n2, values, stride, j));
}

// shared memory per visit CTA: keys, live flags, live positions, drawn ids
// (m each) and the visit mask
inline size_t sampler_smem(int m)
{
    return (size_t)m * (8 + 4 + 4 + 4) + 8 * (size_t)mask_words(m);
}

__global__ void __launch_bounds__(SBLOCK) sample_k(bct::SamplerParams p)
{
    extern __shared__ double smem_d[];
    const int m = p.m, mw = p.mw;
    double *key_s = smem_d;
    int *live_s = reinterpret_cast<int *>(key_s + m);
    int *pos_s = live_s + m;
    int *ids_s = pos_s + m;
    unsigned long long *vmask = reinterpret_cast<unsigned long long *>(
        smem_d + ((size_t)m * 20 + 7) / 8);
    __shared__ double top_s;
    const int v = blockIdx.x;
    const bct::SampleVisit V = p.visits[v];
    if (threadIdx.x == 0) top_s = 0.0;
    for (int w = threadIdx.x; w < mw; w += SBLOCK) vmask[w] = 0ull;
    for (int i = threadIdx.x; i < m; i += SBLOCK) {
        const double raw = p.values[(int64_t)i * p.n_panels + V.j];
        live_s[i] = raw > 0.0 ? 1 : 0;
    }
    __syncthreads();
    // max over live raw (order-free), positions of live blocks (exclusive count)
    for (int i = threadIdx.x; i < m; i += SBLOCK) {
        const double raw = p.values[(int64_t)i * p.n_panels + V.j];
        // doubles > 0 order like their bit patterns
        if (live_s[i] && p.strategy != 0)
            atomicMax(reinterpret_cast<unsigned long long *>(&top_s), __double_as_longlong(raw));
        int pos = 0;
        for (int q = 0; q < i; ++q) pos += live_s[q];
        pos_s[i] = pos;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += SBLOCK) {
        const double raw = p.values[(int64_t)i * p.n_panels + V.j];
        double w = raw;
        if (p.strategy != 0 && live_s[i])
            w = __dadd_rn(raw, __dmul_rn(p.theta, __dsub_rn(top_s, raw)));
        key_s[i] = live_s[i] ? p.exp[V.var_off + pos_s[i]] / w : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += SBLOCK) {
        if (!live_s[i]) continue;
        const double k = key_s[i];
        int rank = 0;
        for (int q = 0; q < m; ++q)
            if (live_s[q] && (key_s[q] < k || (key_s[q] == k && q < i))) ++rank;
        if (rank < V.draws) {
            ids_s[rank] = i;
            p.plan_ids[V.id_off + rank] = i;
            atomicOr(&vmask[i >> 6], 1ull << (i & 63));
        }
    }
    __syncthreads();
    for (int w = threadIdx.x; w < mw; w += SBLOCK)
        if (vmask[w]) atomicOr(reinterpret_cast<unsigned long long *>(p.masks + w), vmask[w]);
    if (V.task_base < 0) return;   // another rank's column block: record only
    const int n_groups = (V.draws + p.group_size - 1) / p.group_size;
    for (int t = threadIdx.x; t < n_groups; t += SBLOCK) {
        const int q0 = t * p.group_size;
        const int n = min(p.group_size, V.draws - q0);
        const int64_t k = V.task_base + t;
        TaskDev &T = p.tasks[k];
        // the host uploaded zeroed masks for this task
        uint64_t *mk = p.masks + task_mask_off(k, mw);
        uint64_t *vk = p.masks + visit_mask_off(k, mw);
        for (int q = 0; q < n; ++q) mk[ids_s[q0 + q] >> 6] |= 1ull << (ids_s[q0 + q] & 63);
        for (int w = 0; w < mw; ++w) vk[w] = vmask[w];
        const double s = np_pairwise(ids_s + q0, n, p.values, p.n_panels, V.j);
        T.beta = __dmul_rn(p.b, s) / p.totals[V.j];
    }
}

}  // namespace

namespace bct {

void launch_sampler(const SamplerParams &p, int n_visits, cudaStream_t s, cudaError_t *err)
{
    const size_t smem = sampler_smem(p.m);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(sample_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (n_visits > 0) sample_k<<<n_visits, SBLOCK, smem, s>>>(p);
    *err = cudaGetLastError();
}

}  // namespace bct
