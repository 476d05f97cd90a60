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

constexpr int SBLOCK = 256;   // >= BCT_MAX_M

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

__global__ void __launch_bounds__(SBLOCK) sample_k(bct::SamplerParams p)
{
    __shared__ double key_s[SBLOCK];
    __shared__ int live_s[SBLOCK];
    __shared__ int ids_s[SBLOCK];
    __shared__ double top_s;
    __shared__ unsigned long long vmask[BCT_MASKW];
    const int v = blockIdx.x;
    const bct::SampleVisit V = p.visits[v];
    const int i = threadIdx.x;
    const int m = p.m;
    const double raw = i < m ? p.values[(int64_t)i * p.n_panels + V.j] : 0.0;
    const int live = raw > 0.0 ? 1 : 0;
    live_s[i] = live;
    if (i == 0) top_s = 0.0;
    if (i < BCT_MASKW) vmask[i] = 0ull;
    __syncthreads();
    // max over live raw (order-free), positions of live blocks (exclusive count)
    if (live && p.strategy != 0) {
        // doubles > 0 order like their bit patterns
        atomicMax(reinterpret_cast<unsigned long long *>(&top_s), __double_as_longlong(raw));
    }
    int pos = 0;
    for (int q = 0; q < i; ++q) pos += live_s[q];
    __syncthreads();
    double w = raw;
    if (p.strategy != 0 && live)
        w = __dadd_rn(raw, __dmul_rn(p.theta, __dsub_rn(top_s, raw)));
    key_s[i] = live ? p.exp[V.var_off + pos] / w : 0.0;
    __syncthreads();
    if (live) {
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
    if (i < BCT_MASKW && vmask[i])
        atomicOr(reinterpret_cast<unsigned long long *>(&p.hdr->epoch_mask[i]), vmask[i]);
    if (V.task_base < 0) return;   // another rank's column block: record only
    const int n_groups = (V.draws + p.group_size - 1) / p.group_size;
    for (int t = i; t < n_groups; t += SBLOCK) {
        const int q0 = t * p.group_size;
        const int n = min(p.group_size, V.draws - q0);
        TaskDev &T = p.tasks[V.task_base + t];
        unsigned long long mk[BCT_MASKW] = {0ull, 0ull, 0ull, 0ull};
        for (int q = 0; q < n; ++q) mk[ids_s[q0 + q] >> 6] |= 1ull << (ids_s[q0 + q] & 63);
        for (int w4 = 0; w4 < BCT_MASKW; ++w4) {
            T.mask[w4] = mk[w4];
            T.visit_mask[w4] = vmask[w4];
        }
        const double s = np_pairwise(ids_s + q0, n, p.values, p.n_panels, V.j);
        T.beta = __dmul_rn(p.b, s) / p.totals[V.j];
    }
}

}  // namespace

namespace bct {

void launch_sampler(const SamplerParams &p, int n_visits, cudaStream_t s, cudaError_t *err)
{
    if (n_visits > 0) sample_k<<<n_visits, SBLOCK, 0, s>>>(p);
    *err = cudaGetLastError();
}

}  // namespace bct
