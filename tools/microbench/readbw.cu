// Profiling helper: read-only HBM bandwidth of a streaming kernel on this
// B200 (the denominator question for phases A/B: copy peak vs read peak).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o readbw readbw.cu && ./readbw
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(1024, 1) rd(const float4 *p, long long n, float *out)
{
    float acc = 0.f;
    long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    for (; i < n; i += stride) { float4 v = p[i]; acc += v.x + v.y + v.z + v.w; }
    if (acc == 123.f) out[0] = acc;
}

// bulk-copy ring: one elected thread streams 16 KB chunks into a 4-stage ring
__global__ void __launch_bounds__(128, 1) rd_bulk(const char *p, long long bytes, float *out)
{
    constexpr int CH = 32768, NS = 6;
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) unsigned long long full[NS];
    const int tid = threadIdx.x;
    if (tid == 0)
        for (int s = 0; s < NS; ++s)
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"((unsigned)__cvta_generic_to_shared(&full[s])));
    __syncthreads();
    long long nch = bytes / CH;
    long long c0 = blockIdx.x, cs = gridDim.x;
    auto issue = [&](long long c, int s) {
        unsigned mb = (unsigned)__cvta_generic_to_shared(&full[s]);
        unsigned dst = (unsigned)__cvta_generic_to_shared(sm + s * CH);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(mb), "r"(CH));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(dst), "l"(p + c * CH), "r"(CH), "r"(mb) : "memory");
    };
    int k = 0;
    if (tid == 0)
        for (int s = 0; s < NS && c0 + s * cs < nch; ++s) issue(c0 + s * cs, s);
    float acc = 0.f;
    for (long long c = c0; c < nch; c += cs, ++k) {
        const int s = k % NS;
        const unsigned ph = (k / NS) & 1;
        unsigned mb = (unsigned)__cvta_generic_to_shared(&full[s]);
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                         : "=r"(done) : "r"(mb), "r"(ph));
        const float4 *q = reinterpret_cast<const float4 *>(sm + s * CH);
        for (int i = tid; i < CH / 16; i += blockDim.x) { float4 v = q[i]; acc += v.x + v.y + v.z + v.w; }
        __syncthreads();
        if (tid == 0 && c + NS * cs < nch) issue(c + NS * cs, s);
    }
    if (acc == 123.f) out[0] = acc;
}

int main()
{
    const long long bytes = 8ll << 30;
    char *p; float *o;
    cudaMalloc(&p, bytes); cudaMalloc(&o, 4);
    cudaMemset(p, 0, bytes);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto run = [&](const char *name, auto launch) {
        float best = 1e9;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (r) best = ms < best ? ms : best;
        }
        printf("%-28s %.1f GB/s  (%s)\n", name, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    long long n4 = bytes / 16;
    run("ld 1024thr U=4", [&] { rd<4><<<sms, 1024>>>((const float4 *)p, n4, o); });
    run("ld 1024thr U=8", [&] { rd<8><<<sms, 1024>>>((const float4 *)p, n4, o); });
    run("ld 2x512thr U=8", [&] { rd<8><<<2 * sms, 512>>>((const float4 *)p, n4, o); });
    cudaFuncSetAttribute(rd_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    run("bulk ring 6x32KB 1CTA/SM", [&] { rd_bulk<<<sms, 128, 6 * 32768>>>(p, bytes, o); });
    cudaMemcpy(p, p + bytes / 2, bytes / 2, cudaMemcpyDeviceToDevice);
    run("memcpy d2d (r+w)", [&] { cudaMemcpy(p, p + bytes / 2, bytes / 2, cudaMemcpyDeviceToDevice); });
    return 0;
}
