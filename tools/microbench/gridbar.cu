// Grid-barrier cost on the epoch kernel's launch shape (one 1024-thread CTA
// per SM, cooperative launch): N back-to-back barriers, us per barrier, for
// the epoch kernel's release-add / acquire-poll barrier, the fenced variant
// and cooperative_groups::this_grid().sync().
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 gridbar.cu -o gridbar && ./gridbar
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ void bar_relacq(unsigned int *bar)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int nb = gridDim.x;
        unsigned int inc = (blockIdx.x == 0) ? (0x80000000u - (nb - 1)) : 1u;
        unsigned int old, cur;
        asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(bar), "r"(inc) : "memory");
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];\n" : "=r"(cur) : "l"(bar) : "memory");
        } while (((old ^ cur) & 0x80000000u) == 0);
    }
    __syncthreads();
}

__device__ __forceinline__ void bar_fenced(unsigned int *bar)
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

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(unsigned int *bar, int n, double *sink)
{
    double acc = threadIdx.x;
    for (int i = 0; i < n; ++i) {
        if (MODE == 0) bar_relacq(bar);
        else if (MODE == 1) bar_fenced(bar);
        else cg::this_grid().sync();
        acc += 1.0;
    }
    if (acc < 0) *sink = acc;
}

int main()
{
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    unsigned int *bar;
    double *sink;
    cudaMalloc(&bar, 4);
    cudaMalloc(&sink, 8);
    cudaMemset(bar, 0, 4);
    const char *names[3] = {"release-add / acquire-poll (epoch kernel)", "fenced atomicAdd / volatile poll",
                            "cooperative_groups grid.sync"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int n : {1, 2001}) {
            void *f = mode == 0 ? (void *)k<0> : mode == 1 ? (void *)k<1> : (void *)k<2>;
            void *args[] = {&bar, &n, &sink};
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaLaunchCooperativeKernel(f, sms, 1024, args, 0, 0);   // warm-up
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel(f, sms, 1024, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (n > 1) printf("%-45s %7.3f us per barrier (%d CTAs x 1024)\n", names[mode], 1e3 * ms / n, sms);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
