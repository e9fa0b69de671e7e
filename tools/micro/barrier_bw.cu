// Microbenchmark: cost of a grid-wide barrier in a cooperative persistent
// kernel at the decode kernel's shape (4 blocks x 256 threads per SM), for the
// barrier the kernels use (kernels.cuh grid_barrier: sc fences + relaxed
// polling with nanosleep) and two variants: acquire/release atomics without
// the full fences, and the same without the sleep in the polling loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_bw barrier_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2001_07979_b200/csrc/kernels.cuh"

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v)
{
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void red_release(unsigned* p, unsigned v)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

template <int SLEEP>
__device__ __forceinline__ void barrier_acqrel(unsigned* bar)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = ld_acquire(bar + 1);
        if (atom_add_acqrel(bar, 1u) == gridDim.x - 1) {
            bar[0] = 0;
            red_release(bar + 1, 1u);
        } else {
            while (ld_acquire(bar + 1) == gen)
                if (SLEEP) __nanosleep(SLEEP);
        }
    }
    __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(256, 4) kern(unsigned* bar, int iters, unsigned* sink)
{
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) mbp::grid_barrier(bar);
        else if (MODE == 1) barrier_acqrel<32>(bar);
        else barrier_acqrel<0>(bar);
        acc += threadIdx.x;
    }
    if (acc == 12345u) sink[0] = acc;
}

int main()
{
    int sm = 0;
    cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
    unsigned *bar, *sink;
    cudaMalloc(&bar, 64);
    cudaMalloc(&sink, 64);
    const char* names[] = {"grid_barrier (kernels.cuh)", "acq_rel + nanosleep(32)", "acq_rel, spin"};
    for (int blocks_per_sm : {1, 4}) {
        for (int mode = 0; mode < 3; ++mode) {
            int iters = 2000;
            void* args[] = {&bar, &iters, &sink};
            const void* k = mode == 0 ? (const void*)kern<0> : mode == 1 ? (const void*)kern<1> : (const void*)kern<2>;
            cudaMemset(bar, 0, 64);
            cudaLaunchCooperativeKernel(k, dim3(sm * blocks_per_sm), dim3(256), args, 0, 0);   // warm-up
            cudaDeviceSynchronize();
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel(k, dim3(sm * blocks_per_sm), dim3(256), args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            cudaError_t e = cudaGetLastError();
            printf("%3d blocks  %-28s %.2f us per barrier  (%s)\n", sm * blocks_per_sm, names[mode], 1e3f * ms / iters,
                   cudaGetErrorString(e));
        }
    }
    return 0;
}
