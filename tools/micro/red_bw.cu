// Microbenchmark: throughput of warp-wide (32 lanes, one line) red.add.f64 /
// red.add.f32 / st.f32 / ld.f32 on pseudo-random lines of a buffer of a given
// size (the L2-resident scatter-accumulate question of the decode design).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE, bool SEQ = false>
__global__ void kern(float* f, double* d, long long nlines, int iters, float* sink) {
    const int lane = threadIdx.x & 31;
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float acc = 0.f;
#pragma unroll 8
    for (int it = 0; it < iters; ++it) {
        const long long line = SEQ ? ((long long)w * iters + it) & (nlines - 1) : hash32(w * 7919u + it * 104729u) & (nlines - 1);
        if (MODE == 0) atomicAdd(d + line * 32 + lane, 1.0);                 // red.f64, 256 B line
        else if (MODE == 1) atomicAdd(f + line * 32 + lane, 1.0f);           // red.f32, 128 B line
        else if (MODE == 2) __stcg(f + line * 32 + lane, (float)it);         // st.f32
        else if (MODE == 3) acc += __ldcg(f + line * 32 + lane);              // ld.f32
        else if (MODE == 4) { long long* q = (long long*)d; atomicAdd((unsigned long long*)(q + line * 32 + lane), 1ull); }
    }
    if (MODE == 3 && acc == 12345.f) sink[0] = acc;
}

int main() {
    const long long sizes[] = {8ll << 20, 32ll << 20, 64ll << 20, 96ll << 20, 256ll << 20, 1024ll << 20};
    char* buf; cudaMalloc(&buf, 1024ll << 20);
    float* sink; cudaMalloc(&sink, 4);
    cudaMemset(buf, 0, 1024ll << 20);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 2048;
    const char* names[] = {"red.f64(256B)", "red.f32(128B)", "st.f32(128B)", "ld.f32(128B)", "red.u64(256B)", "st.f32 seq", "ld.f32 seq", "red.f64 seq"};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 8; ++mode) {
        for (long long S : sizes) {
            const long long linesz = (mode == 0 || mode == 4 || mode == 7) ? 256 : 128;
            const long long nl = S / linesz;
            auto launch = [&] {
                switch (mode) {
                case 0: kern<0><<<blocks, threads>>>((float*)buf, (double*)buf, nl, iters, sink); break;
                case 1: kern<1><<<blocks, threads>>>((float*)buf, (double*)buf, nl, iters, sink); break;
                case 2: kern<2><<<blocks, threads>>>((float*)buf, (double*)buf, nl, iters, sink); break;
                case 3: kern<3><<<blocks, threads>>>((float*)buf, (double*)buf, nl, iters, sink); break;
                case 4: kern<4><<<blocks, threads>>>((float*)buf, (double*)buf, nl, iters, sink); break;
                case 5: kern<2, true><<<blocks, threads>>>((float*)buf, (double*)buf, nl, iters, sink); break;
                case 6: kern<3, true><<<blocks, threads>>>((float*)buf, (double*)buf, nl, iters, sink); break;
                case 7: kern<0, true><<<blocks, threads>>>((float*)buf, (double*)buf, nl, iters, sink); break;
                }
            };
            launch(); cudaDeviceSynchronize();
            cudaEventRecord(a);
            for (int r = 0; r < 5; ++r) launch();
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
            const double ops = (double)blocks * threads / 32 * iters;
            printf("%-14s buf %5lld MB: %8.3f ms  %8.1f GB/s  %7.2f Gline/s\n", names[mode], S >> 20, ms,
                   ops * linesz / ms / 1e6, ops / ms / 1e6);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
