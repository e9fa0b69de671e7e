// launch.h -- kernel launchers shared between mbp.cu (host/C ABI) and the
// kernel translation units (one per group of template instantiations, so
// the library builds in parallel).
#pragma once

#include "scatter.cuh"

namespace mbp {

// Cooperative launch of one persistent decode kernel instance sized to the
// device (resident blocks per SM x sm_count).  Return cudaErrorNotSupported
// when no instance exists for the requested degree bound.
cudaError_t launch_explicit_f32(const DecodeArgs<float>& A, int D, bool damp, bool iso, int sm_count,
                                cudaStream_t s);
cudaError_t launch_explicit_f64(const DecodeArgs<double>& A, int D, bool damp, bool iso, int sm_count,
                                cudaStream_t s);
cudaError_t launch_explicit_f64_wide(const DecodeArgs<double>& A, int D, bool damp, bool iso, int sm_count,
                                     cudaStream_t s);   // D >= 32
// hot = true: the hot instance of decode_scatter_kernel (D <= 16 only)
cudaError_t launch_scatter_small(const ScatterArgs& A, int D, bool hot, int sm_count, cudaStream_t s);   // D 3..8
cudaError_t launch_scatter_mid(const ScatterArgs& A, int D, bool hot, int sm_count, cudaStream_t s);     // D 9..16
cudaError_t launch_scatter_large(const ScatterArgs& A, int D, int sm_count, cudaStream_t s);             // D 20..64

// smem: dynamic shared memory per block (opted in above 48 KB)
template <class Kern, class Args>
cudaError_t launch_coop(Kern kern, const Args& A, int sm_count, cudaStream_t s, size_t smem = 0)
{
    cudaError_t err;
    if (smem > 48 * 1024 &&
        (err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
        return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDecodeThreads, smem);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    void* args[] = {(void*)&A};
    return cudaLaunchCooperativeKernel((const void*)kern, dim3(per_sm * sm_count), dim3(kDecodeThreads), args, smem, s);
}

template <int D, bool HOT>
cudaError_t launch_scatter(const ScatterArgs& A, int sm_count, cudaStream_t s)
{
    return launch_coop(decode_scatter_kernel<D, HOT>, A, sm_count, s, ScatterSmem<D>::bytes);
}

}  // namespace mbp
