// k_explicit.cu -- instances of the explicit-message decode kernel
// (decode.cuh): fp64 parity mode, damping, isolated-per-matrix, and fp32
// runs that keep every message readable (MBP_KEEP_STATE / MBP_EXPLICIT_MESSAGES).
#include "launch.h"

namespace mbp {

template <class Real, int D>
static cudaError_t variant(const DecodeArgs<Real>& A, bool damp, bool iso, int sm, cudaStream_t s)
{
    if (damp && iso) return launch_coop(decode_kernel<Real, D, true, true>, A, sm, s);
    if (damp) return launch_coop(decode_kernel<Real, D, true, false>, A, sm, s);
    if (iso) return launch_coop(decode_kernel<Real, D, false, true>, A, sm, s);
    return launch_coop(decode_kernel<Real, D, false, false>, A, sm, s);
}

template <class Real>
static cudaError_t dispatch(const DecodeArgs<Real>& A, int D, bool damp, bool iso, int sm, cudaStream_t s)
{
    switch (D) {
    case 8: return variant<Real, 8>(A, damp, iso, sm, s);
    case 16: return variant<Real, 16>(A, damp, iso, sm, s);
    case 32: return variant<Real, 32>(A, damp, iso, sm, s);
    case 64: return variant<Real, 64>(A, damp, iso, sm, s);
    default: return cudaErrorNotSupported;
    }
}

// fp64 instances are split over two objects (MBP_EXPLICIT_F64 = 1: D <= 16,
// 2: D >= 32) so the slowest unit of the parallel build halves
#if defined(MBP_EXPLICIT_F64) && MBP_EXPLICIT_F64 == 1
cudaError_t launch_explicit_f64(const DecodeArgs<double>& A, int D, bool damp, bool iso, int sm, cudaStream_t s)
{
    switch (D) {
    case 8: return variant<double, 8>(A, damp, iso, sm, s);
    case 16: return variant<double, 16>(A, damp, iso, sm, s);
    default: return launch_explicit_f64_wide(A, D, damp, iso, sm, s);
    }
}
#elif defined(MBP_EXPLICIT_F64) && MBP_EXPLICIT_F64 == 2
cudaError_t launch_explicit_f64_wide(const DecodeArgs<double>& A, int D, bool damp, bool iso, int sm, cudaStream_t s)
{
    switch (D) {
    case 32: return variant<double, 32>(A, damp, iso, sm, s);
    case 64: return variant<double, 64>(A, damp, iso, sm, s);
    default: return cudaErrorNotSupported;
    }
}
#else
cudaError_t launch_explicit_f32(const DecodeArgs<float>& A, int D, bool damp, bool iso, int sm, cudaStream_t s)
{
    return dispatch<float>(A, D, damp, iso, sm, s);
}
#endif

}  // namespace mbp
