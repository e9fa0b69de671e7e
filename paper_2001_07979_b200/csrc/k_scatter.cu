// k_scatter.cu -- instances of the production scatter decode kernel
// (scatter.cuh), one per exact degree bound.  Compiled three times
// (MBP_SCATTER_PART = 0/1/2) to split the instantiations across objects.
#include "launch.h"

namespace mbp {

#define MBP_SC(DD) case DD: return launch_coop(decode_scatter_kernel<DD>, A, sm, s);

#if MBP_SCATTER_PART == 0
cudaError_t launch_scatter_small(const ScatterArgs& A, int D, int sm, cudaStream_t s)
{
    switch (D) {
    MBP_SC(3) MBP_SC(4) MBP_SC(5) MBP_SC(6) MBP_SC(7) MBP_SC(8)
    default: return cudaErrorNotSupported;
    }
}
#elif MBP_SCATTER_PART == 1
cudaError_t launch_scatter_mid(const ScatterArgs& A, int D, int sm, cudaStream_t s)
{
    switch (D) {
    MBP_SC(9) MBP_SC(10) MBP_SC(11) MBP_SC(12) MBP_SC(13) MBP_SC(14) MBP_SC(15) MBP_SC(16)
    default: return cudaErrorNotSupported;
    }
}
#else
cudaError_t launch_scatter_large(const ScatterArgs& A, int D, int sm, cudaStream_t s)
{
    switch (D) {
    MBP_SC(20) MBP_SC(24) MBP_SC(32) MBP_SC(48) MBP_SC(64)
    default: return cudaErrorNotSupported;
    }
}
#endif

#undef MBP_SC

}  // namespace mbp
