// k_scatter.cu -- instances of the production scatter decode kernel
// (scatter.cuh), one per exact degree bound.  Compiled three times
// (MBP_SCATTER_PART = 0/1/2) to split the instantiations across objects.
// Degree bounds <= 16 also get the hot instance (sweeps 1..kHotSweeps).
#include "launch.h"

namespace mbp {

#define MBP_SC(DD) case DD: return launch_scatter<DD, false>(A, sm, s);
#define MBP_SCH(DD) case DD: return hot ? launch_scatter<DD, true>(A, sm, s) : launch_scatter<DD, false>(A, sm, s);

#if MBP_SCATTER_PART == 0
cudaError_t launch_scatter_small(const ScatterArgs& A, int D, bool hot, int sm, cudaStream_t s)
{
    switch (D) {
    MBP_SCH(3) MBP_SCH(4) MBP_SCH(5) MBP_SCH(6) MBP_SCH(7) MBP_SCH(8)
    default: return cudaErrorNotSupported;
    }
}
#elif MBP_SCATTER_PART == 1
cudaError_t launch_scatter_mid(const ScatterArgs& A, int D, bool hot, int sm, cudaStream_t s)
{
    switch (D) {
    MBP_SCH(9) MBP_SCH(10) MBP_SCH(11) MBP_SCH(12) MBP_SCH(13) MBP_SCH(14) MBP_SCH(15) MBP_SCH(16)
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
#undef MBP_SCH

}  // namespace mbp
