// TMA + tcgen05 split-KV LongFlow decode step (G >= 2): see DESIGN.md "Kernels".
#include "lf_internal.h"

namespace lf {

bool tc_supported(int, int) { return false; }

Plan tc_plan(int, int, int, int, int, int) {
    Plan pl;
    pl.kernel = LF_KERNEL_TCGEN05;
    pl.splits = -1;
    pl.chunk = 0;
    pl.smem = 0;
    return pl;
}

cudaError_t tc_launch(const StepParams&, const Plan&, cudaStream_t) { return cudaErrorNotSupported; }

}  // namespace lf
