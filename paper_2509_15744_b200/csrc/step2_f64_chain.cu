// Two-step (temporal blocking) engine for double, dataflow-chained passes; see launchers.cuh.
#include "step_launch_impl.cuh"

namespace wb {
template void launch_step2_mode<double, T2_CHAIN>(const StepSel&, int, dim3, cudaStream_t,
                                           const Step2Args<double>&, const Tma2Maps&);
template void preload_step2_mode<double, T2_CHAIN>();
}  // namespace wb
