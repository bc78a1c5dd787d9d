// Single-step engines (scalar, pair, TMA, TMA 2x2) for float; see launchers.cuh.
#include "step_launch_impl.cuh"

namespace wb {
template void launch_step_engine<float>(int, const StepSel&, dim3, dim3, cudaStream_t,
                                     const StepArgs<float>&, const TmaMaps&);
template void preload_step_kernels<float>();
}  // namespace wb
