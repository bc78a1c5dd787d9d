// Two-step (temporal blocking) engine for float, base feature level (32-bit offsets, whole-grid dependency) and the material pass; see launchers.cuh.
#include "step_launch_impl.cuh"

namespace wb {
template void launch_step2_mode<float, T2_BASE>(const StepSel&, int, dim3, cudaStream_t,
                                           const Step2Args<float>&, const Tma2Maps&);
template void preload_step2_mode<float, T2_BASE>();
template void launch_material4<float>(int, cudaStream_t, const float*, const MatScalars<float>&, int,
                                     int, int, float*);
template void preload_material4_kernels<float>();
}  // namespace wb
