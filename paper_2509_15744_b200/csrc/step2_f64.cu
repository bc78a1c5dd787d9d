// Two-step (temporal blocking) engine for double, base feature level (32-bit offsets, whole-grid dependency) and the material pass; see launchers.cuh.
#include "step_launch_impl.cuh"

namespace wb {
template void launch_step2_mode<double, T2_BASE>(const StepSel&, int, dim3, cudaStream_t,
                                           const Step2Args<double>&, const Tma2Maps&);
template void preload_step2_mode<double, T2_BASE>();
template void launch_material4<double>(int, cudaStream_t, const double*, const MatScalars<double>&, int,
                                     int, int, double*);
template void preload_material4_kernels<double>();
}  // namespace wb
