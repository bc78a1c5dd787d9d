// Two-step (temporal blocking) engine for double; see launchers.cuh.
#include "step_launch_impl.cuh"

namespace wb {
template void launch_step2_engine<double>(const StepSel&, int, dim3, cudaStream_t,
                                      const Step2Args<double>&, const Tma2Maps&);
template void launch_material4<double>(int, cudaStream_t, const double*, const MatScalars<double>&, int,
                                     int, int, double*);
template void preload_step2_kernels<double>();
}  // namespace wb
