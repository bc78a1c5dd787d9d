// Host-side launchers of the sweep step kernels, one translation unit per
// kernel family and dtype (step_f32.cu, step_f64.cu, step2_f32.cu,
// step2_f64.cu) so the library builds in parallel.  capi.cu picks the
// engine and fills the argument blocks; these functions only map the runtime
// selection onto the template instantiation and launch it on the stream.
#pragma once

#include <cuda_runtime.h>

#include "cluster_reg.cuh"
#include "step2_kernel.cuh"
#include "step_kernel.cuh"
#include "tma_common.cuh"

namespace wb {

// single-step engines
enum StepEngine : int { ENGINE_SCALAR = 0, ENGINE_PAIR = 1, ENGINE_TMA4 = 3 };

struct StepSel {
    int flavor;   // RHO_SCALED / ACOUSTIC
    bool fast;    // verified fast division
    bool acc;     // kernel increment
    bool check;   // stability max
    int sup;      // SUP_NONE / SUP_GATHER / SUP_INJECT (TMA engines)
};

// Plain launches instead of programmatic dependent launch on this thread
// (set by the C ABI around launches that stream memory operations separate:
// peer-store slabs; defined in capi.cu).
extern thread_local bool t_no_pdl;

template <typename T>
void launch_step_engine(int engine, const StepSel& k, dim3 grid, dim3 block, cudaStream_t s,
                        const StepArgs<T>& a, const TmaMaps& maps);

// two-step pass (no divisions on the dense path; checks are runtime flags)
// geometry: GEO_WIDE (64 x 8 tiles) or GEO_TALL (32 x 16 tiles)
enum Step2Geo : int { GEO_NONE = 0, GEO_WIDE = 1, GEO_TALL = 2 };
// one translation unit per (dtype, T2Mode) instantiates launch_step2_mode
template <typename T, int MODE>
void launch_step2_mode(const StepSel& k, int geo, dim3 grid, cudaStream_t s,
                       const Step2Args<T>& a, const Tma2Maps& maps);
template <typename T, int MODE> void preload_step2_mode();

// mode: T2Mode (step2_kernel.cuh) — the feature level the launch needs
template <typename T>
inline void launch_step2_engine(const StepSel& k, int geo, int mode, dim3 grid, cudaStream_t s,
                                const Step2Args<T>& a, const Tma2Maps& maps) {
    if (mode == T2_FULL) launch_step2_mode<T, T2_FULL>(k, geo, grid, s, a, maps);
    else if (mode == T2_CHAIN) launch_step2_mode<T, T2_CHAIN>(k, geo, grid, s, a, maps);
    else launch_step2_mode<T, T2_BASE>(k, geo, grid, s, a, maps);
}

// coef | +k | +j | +i face arrays (4 consecutive fields at out) of a material
template <typename T>
void launch_material4(int flavor, cudaStream_t s, const T* gamma, const MatScalars<T>& M, int n0,
                      int n1, int n2, T* out);

// Load every step / two-step / material kernel instantiation now.  With the
// CUDA runtime's lazy module loading (the CUDA 12 default) the first launch
// of a kernel loads it, which synchronises the context: while a peer-store
// slab's stream waits on a neighbour's flag that only a later-enqueued launch
// of this process will set, such a load would wait forever.  The peer-store
// setup (wo_slab_peers) therefore loads them all up front.
template <typename T> void preload_step_kernels();

// whole sweep of a small 2D grid in one cluster launch (cluster_sweep.cuh);
// probe = only check that the device can hold the cluster
template <typename T>
cudaError_t launch_cluster_sweep(int flavor, bool acc, const ClusterSweepArgs<T>& a, int cl,
                                 cudaStream_t s, bool probe);
template <typename T> void preload_material4_kernels();
template <typename T>
inline void preload_step2_kernels() {
    preload_step2_mode<T, T2_BASE>();
    preload_step2_mode<T, T2_CHAIN>();
    preload_step2_mode<T, T2_FULL>();
    preload_material4_kernels<T>();
}


}  // namespace wb
