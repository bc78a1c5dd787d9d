// Template bodies of launch_step_engine / launch_step2_engine (launchers.cuh),
// included by the per-dtype translation units.
#pragma once

#include <atomic>

#include "launchers.cuh"
#include "step_kernel_tma4.cuh"
#include "step_kernel_v2.cuh"

namespace wb {

// Opt a kernel into more than 48 KB of dynamic shared memory, once per
// kernel and device (the attribute is per device; one process may drive
// several GPUs, e.g. slabs on peer devices).
template <auto Kernel>
void smem_opt_in(size_t bytes) {
    static std::atomic<unsigned long long> done{0};   // one flag set per kernel
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_relaxed) & bit) return;
    cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    done.fetch_or(bit);
}

// Launch with programmatic stream serialisation (WB_T2_PDL): the kernel may
// start while the previous kernel of the stream drains; it executes
// griddepcontrol.wait before touching global memory.  Measured: 2D 256^2
// superposed gradient 22.2 -> 26.7 Gcell-upd/s (launch-latency-bound), 256^3
// unchanged.
template <typename Kernel, typename A, typename M>
void launch_pdl(Kernel kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s, const A& a,
                const M& maps) {
    if (t_no_pdl) {
        kernel<<<grid, block, smem, s>>>(a, maps);
        return;
    }
#if WB_T2_PDL
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, a, maps);
#else
    kernel<<<grid, block, smem, s>>>(a, maps);
#endif
}

template <typename T, int FL, bool FAST, bool ACC, bool CHK, int SUP>
void go_step(int engine, dim3 grid, dim3 block, cudaStream_t s, const StepArgs<T>& a,
             const TmaMaps& maps) {
    if (engine == ENGINE_TMA4) {   // 128 threads, 2x2 cells each, unrolled stages
        const size_t sm = tma4_smem_bytes<T>();
        smem_opt_in<step_kernel_tma4<T, FL, FAST, ACC, CHK, SUP>>(sm);
        launch_pdl(step_kernel_tma4<T, FL, FAST, ACC, CHK, SUP>, grid, dim3(32, 4, 1), sm, s, a,
                   maps);
    } else if (SUP == SUP_NONE) {   // pair / scalar kernels read a.sup_mode at run time
        if (engine == ENGINE_PAIR)
            step_kernel_pair<T, FL, FAST, ACC, CHK><<<grid, block, 0, s>>>(a);
        else
            step_kernel<T, FL, FAST, ACC, CHK><<<grid, block, 0, s>>>(a);
    }
}

template <typename T, int FL, bool FAST, bool ACC, bool CHK>
void go_step_sup(int engine, int sup, dim3 grid, dim3 block, cudaStream_t s,
                 const StepArgs<T>& a, const TmaMaps& maps) {
    if (engine != ENGINE_TMA4) sup = SUP_NONE;
    if (sup == SUP_GATHER) go_step<T, FL, FAST, ACC, CHK, SUP_GATHER>(engine, grid, block, s, a, maps);
    else if (sup == SUP_INJECT) go_step<T, FL, FAST, ACC, CHK, SUP_INJECT>(engine, grid, block, s, a, maps);
    else go_step<T, FL, FAST, ACC, CHK, SUP_NONE>(engine, grid, block, s, a, maps);
}

template <typename T, int FL, bool FAST>
void go_step_ac(int engine, const StepSel& k, dim3 grid, dim3 block, cudaStream_t s,
                const StepArgs<T>& a, const TmaMaps& maps) {
    if (k.acc) {
        if (k.check) go_step_sup<T, FL, FAST, true, true>(engine, k.sup, grid, block, s, a, maps);
        else go_step_sup<T, FL, FAST, true, false>(engine, k.sup, grid, block, s, a, maps);
    } else {
        if (k.check) go_step_sup<T, FL, FAST, false, true>(engine, k.sup, grid, block, s, a, maps);
        else go_step_sup<T, FL, FAST, false, false>(engine, k.sup, grid, block, s, a, maps);
    }
}

template <typename T>
void launch_step_engine(int engine, const StepSel& k, dim3 grid, dim3 block, cudaStream_t s,
                        const StepArgs<T>& a, const TmaMaps& maps) {
    if (k.flavor == RHO_SCALED) {
        if (k.fast) go_step_ac<T, RHO_SCALED, true>(engine, k, grid, block, s, a, maps);
        else go_step_ac<T, RHO_SCALED, false>(engine, k, grid, block, s, a, maps);
    } else {
        if (k.fast) go_step_ac<T, ACOUSTIC, true>(engine, k, grid, block, s, a, maps);
        else go_step_ac<T, ACOUSTIC, false>(engine, k, grid, block, s, a, maps);
    }
}

template <typename T, typename G, int FL, bool ACC, int SUP, int MODE>
void go_step2(dim3 grid, cudaStream_t s, const Step2Args<T>& a, const Tma2Maps& maps) {
    const size_t sm = step2_smem_bytes<T, G>();
    smem_opt_in<step2_kernel_tma<T, G, FL, ACC, SUP, MODE>>(sm);
    launch_pdl(step2_kernel_tma<T, G, FL, ACC, SUP, MODE>, grid, dim3(G::TX, G::TY, 1), sm, s, a,
               maps);
}

template <typename T, typename G, int FL, bool ACC, int MODE>
void go_step2_sup(int sup, dim3 grid, cudaStream_t s, const Step2Args<T>& a, const Tma2Maps& maps) {
    if (sup == SUP_GATHER) go_step2<T, G, FL, ACC, SUP_GATHER, MODE>(grid, s, a, maps);
    else if (sup == SUP_INJECT) go_step2<T, G, FL, ACC, SUP_INJECT, MODE>(grid, s, a, maps);
    else go_step2<T, G, FL, ACC, SUP_NONE, MODE>(grid, s, a, maps);
}

template <typename T, typename G, int MODE>
void go_step2_geo(const StepSel& k, dim3 grid, cudaStream_t s, const Step2Args<T>& a,
                  const Tma2Maps& maps) {
    if (k.flavor == RHO_SCALED) {
        if (k.acc) go_step2_sup<T, G, RHO_SCALED, true, MODE>(k.sup, grid, s, a, maps);
        else go_step2_sup<T, G, RHO_SCALED, false, MODE>(k.sup, grid, s, a, maps);
    } else {
        if (k.acc) go_step2_sup<T, G, ACOUSTIC, true, MODE>(k.sup, grid, s, a, maps);
        else go_step2_sup<T, G, ACOUSTIC, false, MODE>(k.sup, grid, s, a, maps);
    }
}

template <typename T, int MODE>
void launch_step2_mode(const StepSel& k, int geo, dim3 grid, cudaStream_t s,
                       const Step2Args<T>& a, const Tma2Maps& maps) {
    if (geo == GEO_TALL) go_step2_geo<T, GeoTall, MODE>(k, grid, s, a, maps);
    else go_step2_geo<T, GeoWide, MODE>(k, grid, s, a, maps);
}

template <typename T>
void launch_material4(int flavor, cudaStream_t s, const T* gamma, const MatScalars<T>& M, int n0,
                      int n1, int n2, T* out) {
    const size_t f = (size_t)n0 * n1 * n2;
    if (flavor == RHO_SCALED)
        material4_kernel<T, RHO_SCALED><<<592, 256, 0, s>>>(gamma, M, n0, n1, n2, out, out + f,
                                                           out + 2 * f, out + 3 * f);
    else
        material4_kernel<T, ACOUSTIC><<<592, 256, 0, s>>>(gamma, M, n0, n1, n2, out, out + f,
                                                         out + 2 * f, out + 3 * f);
}

template <typename K>
void load_kernel(K kernel) {
    cudaFuncAttributes attr;
    cudaFuncGetAttributes(&attr, kernel);
}

template <typename T, int FL, bool FAST, bool ACC, bool CHK>
void preload_step_variant() {
    load_kernel(step_kernel_tma4<T, FL, FAST, ACC, CHK, SUP_NONE>);
    load_kernel(step_kernel_tma4<T, FL, FAST, ACC, CHK, SUP_GATHER>);
    load_kernel(step_kernel_tma4<T, FL, FAST, ACC, CHK, SUP_INJECT>);
    smem_opt_in<step_kernel_tma4<T, FL, FAST, ACC, CHK, SUP_NONE>>(tma4_smem_bytes<T>());
    smem_opt_in<step_kernel_tma4<T, FL, FAST, ACC, CHK, SUP_GATHER>>(tma4_smem_bytes<T>());
    smem_opt_in<step_kernel_tma4<T, FL, FAST, ACC, CHK, SUP_INJECT>>(tma4_smem_bytes<T>());
    load_kernel(step_kernel_pair<T, FL, FAST, ACC, CHK>);
    load_kernel(step_kernel<T, FL, FAST, ACC, CHK>);
}

template <typename T, int FL, bool FAST>
void preload_step_fl() {
    preload_step_variant<T, FL, FAST, false, false>();
    preload_step_variant<T, FL, FAST, false, true>();
    preload_step_variant<T, FL, FAST, true, false>();
    preload_step_variant<T, FL, FAST, true, true>();
}

template <typename T>
void preload_step_kernels() {
    preload_step_fl<T, RHO_SCALED, false>();
    preload_step_fl<T, RHO_SCALED, true>();
    preload_step_fl<T, ACOUSTIC, false>();
    preload_step_fl<T, ACOUSTIC, true>();
}

template <typename T, typename G, int FL, bool ACC, int MODE>
void preload_step2_variant() {
    const size_t sm = step2_smem_bytes<T, G>();
    load_kernel(step2_kernel_tma<T, G, FL, ACC, SUP_NONE, MODE>);
    load_kernel(step2_kernel_tma<T, G, FL, ACC, SUP_GATHER, MODE>);
    load_kernel(step2_kernel_tma<T, G, FL, ACC, SUP_INJECT, MODE>);
    smem_opt_in<step2_kernel_tma<T, G, FL, ACC, SUP_NONE, MODE>>(sm);
    smem_opt_in<step2_kernel_tma<T, G, FL, ACC, SUP_GATHER, MODE>>(sm);
    smem_opt_in<step2_kernel_tma<T, G, FL, ACC, SUP_INJECT, MODE>>(sm);
}

template <typename T, int MODE>
void preload_step2_mode() {
    preload_step2_variant<T, GeoWide, RHO_SCALED, false, MODE>();
    preload_step2_variant<T, GeoWide, RHO_SCALED, true, MODE>();
    preload_step2_variant<T, GeoWide, ACOUSTIC, false, MODE>();
    preload_step2_variant<T, GeoWide, ACOUSTIC, true, MODE>();
    preload_step2_variant<T, GeoTall, RHO_SCALED, false, MODE>();
    preload_step2_variant<T, GeoTall, RHO_SCALED, true, MODE>();
    preload_step2_variant<T, GeoTall, ACOUSTIC, false, MODE>();
    preload_step2_variant<T, GeoTall, ACOUSTIC, true, MODE>();
}

template <typename T>
void preload_material4_kernels() {
    load_kernel(material4_kernel<T, RHO_SCALED>);
    load_kernel(material4_kernel<T, ACOUSTIC>);
}

}  // namespace wb
