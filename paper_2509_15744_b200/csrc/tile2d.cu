// K-steps-per-launch engine for 2D grids (tile2d_kernel.cuh).
#include "launchers.cuh"
#include "tile2d_kernel.cuh"

namespace wb {

template <typename T, int FL, bool ACC>
static cudaError_t go_tile2d(const Tile2DArgs<T>& a, cudaStream_t s) {
    constexpr int K = TL_MAXK;
    auto kernel = tile2d_kernel<T, FL, ACC, K>;
    const size_t smem = tile2d_smem<T, K>();
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const dim3 grid((a.n2 + TL_TX - 1) / TL_TX, (a.n1 + TL_TY - 1) / TL_TY, 1);
#if WB_T2_PDL
    if (!t_no_pdl) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(TL_THREADS, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr{};
        attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr.val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kernel, a);
    }
#endif
    kernel<<<grid, TL_THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_tile2d(int flavor, bool acc, const Tile2DArgs<T>& a, cudaStream_t s) {
    if (flavor == RHO_SCALED)
        return acc ? go_tile2d<T, RHO_SCALED, true>(a, s) : go_tile2d<T, RHO_SCALED, false>(a, s);
    return acc ? go_tile2d<T, ACOUSTIC, true>(a, s) : go_tile2d<T, ACOUSTIC, false>(a, s);
}

template cudaError_t launch_tile2d<float>(int, bool, const Tile2DArgs<float>&, cudaStream_t);
template cudaError_t launch_tile2d<double>(int, bool, const Tile2DArgs<double>&, cudaStream_t);
}  // namespace wb
