// Cluster-resident whole-sweep engine for small 2D grids (cluster_sweep.cuh).
#include "cluster_reg.cuh"
#include "launchers.cuh"

namespace wb {

template <typename T, int FL, bool ACC>
static cudaError_t go_cluster(const ClusterSweepArgs<T>& a, int cl, size_t smem, cudaStream_t s,
                              bool probe) {
    const bool full = a.n2 % (2 * a.pc) == 0;   // whole packed pairs in every thread row
    auto kernel = !a.reg       ? cluster_sweep_kernel<T, FL, ACC>
                  : a.pc == 2 ? (full ? cluster_reg_kernel<T, FL, ACC, 2, true>
                                      : cluster_reg_kernel<T, FL, ACC, 2, false>)
                              : (full ? cluster_reg_kernel<T, FL, ACC, 1, true>
                                      : cluster_reg_kernel<T, FL, ACC, 1, false>);
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cl, 1, 1);
    const int nthr = cr_txn(a.n2, a.pc) * (a.rows / 2);
    cfg.blockDim = dim3(a.reg ? (nthr + 31) / 32 * 32 : CS_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cl;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    if (probe) {   // can the device hold one such cluster at all?
        int n = 0;
        e = cudaOccupancyMaxActiveClusters(&n, kernel, &cfg);
        return e != cudaSuccess ? e : (n > 0 ? cudaSuccess : cudaErrorInvalidConfiguration);
    }
    return cudaLaunchKernelEx(&cfg, kernel, a);
}

template <typename T>
cudaError_t launch_cluster_sweep(int flavor, bool acc, const ClusterSweepArgs<T>& a, int cl,
                                 cudaStream_t s, bool probe) {
    const size_t smem = a.reg ? cluster_reg_smem<T>(a.rows, a.n2, a.sup_cap, a.pc)
                              : cluster_sweep_smem<T>(a.rows, a.n2);
    if (flavor == RHO_SCALED)
        return acc ? go_cluster<T, RHO_SCALED, true>(a, cl, smem, s, probe)
                   : go_cluster<T, RHO_SCALED, false>(a, cl, smem, s, probe);
    return acc ? go_cluster<T, ACOUSTIC, true>(a, cl, smem, s, probe)
               : go_cluster<T, ACOUSTIC, false>(a, cl, smem, s, probe);
}

template cudaError_t launch_cluster_sweep<float>(int, bool, const ClusterSweepArgs<float>&, int,
                                                 cudaStream_t, bool);
template cudaError_t launch_cluster_sweep<double>(int, bool, const ClusterSweepArgs<double>&, int,
                                                  cudaStream_t, bool);
}  // namespace wb
