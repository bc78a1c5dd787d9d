// Standalone TMA probe (dev tool): checks a 3D halo-box TMA load with the same
// descriptor recipe and PTX helpers as csrc/step_kernel_tma.cuh.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2509_15744_b200/csrc \
//        profiles/tma_probe.cu -o /tmp/tma_probe && /tmp/tma_probe <variant>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "step_kernel_tma.cuh"

using namespace wb;

struct Maps {
    CUtensorMap m[2];
    int sel;
};

__global__ void probe2(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, float* out,
                       int variant) {
    extern __shared__ __align__(128) unsigned char dyn[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<unsigned long long>(dyn) + 127ull) & ~127ull);
    float* box = reinterpret_cast<float*>(base);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(base + 4096);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (variant == 10) {          // arrive/expect only, no TMA
            mbar_expect_tx(bar, 0);
        } else if (variant == 20) {   // plain bulk copy (no tensor map)
            mbar_expect_tx(bar, 2048);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                ::"r"(smem_addr(box)), "l"(reinterpret_cast<unsigned long long>(out + 1024)),
                "r"(2048), "r"(smem_addr(bar)) : "memory");
        } else if (variant == 21) {   // in-bounds box at the origin
            mbar_expect_tx(bar, 68 * 10 * 4);
            tma_load_3d(box, &map, 0, 0, 0, bar);
        } else if (variant >= 30 && variant < 40) {   // coordinate sweep
            const int cs[][2] = {{-4, -1}, {-2, 0}, {2, 0}, {0, -1}, {4, 0}, {-8, 0}};
            mbar_expect_tx(bar, 68 * 10 * 4);
            tma_load_3d(box, &map, cs[variant - 30][0], cs[variant - 30][1], 0, bar);
        } else if (variant == 22) {   // shared::cta destination form
            mbar_expect_tx(bar, 68 * 10 * 4);
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(box)),
                "l"(reinterpret_cast<unsigned long long>(&map)), "r"(-2), "r"(-1), "r"(0),
                "r"(smem_addr(bar)) : "memory");
        } else {
            const CUtensorMap* mp = variant == 11 ? &map : gmap;
            mbar_expect_tx(bar, 68 * 10 * 4);
            tma_load_3d(box, mp, -2, -1, 0, bar);
        }
    }
    mbar_wait(bar, 0);
    __syncthreads();
    for (int i = threadIdx.x; i < 680; i += blockDim.x) out[i] = variant == 10 ? 0.f : box[i];
}

__global__ void probe(const __grid_constant__ Maps maps, float* out, int variant) {
    extern __shared__ __align__(128) unsigned char dyn[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<unsigned long long>(dyn) + 127ull) & ~127ull);
    float* box = reinterpret_cast<float*>(base);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(base + 4096);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (variant >= 1) {
        if (threadIdx.x == 0) {
            const CUtensorMap* mp = maps.sel ? &maps.m[1] : &maps.m[0];
            if (variant >= 3) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar, 68 * 10 * 4);
            tma_load_3d(box, mp, -2, -1, 0, bar);
        }
        if (variant >= 2) mbar_wait(bar, 0);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 680; i += blockDim.x) out[i] = variant >= 2 ? box[i] : 0.f;
}

int main(int argc, char** argv) {
    const int variant = argc > 1 ? atoi(argv[1]) : 3;
    const int n0 = 4, n1 = 16, n2 = 64;
    std::vector<float> h(n0 * n1 * n2);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float *d = nullptr, *out = nullptr;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&out, 4096 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    Maps maps{};
    const cuuint64_t dims[3] = {(cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)n0};
    const cuuint64_t strides[2] = {(cuuint64_t)n2 * 4, (cuuint64_t)n1 * n2 * 4};
    const cuuint32_t boxd[3] = {68, 10, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    for (int b = 0; b < 2; ++b) {
        CUresult r = enc(&maps.m[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, boxd,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("encode %d -> %d\n", b, (int)r);
    }
    maps.sel = 1;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    CUtensorMap* gmap = nullptr;
    cudaMalloc(&gmap, sizeof(CUtensorMap));
    cudaMemcpy(gmap, &maps.m[0], sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    if (variant >= 10) probe2<<<1, 128, 8192>>>(maps.m[0], gmap, out, variant);
    else probe<<<1, 128, 8192>>>(maps, out, variant);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", variant, cudaGetErrorString(e));
    std::vector<float> o(680);
    cudaMemcpy(o.data(), out, 680 * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 10; ++r)
        for (int c = 0; c < 68; ++c) {
            const int j = r - 1, k = c - 2;
            const float want = (j >= 0 && j < n1 && k >= 0 && k < n2) ? h[j * n2 + k] : 0.f;
            if ((variant >= 2 && variant != 10) && o[r * 68 + c] != want) ++bad;
        }
    printf("mismatches %d\n", bad);
    return 0;
}
