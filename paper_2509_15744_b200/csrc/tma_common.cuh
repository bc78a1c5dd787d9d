// TMA infrastructure shared by the TMA step kernels (step_kernel_tma4.cuh,
// step2_kernel.cuh): halo box geometry, the tensor-map set of a context,
// mbarrier helpers and the 3D bulk-tensor load.
//   * one producer thread per CTA streams per plane boxes into a ring of
//     shared-memory stages with cp.async.bulk.tensor (TMA); completion is
//     tracked by one mbarrier (expect_tx) per stage;
//   * TMA fills out-of-range box elements with zeros; the kernels never read
//     them — neighbours are addressed through clamped (mirrored) offsets
//     fixed at kernel start, and the mirrored boundary terms are exactly +0
//     (step_kernel.cuh header), so results stay bit-identical to the
//     reference.
#pragma once

#include <cuda.h>

#include <type_traits>

#include "common.cuh"
#include "step_kernel.cuh"
#include "step_kernel_v2.cuh"

namespace wb {

constexpr int TH_H = BY + 2;          // halo box height (j0-1 .. j0+8)
// The innermost TMA box coordinate must be 16-byte aligned (measured: an
// offset of -2 floats traps), so the halo box starts HO = 16/sizeof(T) cells
// left of the tile and is PBX + 2*HO wide.
template <typename T> __host__ __device__ constexpr int th_ho() { return 16 / (int)sizeof(T); }
template <typename T> __host__ __device__ constexpr int th_w() { return PBX + 2 * th_ho<T>(); }
constexpr int TH_WMAX = PBX + 8;

struct TmaMaps {
    CUtensorMap u_halo[4];   // level buffers 0..3, (th_w, TH_H, 1) boxes
    CUtensorMap u_ctr[4];    // level buffers 0..3, (PBX, BY, 1) boxes
    CUtensorMap g_halo;      // gamma, (th_w, TH_H, 1)
    CUtensorMap a_ctr;       // accumulator, (PBX, BY, 1)
    int cur, prev;           // buffers holding u^n and u^{n-1}
    int lo;                  // ghost planes below plane 0 (map plane = p + lo)
};

// constant-offset selects keep a descriptor in parameter space
__device__ __forceinline__ const CUtensorMap* pick_map(const CUtensorMap (&m)[4], int i) {
    switch (i) {
        case 1: return &m[1];
        case 2: return &m[2];
        case 3: return &m[3];
        default: return &m[0];
    }
}

template <typename T> struct TmaStage {   // every TMA destination 128-byte aligned
    alignas(128) T U[TH_H][th_w<T>()];
    alignas(128) T G[TH_H][th_w<T>()];
    alignas(128) T P[BY][PBX];
    alignas(128) T A[BY][PBX];
};

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2),
        "r"(smem_addr(bar))
        : "memory");
}

}  // namespace wb
