// Whole sweeps of small 2D grids in ONE launch: a thread-block cluster of up
// to 16 CTAs keeps the entire problem in distributed shared memory.
//
// C1 (2D 256^2, N = 3200) is launch/latency-bound: 65,536 cells
// per step are ~5 us of launch overhead and L2 round trips per two-step pass
// however the step is written.  Here CTA r of the cluster owns rows
// [r R, r R + R) of the (axis 1, axis 2) plane and holds, in its shared
// memory, both window levels of its rows (plus one halo row above and below),
// coef and the two face-weight arrays (computed once from gamma with the
// operations of solver.py:89-119) and its rows of the accumulator.  Per step:
//   1. halo rows of u^n from the neighbour CTAs' shared memory (DSMEM,
//      ld.shared::cluster)
//   2. every own cell: stencil (kernels.py:30-44, boundary faces skipped),
//      sources, support gather (u^n) / adjoint injection (solver.py:154-170,
//      gradients.py:237, 268), self-kernel increment (kernels.py:86-102),
//      stability max (solver.py:180-186) — the per-cell operation order of
//      the step kernels, so results are bit-identical
//   3. one cluster barrier (arrive.release / wait.acquire): the new level is
//      visible to the neighbours, and nobody still reads the level the next
//      step overwrites (u^{n+1} is written in place over u^{n-1}; neighbours
//      only ever read u^n rows)
// The window and the accumulator go back to global memory at the end.
#pragma once

#include "common.cuh"
#include "step_kernel.cuh"

namespace wb {

constexpr int CS_THREADS = 1024;
constexpr int CS_MAX_CLUSTER = 16;
constexpr int CS_MAXC = 12;   // cells per thread (R * n2 <= 12 * 1024)

template <typename T> struct ClusterSweepArgs {
    int n1, n2;                 // kernel-space plane (2D grid: rows j, columns k)
    int rows;                   // rows per CTA (R); the last CTAs may own fewer
    int backward;               // 0: n = n_first, n_first+1, ...; 1: n = n_first, n_first-1, ...
    int n_first, n_count;
    long long N;                // steps of the whole sweep (check positions)
    const T* gamma;
    const T* u_prev_in;         // window at entry
    const T* u_cur_in;
    T* u_prev_out;              // window at exit (may alias the inputs: rows are disjoint)
    T* u_cur_out;
    T* acc;
    int accumulate;
    MatScalars<T> mat;
    T cv, cg, inv2dt, inv2dx, sdt;
    int n_src;
    int src_j[MAX_SRC], src_k[MAX_SRC];
    const double* src_amp;      // [n_src][N] fp64 amplitudes (device)
    int sup_mode;               // SUP_NONE / SUP_GATHER / SUP_INJECT
    long long n_sup;
    const unsigned int* sup_mask;
    const int* sup_prefix;
    T* store;                   // [N][n_sup]
    typename FTraits<T>::Bits* maxslots;
    // register-resident engine (cluster_reg.cuh)
    int reg;                    // 1: cluster_reg_kernel
    int pc;                     // its packed pairs per thread row (1 or 2)
    int sup_cap;                // support slots per CTA (even)
    unsigned long long negz2;   // fp32 (-0, -0) addend of the exact packed products
};

template <typename T>
__host__ __device__ constexpr size_t cluster_sweep_smem(int rows, int n2) {
    // U[2][R+2][n2], COEF[R][n2], WJ[R+1][n2], WK[R][n2+1], ACC[R][n2]
    return sizeof(T) * ((size_t)2 * (rows + 2) * n2 + (size_t)rows * n2 + (size_t)(rows + 1) * n2 +
                        (size_t)rows * (n2 + 1) + (size_t)rows * n2) +
           // support bits of the own rows (+1 word of slack each side)
           sizeof(unsigned int) * (((size_t)rows * n2 + 31) / 32 + 2);
}

__device__ __forceinline__ unsigned cs_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cs_nranks() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cs_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared-memory address of `p` in CTA `rank` of the cluster
__device__ __forceinline__ unsigned cs_remote(const void* p, unsigned rank) {
    unsigned local = static_cast<unsigned>(__cvta_generic_to_shared(p)), remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
    return remote;
}
__device__ __forceinline__ float cs_ld_remote(unsigned addr, float) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ double cs_ld_remote(unsigned addr, double) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}

template <typename T, int FLAVOR, bool ACC>
__global__ void __launch_bounds__(CS_THREADS, 1) cluster_sweep_kernel(const ClusterSweepArgs<T> a) {
    using P = Mat<T, FLAVOR, false>;
    using Bits = typename FTraits<T>::Bits;
    extern __shared__ __align__(16) unsigned char cs_smem[];
    const int n1 = a.n1, n2 = a.n2, R = a.rows;
    const unsigned rank = cs_rank(), nranks = cs_nranks();
    const int j0 = (int)rank * R;
    const int own = max(0, min(R, n1 - j0));       // rows owned by this CTA
    T* U0 = reinterpret_cast<T*>(cs_smem);          // [R+2][n2], row 0 = halo above
    T* U1 = U0 + (size_t)(R + 2) * n2;
    T* CO = U1 + (size_t)(R + 2) * n2;              // [R][n2]
    T* WJ = CO + (size_t)R * n2;                    // [R+1][n2]: face (j-1, j) of own row r at r
    T* WK = WJ + (size_t)(R + 1) * n2;              // [R][n2+1]: face (k-1, k) at k
    T* AC = WK + (size_t)R * (n2 + 1);              // [R][n2]
    unsigned int* SB = reinterpret_cast<unsigned int*>(AC + (size_t)R * n2);   // support bits
    __shared__ Bits smax[CS_THREADS / 32];
    const int tid = threadIdx.x;
    const int ncell = own * n2;
    // this thread's cells, fixed for the sweep: c = tid + i * CS_THREADS
    const int nmine = ncell > tid ? (ncell - tid + CS_THREADS - 1) / CS_THREADS : 0;
    int cr[CS_MAXC], ck[CS_MAXC];
#pragma unroll
    for (int i = 0; i < CS_MAXC; ++i) {
        const int c = tid + i * CS_THREADS;
        cr[i] = c / n2;
        ck[i] = c - cr[i] * n2;
    }

    // ---- prologue: material, window, accumulator ----
    auto mg = [&](int j, int k) { return P::m(a.mat, __ldg(a.gamma + (long long)j * n2 + k)); };
    for (int c = tid; c < ncell; c += CS_THREADS) {
        const int r = c / n2, k = c - r * n2, j = j0 + r;
        const long long g = (long long)j * n2 + k;
        const T gam = __ldg(a.gamma + g);
        const T m = P::m(a.mat, gam);
        T kap;
        CO[c] = P::coef(a.mat, gam, kap);
        WJ[(size_t)r * n2 + k] = j > 0 ? P::face(mg(j - 1, k), m) : T(0);
        if (r == own - 1) WJ[(size_t)own * n2 + k] = j + 1 < n1 ? P::face(m, mg(j + 1, k)) : T(0);
        WK[(size_t)r * (n2 + 1) + k] = k > 0 ? P::face(mg(j, k - 1), m) : T(0);
        if (k == n2 - 1) WK[(size_t)r * (n2 + 1) + n2] = T(0);
        U0[(size_t)(r + 1) * n2 + k] = a.u_prev_in[g];
        U1[(size_t)(r + 1) * n2 + k] = a.u_cur_in[g];
        if (ACC) AC[c] = a.acc[g];
    }
    unsigned my_src = 0;
    for (int s = 0; s < a.n_src; ++s)
        if (a.src_j[s] >= j0 && a.src_j[s] < j0 + own) my_src |= 1u << s;
    const bool has_sup = a.sup_mode != SUP_NONE && a.n_sup > 0;
    // support bits of the own cells, local cell index c (bit c of SB)
    const long long gbase = (long long)j0 * n2;
    if (has_sup)
        for (int w = tid; w < (ncell + 31) / 32; w += CS_THREADS) {
            unsigned int v = 0;
            for (int b = 0; b < 32 && w * 32 + b < ncell; ++b) {
                const long long g = gbase + w * 32 + b;
                v |= ((__ldg(a.sup_mask + (g >> 5)) >> (g & 31)) & 1u) << b;
            }
            SB[w] = v;
        }
    cs_cluster_sync();   // every CTA's rows are loaded before the first halo read

    // remote addresses of the neighbours' boundary rows (both level buffers)
    const bool up_nb = rank > 0, dn_nb = rank + 1 < nranks && j0 + own < n1;
    T* pv = U0;   // u^{n-1} (forward) / u^{n+1} (backward): written in place
    T* cu = U1;   // u^n
    Bits lmax = 0;
    for (int it = 0; it < a.n_count; ++it) {
        const long long n = a.backward ? (long long)a.n_first - it : (long long)a.n_first + it;
        // ---- 1: halo rows of u^n ----
        for (int k = tid; k < n2; k += CS_THREADS) {
            if (up_nb)   // upper neighbour's last own row (it owns R rows)
                cu[k] = cs_ld_remote(cs_remote(cu + (size_t)R * n2 + k, rank - 1), T(0));
            if (dn_nb)   // lower neighbour's first own row
                cu[(size_t)(own + 1) * n2 + k] = cs_ld_remote(cs_remote(cu + n2 + k, rank + 1), T(0));
        }
        __syncthreads();
        const bool check = a.backward ? (n % 50 == 0 || n == 1) : (n % 50 == 0 || n == a.N - 1);
        T* srow = has_sup ? a.store + n * a.n_sup : nullptr;
        // ---- 2: the own cells ----
#pragma unroll
        for (int i = 0; i < CS_MAXC; ++i) {
            if (i >= nmine) break;
            const int r = cr[i], k = ck[i], j = j0 + r;
            const int c = tid + i * CS_THREADS;
            const size_t o = (size_t)(r + 1) * n2 + k;
            const T uc = cu[o];
            const T up = pv[o];
            const T uj_m = cu[o - n2], uj_p = cu[o + n2];
            const T uk_m = k > 0 ? cu[o - 1] : uc, uk_p = k < n2 - 1 ? cu[o + 1] : uc;
            T s = uc - uc;
            if (j < n1 - 1) s += (uj_p - uc) * WJ[(size_t)(r + 1) * n2 + k];
            if (j > 0) s -= (uc - uj_m) * WJ[(size_t)r * n2 + k];
            if (k < n2 - 1) s += (uk_p - uc) * WK[(size_t)r * (n2 + 1) + k + 1];
            if (k > 0) s -= (uc - uk_m) * WK[(size_t)r * (n2 + 1) + k];
            T out = ((uc + uc) - up) + CO[c] * s;
            // nodal sources, then the support (solver.py:167-170)
            if (my_src) {
                const long long g = gbase + c;
                for (int q = 0; q < a.n_src; ++q) {
                    if (!((my_src >> q) & 1u) || a.src_j[q] != j || a.src_k[q] != k) continue;
                    const T gam = __ldg(a.gamma + g);
                    T kap;
                    (void)P::coef(a.mat, gam, kap);
                    out = out + P::fc(a.mat, gam, kap) * (T)a.src_amp[(long long)q * a.N + n];
                }
            }
            if (has_sup && ((SB[c >> 5] >> (c & 31)) & 1u)) {
                const long long g = gbase + c;
                const unsigned int w = __ldg(a.sup_mask + (g >> 5));
                const unsigned int bit = (unsigned int)(g & 31);
                const int qi = __ldg(a.sup_prefix + (g >> 5)) + __popc(w & ((1u << bit) - 1u));
                if (a.sup_mode == SUP_GATHER) {
                    srow[qi] = uc;                    // trace entry n = u^n
                } else {
                    const T gam = __ldg(a.gamma + g);
                    T kap;
                    (void)P::coef(a.mat, gam, kap);
                    out = out + P::fc(a.mat, gam, kap) * srow[qi];
                }
            }
            if (ACC) {
                // self-kernel increment; (cv*va)*va is sign-invariant, the
                // absent axis 0 contributes (0*0) + ... = the 2D sum exactly
                const T va = (out - up) * a.inv2dt;
                const T gj = ((j < n1 - 1 ? uj_p : uc) - (j > 0 ? uj_m : uc)) * a.inv2dx;
                const T gk = (uk_p - uk_m) * a.inv2dx;
                AC[c] = AC[c] + a.sdt * ((a.cv * va) * va + a.cg * ((gj * gj) + (gk * gk)));
            }
            pv[o] = out;
            if (check) {
                const Bits b = FTraits<T>::abs_bits(out);
                lmax = b > lmax ? b : lmax;
            }
        }
        if (check) {   // block max -> global slot n
            for (int d = 16; d > 0; d >>= 1) {
                const Bits v = __shfl_xor_sync(0xffffffffu, lmax, d);
                lmax = v > lmax ? v : lmax;
            }
            if ((tid & 31) == 0) smax[tid >> 5] = lmax;
            __syncthreads();
            if (tid < 32) {
                Bits v = tid < CS_THREADS / 32 ? smax[tid] : 0;
                for (int d = 16; d > 0; d >>= 1) {
                    const Bits w = __shfl_xor_sync(0xffffffffu, v, d);
                    v = w > v ? w : v;
                }
                if (tid == 0 && v) atomicMax(a.maxslots + n, v);
            }
            lmax = 0;
        }
        // ---- 3: publish the new level; the old u^{n-1} buffer is free ----
        cs_cluster_sync();
        T* t = pv;
        pv = cu;
        cu = t;
    }

    // ---- epilogue: window (prev, cur) and the accumulator to global ----
    for (int c = tid; c < ncell; c += CS_THREADS) {
        const int r = c / n2, k = c - r * n2;
        const long long g = (long long)(j0 + r) * n2 + k;
        const size_t o = (size_t)(r + 1) * n2 + k;
        a.u_prev_out[g] = pv[o];
        a.u_cur_out[g] = cu[o];
        if (ACC) a.acc[g] = AC[c];
    }
}

}  // namespace wb
