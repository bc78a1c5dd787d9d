// K time steps per launch on 2D grids (temporal tiling in shared memory).
//
// C1 / C3-2D (256^2 and 512^2) are latency-bound: a whole step of
// 65-262 K cells is a few microseconds of launch and L2 round trip, whatever
// the per-cell cost.  Here a CTA owns a TX x TY tile and loads the tile plus
// a ring of K cells (u^{n-1}, u^n and gamma; the material of the region is
// derived once with the operations of solver.py:89-119), then advances the
// window K steps in shared memory: step s computes the tile plus a ring of
// K-1-s cells (the ring shrinks by one per step: every value it needs is
// already in shared memory), writing u^{n+1} in place over u^{n-1}.  Own
// cells gather the support (u^n), accumulate the self-kernel and feed the
// stability max; sources and the backward adjoint forces are injected on the
// whole computed region (the recomputed ring must reproduce the neighbours'
// values bit for bit).  The own cells' last two levels go to two further
// level buffers (neighbouring CTAs still read this launch's inputs), so the
// window rotates through four buffers like the two-step passes.
// Per-cell operation order: that of the step kernels (kernels.py:30-44 with
// skipped boundary faces, solver.py:167-170, kernels.py:86-102).
#pragma once

#include "common.cuh"
#include "step_kernel.cuh"

namespace wb {

constexpr int TL_TX = 32, TL_TY = 16, TL_THREADS = 256;
constexpr int TL_MAXK = 8;

template <typename T> struct Tile2DArgs {
    int n1, n2;                        // 2D grid (kernel space (1, n1, n2)): rows j, columns k
    int backward;
    int K;                             // steps of this launch (<= TL_MAXK)
    int n_first;                       // steps n_first, n_first +- 1, ...
    long long N;
    const T* gamma;
    const T* u_prev;                   // window at entry
    const T* u_cur;
    T* o_prev;                         // window at exit (own cells), other buffers
    T* o_cur;
    T* acc;
    MatScalars<T> mat;
    T cv, cg, inv2dt, inv2dx, sdt;
    int n_src;
    int src_j[MAX_SRC], src_k[MAX_SRC];
    T src_val[TL_MAXK][MAX_SRC];       // source values of the K steps
    int sup_mode;
    long long n_sup;
    const unsigned int* sup_mask;
    const int* sup_prefix;
    T* store;                          // [N][n_sup]
    typename FTraits<T>::Bits* maxslots;
};

template <typename T, int K>
__host__ __device__ constexpr size_t tile2d_smem() {
    // U0, U1, CO, WJ, WK over the region (TX + 2K) x (TY + 2K)
    return sizeof(T) * 5 * (size_t)(TL_TX + 2 * K) * (TL_TY + 2 * K);
}

template <typename T, int FLAVOR, bool ACC, int K>
__global__ void __launch_bounds__(TL_THREADS) tile2d_kernel(const __grid_constant__ Tile2DArgs<T> a) {
    using P = Mat<T, FLAVOR, false>;
    using Bits = typename FTraits<T>::Bits;
    constexpr int RX = TL_TX + 2 * K, RY = TL_TY + 2 * K, RC = RX * RY;
    extern __shared__ __align__(16) unsigned char tl_smem[];
    T* U0 = reinterpret_cast<T*>(tl_smem);
    T* U1 = U0 + RC;
    T* CO = U1 + RC;
    T* WJ = CO + RC;     // face (row-1, row) of region cell
    T* WK = WJ + RC;     // face (col-1, col)
    const int tid = threadIdx.x;
    const int n1 = a.n1, n2 = a.n2;
    const int k0 = blockIdx.x * TL_TX - K, j0 = blockIdx.y * TL_TY - K;   // region origin
#if WB_T2_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    // ---- prologue: levels and material of the region (clamped reads; cells
    // outside the grid are never computed) ----
    auto gidx = [&](int j, int k) { return (long long)min(max(j, 0), n1 - 1) * n2 + min(max(k, 0), n2 - 1); };
    auto mat_m = [&](int j, int k) { return P::m(a.mat, __ldg(a.gamma + gidx(j, k))); };
    for (int c = tid; c < RC; c += TL_THREADS) {
        const int r = c / RX, q = c - r * RX, j = j0 + r, k = k0 + q;
        const long long g = gidx(j, k);
        U0[c] = a.u_prev[g];
        U1[c] = a.u_cur[g];
        const T gam = __ldg(a.gamma + g);
        const T m = P::m(a.mat, gam);
        T kap;
        CO[c] = P::coef(a.mat, gam, kap);
        WJ[c] = (j > 0 && j < n1) ? P::face(mat_m(j - 1, k), m) : T(0);
        WK[c] = (k > 0 && k < n2) ? P::face(mat_m(j, k - 1), m) : T(0);
    }
    unsigned my_src = 0;
    for (int s = 0; s < a.n_src; ++s)
        if (a.src_j[s] >= j0 + 1 && a.src_j[s] < j0 + RY - 1 && a.src_k[s] >= k0 + 1 &&
            a.src_k[s] < k0 + RX - 1)
            my_src |= 1u << s;
    const bool has_sup = a.sup_mode != SUP_NONE && a.n_sup > 0;
    __syncthreads();

    T* pv = U0;
    T* cu = U1;
    // own cells' accumulator, in shared memory: the thread visiting an own
    // cell changes from step to step (the computed region shrinks)
    __shared__ T AC[TL_TY][TL_TX];
    if (ACC) {
        for (int c = tid; c < TL_TX * TL_TY; c += TL_THREADS) {
            const int r = c / TL_TX, q = c - r * TL_TX;
            const int j = j0 + K + r, k = k0 + K + q;
            AC[r][q] = (j < n1 && k < n2) ? a.acc[(long long)j * n2 + k] : T(0);
        }
    }
    __syncthreads();

#pragma unroll 1
    for (int s = 0; s < a.K; ++s) {
        const long long n = a.backward ? (long long)a.n_first - s : (long long)a.n_first + s;
        const bool check = a.backward ? (n % 50 == 0 || n == 1) : (n % 50 == 0 || n == a.N - 1);
        const int ring = a.K - 1 - s;                        // cells computed beyond the tile
        const int cx0 = K - ring, cy0 = K - ring;            // computed region in the frame
        const int cw = TL_TX + 2 * ring, ch = TL_TY + 2 * ring;
        T* srow = has_sup ? a.store + n * a.n_sup : nullptr;
        Bits lmax = 0;
        for (int c = tid; c < cw * ch; c += TL_THREADS) {
            const int rr = c / cw, qq = c - rr * cw;
            const int r = cy0 + rr, q = cx0 + qq;
            const int j = j0 + r, k = k0 + q;
            if (j < 0 || j >= n1 || k < 0 || k >= n2) continue;
            const int o = r * RX + q;
            const T uc = cu[o];
            const T up = pv[o];
            T sum = uc - uc;
            if (j < n1 - 1) sum += (cu[o + RX] - uc) * WJ[o + RX];
            if (j > 0) sum -= (uc - cu[o - RX]) * WJ[o];
            if (k < n2 - 1) sum += (cu[o + 1] - uc) * WK[o + 1];
            if (k > 0) sum -= (uc - cu[o - 1]) * WK[o];
            T out = ((uc + uc) - up) + CO[o] * sum;
            const bool own = r >= K && r < K + TL_TY && q >= K && q < K + TL_TX;
            const long long g = (long long)j * n2 + k;
            // nodal sources, then the support (solver.py:167-170)
            if (my_src) {
                for (int p = 0; p < a.n_src; ++p) {
                    if (!((my_src >> p) & 1u) || a.src_j[p] != j || a.src_k[p] != k) continue;
                    const T gam = __ldg(a.gamma + g);
                    T kap;
                    (void)P::coef(a.mat, gam, kap);
                    out = out + P::fc(a.mat, gam, kap) * a.src_val[s][p];
                }
            }
            if (has_sup) {
                const unsigned int w = __ldg(a.sup_mask + (g >> 5));
                const unsigned int bit = (unsigned int)(g & 31);
                if ((w >> bit) & 1u) {
                    const int qi = __ldg(a.sup_prefix + (g >> 5)) + __popc(w & ((1u << bit) - 1u));
                    if (a.sup_mode == SUP_GATHER) {
                        if (own) srow[qi] = uc;               // trace entry n = u^n
                    } else {
                        const T gam = __ldg(a.gamma + g);
                        T kap;
                        (void)P::coef(a.mat, gam, kap);
                        out = out + P::fc(a.mat, gam, kap) * srow[qi];
                    }
                }
            }
            if (own) {
                if (ACC) {   // self-kernel increment (sign-invariant (cv*va)*va)
                    const T va = (out - up) * a.inv2dt;
                    const T gj = (cu[j < n1 - 1 ? o + RX : o] - cu[j > 0 ? o - RX : o]) * a.inv2dx;
                    const T gk = (cu[k < n2 - 1 ? o + 1 : o] - cu[k > 0 ? o - 1 : o]) * a.inv2dx;
                    T& av = AC[r - K][q - K];
                    av = av + a.sdt * ((a.cv * va) * va + a.cg * ((gj * gj) + (gk * gk)));
                }
                if (check) {
                    const Bits b = FTraits<T>::abs_bits(out);
                    lmax = b > lmax ? b : lmax;
                }
            }
            pv[o] = out;
        }
        if (check) {
            for (int d = 16; d > 0; d >>= 1) {
                const Bits v = __shfl_xor_sync(0xffffffffu, lmax, d);
                lmax = v > lmax ? v : lmax;
            }
            if ((tid & 31) == 0 && lmax) atomicMax(a.maxslots + n, lmax);
        }
        __syncthreads();
        T* t = pv;
        pv = cu;
        cu = t;
    }
    // ---- own cells' last two levels and accumulator ----
    for (int c = tid; c < TL_TX * TL_TY; c += TL_THREADS) {
        const int r = c / TL_TX, q = c - r * TL_TX;
        const int j = j0 + K + r, k = k0 + K + q;
        if (j >= n1 || k >= n2) continue;
        const long long g = (long long)j * n2 + k;
        const int o = (r + K) * RX + q + K;
        a.o_prev[g] = pv[o];
        a.o_cur[g] = cu[o];
        if (ACC) a.acc[g] = AC[r][q];
    }
}

}  // namespace wb
