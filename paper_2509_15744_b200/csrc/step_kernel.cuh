// Fused leapfrog step: stencil + nodal injections + support gather/inject +
// self-kernel sensitivity increment + stability max, one HBM pass per step.
//
// What one launch computes (per cell, in the reference's op order):
//   kernels.py:47-69    out = ((u+u) - u_prev) + coef*acc_faces
//   solver.py:154-170   out += fc*T(f)           (source nodes, host order)
//   gradients.py:237    trace[n][s] = u^n        (forward: support gather)
//   gradients.py:268    out += fc*adj_k[n][s]    (backward: support inject)
//   kernels.py:105-128  K += sdt*((cv*va)*va + cg*((g0*g0 + g1*g1) + g2*g2))
//   solver.py:180-186   max|out| (check steps only)
// Material coefficients (coef, face weights, fc) are recomputed from gamma
// with the exact operations of solver.py:89-119, so gamma is the only
// material array streamed from HBM.
//
// Layout: C-order [n0][n1][n2], axis 2 contiguous.  2D grids run as
// (1, n0, n1) and 1D as (1, 1, n0) — the skipped axis contributes no
// stencil term and a +0 gradient term, which leaves every result bit
// unchanged.
//
// Parallelisation: a CTA owns a BY x BX tile of the (axis1, axis2) plane and
// marches a chunk of axis 0.  The centre column lives in a register queue
// (u[i-1], u[i], u[i+1]; m[i], m[i+1]); the current plane of u and m, with a
// one-cell halo, is staged in double-buffered shared memory, so each plane
// costs one __syncthreads.  Output u^{n+1} is written in place over u^{n-1}
// (each cell reads its own u^{n-1} before writing), which is what keeps the
// device footprint at four field buffers: gamma, two levels, accumulator.
#pragma once

#include "common.cuh"

namespace wb {

constexpr int BX = 32;
constexpr int BY = 8;
constexpr int MAX_SRC = 8;

enum SupportMode : int { SUP_NONE = 0, SUP_GATHER = 1, SUP_INJECT = 2 };

template <typename T> struct StepArgs {
    const T* gamma;     // material indicator at dtype T (ghost planes if slab)
    const T* u_prev;    // u^{n-1} (forward) / u^{n+1} (backward)
    const T* u_cur;     // u^n
    T* u_out;           // may alias u_prev
    T* hist_out;        // optional second copy of u_out (full-history recording)
    T* acc;             // kernel accumulator (ACC only)
    int n0, n1, n2;     // local extents (n0 = planes of this slab)
    int i_off;          // global axis-0 index of local plane 0
    int n0g;            // global axis-0 extent
    int chunk;          // axis-0 planes per CTA
    MatScalars<T> mat;
    // kernel-increment scalars, cast to T on the host (kernels.py:149-152)
    T cv, cg, inv2dt, inv2dx, sdt;
    int backward;       // 1: physical window is (out, cur, prev)
    // nodal sources: local flat index (-1 = not owned) and T(value)
    int n_src;
    long long src_flat[MAX_SRC];
    T src_val[MAX_SRC];
    // support (sensors / objective region)
    int sup_mode;
    const unsigned int* sup_mask;   // bit per cell
    const int* sup_prefix;          // set bits before each mask word
    T* trace_row;                   // SUP_GATHER: row n of the [N][n_sup] store
    const T* adj_row;               // SUP_INJECT: row n of the k-scaled store
    // stability max (CHECK only): atomicMax on |out| bit patterns
    typename FTraits<T>::Bits* max_slot;
};

template <typename T>
__device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }

template <typename T, bool ACC, bool CHECK, bool ONE_D>
__global__ void __launch_bounds__(BX * BY)
step_kernel(const StepArgs<T> a) {
    using Tr = FTraits<T>;
    __shared__ T su[2][BY + 2][BX + 2];
    __shared__ T sm[2][BY + 2][BX + 2];
    __shared__ typename Tr::Bits smax[BX * BY / 32];

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int k = blockIdx.x * BX + tx;
    const int j = blockIdx.y * BY + ty;
    const int n1 = a.n1, n2 = a.n2;
    const bool inb = (j < n1) && (k < n2);
    const long long plane = (long long)n1 * n2;
    const int i0 = blockIdx.z * a.chunk;
    const int i1 = min(i0 + a.chunk, a.n0);
    const MatScalars<T>& M = a.mat;

    // halo roles (the 5-point in-plane stencil needs no corners)
    const int hk = (tx == 0) ? k - 1 : ((tx == BX - 1) ? k + 1 : -1);
    const int hj = (ty == 0) ? j - 1 : ((ty == BY - 1) ? j + 1 : -1);
    const bool has_hk = (hk >= 0) && (hk < n2) && (j < n1);
    const bool has_hj = (hj >= 0) && (hj < n1) && (k < n2);
    const int sxk = (tx == 0) ? 0 : BX + 1;   // smem column of the k-halo
    const int syj = (ty == 0) ? 0 : BY + 1;   // smem row of the j-halo
    const long long cofs = (long long)j * n2 + k;
    const long long hkofs = (long long)j * n2 + hk;
    const long long hjofs = (long long)hj * n2 + k;

    // prologue: centre column queue for plane i0
    T u_m1 = T(0), u_0 = T(0), u_p1 = T(0);
    T g_0 = T(1), g_p1 = T(1);
    T m_0 = T(0), wf0_lo = T(0);
    T hu_k = T(0), hg_k = T(1), hu_j = T(0), hg_j = T(1);
    if (inb) {
        const long long c = (long long)i0 * plane + cofs;
        u_0 = ldg(a.u_cur + c);
        g_0 = ldg(a.gamma + c);
        if (i0 + a.i_off > 0) {
            u_m1 = ldg(a.u_cur + c - plane);
            const T g_m1 = ldg(a.gamma + c - plane);
            m_0 = mat_m(M, g_0);
            wf0_lo = Tr::rcp(mat_m(M, g_m1) + m_0);
        } else {
            m_0 = mat_m(M, g_0);
        }
        if (i0 + a.i_off < a.n0g - 1) {
            u_p1 = ldg(a.u_cur + c + plane);
            g_p1 = ldg(a.gamma + c + plane);
        }
    }
    if (has_hk) {
        hu_k = ldg(a.u_cur + (long long)i0 * plane + hkofs);
        hg_k = ldg(a.gamma + (long long)i0 * plane + hkofs);
    }
    if (has_hj) {
        hu_j = ldg(a.u_cur + (long long)i0 * plane + hjofs);
        hg_j = ldg(a.gamma + (long long)i0 * plane + hjofs);
    }

    typename Tr::Bits local_max = 0;

    for (int i = i0; i < i1; ++i) {
        const int gi = i + a.i_off;
        const int buf = i & 1;
        const long long c = (long long)i * plane + cofs;
        // loads for this plane's epilogue and the next plane's queue
        T up = T(0), acc_old = T(0);
        T u_p2 = T(0), g_p2 = T(1);
        T nhu_k = T(0), nhg_k = T(1), nhu_j = T(0), nhg_j = T(1);
        if (inb) {
            up = ldg(a.u_prev + c);
            if (ACC) acc_old = a.acc[c];
            if (gi + 2 < a.n0g && i + 1 < i1) {
                u_p2 = ldg(a.u_cur + c + 2 * plane);
                g_p2 = ldg(a.gamma + c + 2 * plane);
            }
        }
        if (i + 1 < i1) {
            if (has_hk) {
                nhu_k = ldg(a.u_cur + (long long)(i + 1) * plane + hkofs);
                nhg_k = ldg(a.gamma + (long long)(i + 1) * plane + hkofs);
            }
            if (has_hj) {
                nhu_j = ldg(a.u_cur + (long long)(i + 1) * plane + hjofs);
                nhg_j = ldg(a.gamma + (long long)(i + 1) * plane + hjofs);
            }
        }

        // stage plane i (u and m) with its halo
        su[buf][ty + 1][tx + 1] = u_0;
        sm[buf][ty + 1][tx + 1] = m_0;
        if (has_hk) {
            su[buf][ty + 1][sxk] = hu_k;
            sm[buf][ty + 1][sxk] = mat_m(M, hg_k);
        }
        if (has_hj) {
            su[buf][syj][tx + 1] = hu_j;
            sm[buf][syj][tx + 1] = mat_m(M, hg_j);
        }
        __syncthreads();

        if (inb) {
            const bool has_p = gi < a.n0g - 1, has_m = gi > 0;
            const bool jp = j < n1 - 1, jm = j > 0, kp = k < n2 - 1, km = k > 0;
            T m_p1 = T(0), wf0_hi = T(0);
            if (has_p) {
                m_p1 = mat_m(M, g_p1);
                wf0_hi = Tr::rcp(m_0 + m_p1);
            }
            const T u_jp = jp ? su[buf][ty + 2][tx + 1] : u_0;
            const T u_jm = jm ? su[buf][ty][tx + 1] : u_0;
            const T u_kp = kp ? su[buf][ty + 1][tx + 2] : u_0;
            const T u_km = km ? su[buf][ty + 1][tx] : u_0;

            // ---- stencil, kernels.py:56-69 ----
            T accf = u_0 - u_0;
            if (has_p) accf += (u_p1 - u_0) * wf0_hi;
            if (has_m) accf -= (u_0 - u_m1) * wf0_lo;
            if (jp) accf += (u_jp - u_0) * Tr::rcp(m_0 + sm[buf][ty + 2][tx + 1]);
            if (jm) accf -= (u_0 - u_jm) * Tr::rcp(sm[buf][ty][tx + 1] + m_0);
            if (kp) accf += (u_kp - u_0) * Tr::rcp(m_0 + sm[buf][ty + 1][tx + 2]);
            if (km) accf -= (u_0 - u_km) * Tr::rcp(sm[buf][ty + 1][tx] + m_0);
            T kappa;
            const T coef = mat_coef(M, g_0, kappa);
            T out = ((u_0 + u_0) - up) + coef * accf;

            // ---- nodal injections, solver.py:167-170 (source first) ----
            const long long flat = (long long)i * plane + cofs;
            for (int s = 0; s < a.n_src; ++s)
                if (flat == a.src_flat[s]) out = out + mat_fc(M, g_0, kappa) * a.src_val[s];
            if (a.sup_mode != SUP_NONE) {
                const unsigned int w = __ldg(a.sup_mask + (flat >> 5));
                const unsigned int b = (unsigned int)(flat & 31);
                if ((w >> b) & 1u) {
                    const int s = __ldg(a.sup_prefix + (flat >> 5)) + __popc(w & ((1u << b) - 1u));
                    if (a.sup_mode == SUP_GATHER) a.trace_row[s] = u_0;
                    else out = out + mat_fc(M, g_0, kappa) * ldg(a.adj_row + s);
                }
            }

            // ---- self-kernel increment, kernels.py:105-128 ----
            if (ACC) {
                const T va = a.backward ? (up - out) * a.inv2dt : (out - up) * a.inv2dt;
                const T gz = (has_p ? u_p1 : u_0) - (has_m ? u_m1 : u_0);
                const T g0 = gz * a.inv2dx;
                const T g1 = (u_jp - u_jm) * a.inv2dx;
                const T g2 = (u_kp - u_km) * a.inv2dx;
                T inc;
                if (ONE_D) inc = a.sdt * ((a.cv * va) * va + (a.cg * g2) * g2);
                else inc = a.sdt * ((a.cv * va) * va + a.cg * (((g0 * g0) + (g1 * g1)) + (g2 * g2)));
                a.acc[c] = acc_old + inc;
            }
            a.u_out[c] = out;
            if (a.hist_out) a.hist_out[c] = out;
            if (CHECK) {
                const typename Tr::Bits bits = Tr::abs_bits(out);
                local_max = bits > local_max ? bits : local_max;
            }
            // advance the centre queue
            u_m1 = u_0; u_0 = u_p1; u_p1 = u_p2;
            g_0 = g_p1; g_p1 = g_p2;
            m_0 = m_p1; wf0_lo = wf0_hi;
        }
        hu_k = nhu_k; hg_k = nhg_k; hu_j = nhu_j; hg_j = nhg_j;
    }

    if (CHECK) {
        // NaN bit patterns (exponent all ones, mantissa != 0) compare above +inf
        for (int o = 16; o > 0; o >>= 1) {
            typename Tr::Bits v = __shfl_xor_sync(0xffffffffu, local_max, o);
            local_max = v > local_max ? v : local_max;
        }
        const int lane = (ty * BX + tx) & 31, warp = (ty * BX + tx) >> 5;
        if (lane == 0) smax[warp] = local_max;
        __syncthreads();
        if (warp == 0) {
            typename Tr::Bits v = lane < (BX * BY / 32) ? smax[lane] : 0;
            for (int o = 16; o > 0; o >>= 1) {
                typename Tr::Bits w = __shfl_xor_sync(0xffffffffu, v, o);
                v = w > v ? w : v;
            }
            if (lane == 0 && v) atomicMax(a.max_slot, v);
        }
    }
}

}  // namespace wb
