// Literal per-step drop-ins for waveopt.kernels.apply_step and
// apply_kernel_increment (kernels.py:18-128), taking precomputed face-weight
// and coefficient arrays like the reference does.  One thread per cell; these
// back the per-step C entry points, not the fused sweeps.
#pragma once

#include "common.cuh"

namespace wb {

// shape mapped to 3D (1D -> (1,1,n), 2D -> (1,n0,n1)); each face array is
// indexed with its own extents (n-1 on its axis).  wfX == nullptr: axis absent.
template <typename T>
__global__ void dropin_step_kernel(int n0, int n1, int n2, const T* u_prev, const T* u,
                                   const T* wf0, const T* wf1, const T* wf2, const T* coef,
                                   T* out) {
    const long long n = (long long)n0 * n1 * n2;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(c % n2);
        const int j = (int)((c / n2) % n1);
        const int i = (int)(c / ((long long)n1 * n2));
        const T uc = u[c];
        T acc = uc - uc;
        if (wf0) {
            if (i < n0 - 1) acc += (u[c + (long long)n1 * n2] - uc) * wf0[c];
            if (i > 0) acc -= (uc - u[c - (long long)n1 * n2]) * wf0[c - (long long)n1 * n2];
        }
        if (wf1) {
            const long long c1 = ((long long)i * (n1 - 1) + j) * n2 + k;
            if (j < n1 - 1) acc += (u[c + n2] - uc) * wf1[c1];
            if (j > 0) acc -= (uc - u[c - n2]) * wf1[c1 - n2];
        }
        if (wf2) {
            const long long c2 = ((long long)i * n1 + j) * (n2 - 1) + k;
            if (k < n2 - 1) acc += (u[c + 1] - uc) * wf2[c2];
            if (k > 0) acc -= (uc - u[c - 1]) * wf2[c2 - 1];
        }
        out[c] = ((uc + uc) - u_prev[c]) + coef[c] * acc;
    }
}

// nd = the reference's ndim (1: (cg*ga)*gb ordering, kernels.py:83)
template <typename T>
__global__ void dropin_ki_kernel(int nd, int n0, int n1, int n2, T* acc, const T* ao,
                                 const T* am, const T* an, const T* bo, const T* bm,
                                 const T* bn, T cv, T cg, T inv2dt, T inv2dx, T sdt) {
    const long long n = (long long)n0 * n1 * n2;
    const long long pl = (long long)n1 * n2;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(c % n2);
        const int j = (int)((c / n2) % n1);
        const int i = (int)(c / pl);
        const long long cip = i < n0 - 1 ? c + pl : c, cim = i > 0 ? c - pl : c;
        const long long cjp = j < n1 - 1 ? c + n2 : c, cjm = j > 0 ? c - n2 : c;
        const long long ckp = k < n2 - 1 ? c + 1 : c, ckm = k > 0 ? c - 1 : c;
        const T va = (an[c] - ao[c]) * inv2dt;
        const T vb = (bn[c] - bo[c]) * inv2dt;
        const T ga2 = (am[ckp] - am[ckm]) * inv2dx;
        const T gb2 = (bm[ckp] - bm[ckm]) * inv2dx;
        T inc;
        if (nd == 1) {
            inc = sdt * ((cv * va) * vb + (cg * ga2) * gb2);
        } else {
            const T ga1 = (am[cjp] - am[cjm]) * inv2dx;
            const T gb1 = (bm[cjp] - bm[cjm]) * inv2dx;
            if (nd == 2) {
                inc = sdt * ((cv * va) * vb + cg * ((ga1 * gb1) + (ga2 * gb2)));
            } else {
                const T ga0 = (am[cip] - am[cim]) * inv2dx;
                const T gb0 = (bm[cip] - bm[cim]) * inv2dx;
                inc = sdt * ((cv * va) * vb + cg * (((ga0 * gb0) + (ga1 * gb1)) + (ga2 * gb2)));
            }
        }
        acc[c] = acc[c] + inc;
    }
}

}  // namespace wb

namespace wb {

// One fused step of gradient_reference's adjoint sweep (gradients.py:371-386),
// in the reference's order per cell:
//   out  = ((u+u) - u_prev) + coef*faces(u)      kernels.py:47-69 (no source),
//          material from gamma as solver.py:89-119 (skipped boundary faces)
//   out += fc * adj[n]  on support nodes          gradients.py:374-375
//   acc += dt*((cv*va)*vb + cg*(ga . gb))         kernels.py:72-128 with a = the
//          forward history (n-1, n, n+1), b = the adjoint (out, u, u_prev)
//   max |out| on check steps                      solver.py:180-186
// It replaces a generic step launch plus a separate mixed kernel-increment
// launch per step (one pass over the adjoint and history levels instead of
// two; half the launches of the launch-bound small grids).
template <typename T> struct RefAdjArgs {
    int nd, n0, n1, n2;                 // reference ndim; kernel-space extents
    const T* gamma;
    const T* u_prev;                    // adjoint u^{n+1}
    const T* u_cur;                     // adjoint u^n
    T* u_out;                           // adjoint u^{n-1}
    const T* h_old;                     // forward history n-1, n, n+1
    const T* h_mid;
    const T* h_new;
    T* acc;
    MatScalars<T> mat;
    T cv, cg, inv2dt, inv2dx, sdt;
    const unsigned int* sup_mask;       // support bit per cell
    const int* sup_prefix;
    const T* adj_row;                   // row n of the (unscaled) adjoint store
    int check;
    typename FTraits<T>::Bits* max_slot;
};

template <typename T, int FLAVOR>
__global__ void __launch_bounds__(256) ref_adjoint_step_kernel(const RefAdjArgs<T> a) {
    using P = Mat<T, FLAVOR, false>;
    using Bits = typename FTraits<T>::Bits;
    const long long pl = (long long)a.n1 * a.n2, n = pl * a.n0;
    Bits lmax = 0;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(c % a.n2);
        const int j = (int)((c / a.n2) % a.n1);
        const int i = (int)(c / pl);
        const T g = __ldg(a.gamma + c);
        const T mc = P::m(a.mat, g);
        const T uc = a.u_cur[c];
        T s = uc - uc;
        if (a.n0 > 1) {
            if (i < a.n0 - 1) s += (a.u_cur[c + pl] - uc) * P::face(mc, P::m(a.mat, __ldg(a.gamma + c + pl)));
            if (i > 0) s -= (uc - a.u_cur[c - pl]) * P::face(P::m(a.mat, __ldg(a.gamma + c - pl)), mc);
        }
        if (a.n1 > 1) {
            if (j < a.n1 - 1) s += (a.u_cur[c + a.n2] - uc) * P::face(mc, P::m(a.mat, __ldg(a.gamma + c + a.n2)));
            if (j > 0) s -= (uc - a.u_cur[c - a.n2]) * P::face(P::m(a.mat, __ldg(a.gamma + c - a.n2)), mc);
        }
        if (k < a.n2 - 1) s += (a.u_cur[c + 1] - uc) * P::face(mc, P::m(a.mat, __ldg(a.gamma + c + 1)));
        if (k > 0) s -= (uc - a.u_cur[c - 1]) * P::face(P::m(a.mat, __ldg(a.gamma + c - 1)), mc);
        T kap;
        const T coef = P::coef(a.mat, g, kap);
        const T up = a.u_prev[c];
        T out = ((uc + uc) - up) + coef * s;
        if (a.sup_mask) {
            const unsigned int w = __ldg(a.sup_mask + (c >> 5));
            const unsigned int bit = (unsigned int)(c & 31);
            if ((w >> bit) & 1u) {
                const int q = __ldg(a.sup_prefix + (c >> 5)) + __popc(w & ((1u << bit) - 1u));
                out = out + P::fc(a.mat, g, kap) * a.adj_row[q];
            }
        }
        a.u_out[c] = out;
        // mixed increment: a = history, b = adjoint (old = out, mid = cur, new = prev)
        const long long cip = i < a.n0 - 1 ? c + pl : c, cim = i > 0 ? c - pl : c;
        const long long cjp = j < a.n1 - 1 ? c + a.n2 : c, cjm = j > 0 ? c - a.n2 : c;
        const long long ckp = k < a.n2 - 1 ? c + 1 : c, ckm = k > 0 ? c - 1 : c;
        const T va = (a.h_new[c] - a.h_old[c]) * a.inv2dt;
        const T vb = (up - out) * a.inv2dt;
        const T ga2 = (a.h_mid[ckp] - a.h_mid[ckm]) * a.inv2dx;
        const T gb2 = (a.u_cur[ckp] - a.u_cur[ckm]) * a.inv2dx;
        T inc;
        if (a.nd == 1) {
            inc = a.sdt * ((a.cv * va) * vb + (a.cg * ga2) * gb2);
        } else {
            const T ga1 = (a.h_mid[cjp] - a.h_mid[cjm]) * a.inv2dx;
            const T gb1 = (a.u_cur[cjp] - a.u_cur[cjm]) * a.inv2dx;
            if (a.nd == 2) {
                inc = a.sdt * ((a.cv * va) * vb + a.cg * ((ga1 * gb1) + (ga2 * gb2)));
            } else {
                const T ga0 = (a.h_mid[cip] - a.h_mid[cim]) * a.inv2dx;
                const T gb0 = (a.u_cur[cip] - a.u_cur[cim]) * a.inv2dx;
                inc = a.sdt * ((a.cv * va) * vb +
                               a.cg * (((ga0 * gb0) + (ga1 * gb1)) + (ga2 * gb2)));
            }
        }
        a.acc[c] = a.acc[c] + inc;
        if (a.check) {
            const Bits b = FTraits<T>::abs_bits(out);
            lmax = b > lmax ? b : lmax;
        }
    }
    if (a.check) {
        for (int o = 16; o > 0; o >>= 1) {
            const Bits v = __shfl_xor_sync(0xffffffffu, lmax, o);
            lmax = v > lmax ? v : lmax;
        }
        if ((threadIdx.x & 31) == 0 && lmax) atomicMax(a.max_slot, lmax);
    }
}

}  // namespace wb
