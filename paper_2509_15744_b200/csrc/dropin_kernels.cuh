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
