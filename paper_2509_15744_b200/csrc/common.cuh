// Shared device helpers for the waveb200 sweep kernels.
//
// Arithmetic contract (parity with the reference's Numba kernels,
// /root/reference/pkg/src/waveopt/kernels.py): the whole library is compiled
// with -fmad=false -prec-div=true -ftz=false, so every + - * / below is one
// IEEE-754 round-to-nearest operation in the run dtype, in source order.
// Divisions and reciprocals are correctly rounded: the _rn intrinsics, or the
// verified branch-free sequences of fastdiv.cuh.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "fastdiv.cuh"

namespace wb {

template <typename T> struct FTraits;
template <> struct FTraits<float> {
    using Bits = unsigned int;
    __device__ static __forceinline__ float rcp(float x) { return __frcp_rn(x); }
    __device__ static __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
    __device__ static __forceinline__ Bits abs_bits(float x) {
        return __float_as_uint(x) & 0x7fffffffu;
    }
    __device__ static __forceinline__ Bits bits(float x) { return __float_as_uint(x); }
};
template <> struct FTraits<double> {
    using Bits = unsigned long long;
    __device__ static __forceinline__ double rcp(double x) { return __drcp_rn(x); }
    __device__ static __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
    __device__ static __forceinline__ Bits abs_bits(double x) {
        return (Bits)__double_as_longlong(x) & 0x7fffffffffffffffull;
    }
    __device__ static __forceinline__ Bits bits(double x) { return (Bits)__double_as_longlong(x); }
};

// Material flavors (grids.py:99-100)
enum Flavor : int { RHO_SCALED = 0, ACOUSTIC = 1 };

// Per-run material scalars, all already rounded to T on the host exactly as
// solver.py:93-110 rounds them (dtype.type(python_float)).
template <typename T> struct MatScalars {
    int flavor;
    T two_r2;   // rho_scaled: dtype.type(2.0) * r2, r2 = T((c0*dt/dx)**2)
    T dt2;      // T(dt*dt)
    T rho0;     // rho_scaled: T(rho0)
    T irho1;    // acoustic: T(1/rho1)
    T drho;     // acoustic: T(1/rho2 - 1/rho1)
    T ikap1;    // acoustic: T(1/kappa1)
    T dkap;     // acoustic: T(1/kappa2 - 1/kappa1)
    T s2;       // acoustic: T((dt/dx)**2)
};

// Flavor- and division-specialised material functions (solver.py:89-119).
template <typename T, int FLAVOR, bool FAST> struct Mat {
    using D = Div<T, FAST>;
    // m: reciprocal flux coefficient feeding the face weights (solver.py:95,107)
    __device__ static __forceinline__ T m(const MatScalars<T>& M, T g) {
        if (FLAVOR == RHO_SCALED) return D::rcp(g);              // T(1)/gamma
        return D::rcp(M.irho1 + g * M.drho);                     // T(1)/inv_rho (grids.py:252)
    }
    // coef multiplying the face sum (solver.py:97,109); kappa kept for fc
    __device__ static __forceinline__ T coef(const MatScalars<T>& M, T g, T& kappa) {
        if (FLAVOR == RHO_SCALED) {
            kappa = T(0);
            return D::div(M.two_r2, g);                            // (2*r2)/gamma
        }
        kappa = D::rcp(M.ikap1 + g * M.dkap);                      // T(1)/inv_kappa
        return (T(2) * kappa) * M.s2;                              // (2*kappa)*s2
    }
    // face weight 1/(m_lo + m_hi) (solver.py:111-119)
    __device__ static __forceinline__ T face(T m_lo, T m_hi) { return D::rcp(m_lo + m_hi); }
    // nodal force coefficient (solver.py:98,110) — sparse: always the intrinsic
    __device__ static __forceinline__ T fc(const MatScalars<T>& M, T g, T kappa) {
        if (FLAVOR == RHO_SCALED) return FTraits<T>::div(M.dt2, M.rho0 * g);
        return kappa * M.dt2;
    }
};

// Runtime-flavor versions for the sparse / auxiliary kernels.
template <typename T>
__device__ __forceinline__ T mat_m(const MatScalars<T>& M, T g) {
    return M.flavor == RHO_SCALED ? Mat<T, RHO_SCALED, false>::m(M, g)
                                  : Mat<T, ACOUSTIC, false>::m(M, g);
}
template <typename T>
__device__ __forceinline__ T mat_coef(const MatScalars<T>& M, T g, T& kappa) {
    return M.flavor == RHO_SCALED ? Mat<T, RHO_SCALED, false>::coef(M, g, kappa)
                                  : Mat<T, ACOUSTIC, false>::coef(M, g, kappa);
}
template <typename T>
__device__ __forceinline__ T mat_fc(const MatScalars<T>& M, T g, T kappa) {
    return M.flavor == RHO_SCALED ? Mat<T, RHO_SCALED, false>::fc(M, g, kappa)
                                  : Mat<T, ACOUSTIC, false>::fc(M, g, kappa);
}

}  // namespace wb
