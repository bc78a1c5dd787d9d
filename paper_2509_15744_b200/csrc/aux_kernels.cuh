// Small per-shot / per-sweep kernels around the fused step:
//   misfit_kernel   fwi.py:57-63, tato.py:154-163 — per-step shot cost (fp64)
//                   and the k-scaled adjoint store (gradients.py:239, 263)
//   cost_sum_kernel gradients.py:231-238 — sequential per-step cost sum
//   scale_div_kernel gradients.py:315 — acc /= T(2k)
//   inject_kernel   solver.py:167-170 — sparse nodal += for >MAX_SRC nodes
//   dense_force_kernel solver.py:163-165 — out += fc * T(force)
//   reverse_axes_kernel io.py:29-52 — C-order field -> first-axis-fastest dump
//   adam_clip_kernel optim.py adam_step + clip_bounds on the device (8f-3)
#pragma once

#include "common.cuh"

namespace wb {

enum ShotKind : int { SHOT_NONE = 0, SHOT_FWI = 1, SHOT_TATO = 2 };

// One block per time step n.  store is [N][n_sup] (row n = trace entry n,
// i.e. u^n on the support, device support order).  measured is [n_sup][N]
// fp64 (the reference's layout, rows permuted to device support order).
// cost_n = (((c1 * dot) * c2) * c3) / c4 with
//   FWI : dot = sum r^2, r = double(u) - measured ; (c1..c4) = (0.5, dt, 1, 1)
//   TATO: dot = sum u^2                           ; (sign, cell, dt, area)
// adj (written in place over the trace when write_adj):
//   FWI : T(-r) * T(k)      TATO: T(adj_coef * double(u)) * T(k)
template <typename T>
__global__ void misfit_kernel(T* store, const double* measured, long long n_steps, int n_sup,
                              int kind, double c1, double c2, double c3, double c4,
                              double adj_coef, int write_adj, T k_t, double* partial) {
    __shared__ double sred[256];
    const long long n = blockIdx.x;
    double dot = 0.0;
    // per-thread partial sums in a fixed order, then a fixed tree: deterministic
    for (int s = threadIdx.x; s < n_sup; s += blockDim.x) {
        const double u = (double)store[n * n_sup + s];
        double v;
        if (kind == SHOT_FWI) {
            const double r = u - measured[(long long)s * n_steps + n];
            dot += r * r;
            v = -r;
        } else {
            dot += u * u;
            v = adj_coef * u;
        }
        if (write_adj) store[n * n_sup + s] = (n == 0) ? T(0) : (T)v * k_t;
    }
    sred[threadIdx.x] = dot;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sred[threadIdx.x] += sred[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[n] = (((c1 * sred[0]) * c2) * c3) / c4;
}

__global__ void cost_sum_kernel(const double* partial, long long n_steps, double* out) {
    // the per-step costs staged through shared memory by the whole block
    // (coalesced), then folded left to right by one thread like the
    // reference's per-step `cost +=` (a dependent chain of L2 loads was
    // 124 us at N = 3200)
    constexpr int CH = 1024;
    __shared__ double buf[CH];
    double c = 0.0;
    for (long long base = 0; base < n_steps; base += CH) {
        const int m = (int)(n_steps - base < CH ? n_steps - base : CH);
        for (int i = threadIdx.x; i < m; i += blockDim.x) buf[i] = partial[base + i];
        __syncthreads();
        if (threadIdx.x == 0) {
            int i = 0;
            if (base == 0) c = buf[i++];
            for (; i < m; ++i) c = c + buf[i];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = c;
}

// Nodal force coefficient fc(gamma) of every support node, in compact
// (increasing flat index) order: the two-step kernel's adjoint injection
// (gradients.py:268-269 through solver.py:167-170) multiplies by it instead
// of recomputing it per step from gamma with two IEEE divisions behind a
// chain of dependent global loads (C3 TATO 192^3: the objective region's
// CTAs made the backward sweep 2x the forward one).  Same operations as the
// kernels' per-cell fcoef, so the products are bit-identical.
template <typename T, int FLAVOR>
__global__ void sup_fc_kernel(const T* __restrict__ gamma, MatScalars<T> M,
                              const long long* __restrict__ flat, long long n, T* __restrict__ out) {
    using P = Mat<T, FLAVOR, false>;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const T g = gamma[flat[i]];
        T kap;
        (void)P::coef(M, g, kap);
        out[i] = P::fc(M, g, kap);
    }
}

template <typename T>
__global__ void scale_div_kernel(T* acc, long long n, T denom) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        acc[i] = FTraits<T>::div(acc[i], denom);
}

// out[idx[s]] += fc[idx[s]] * vals[s] for deduplicated idx (last occurrence
// kept by the host, matching numpy fancy-index +=).
template <typename T>
__global__ void inject_kernel(T* out, const T* gamma, MatScalars<T> M, const long long* idx,
                              const T* vals, int n) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const long long c = idx[s];
    T kappa;
    (void)mat_coef(M, gamma[c], kappa);
    out[c] = out[c] + mat_fc(M, gamma[c], kappa) * vals[s];
}

template <typename T>
__global__ void dense_force_kernel(T* out, const T* gamma, MatScalars<T> M, const double* f,
                                   long long n) {
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        T kappa;
        (void)mat_coef(M, gamma[c], kappa);
        out[c] = out[c] + mat_fc(M, gamma[c], kappa) * (T)f[c];
    }
}

template <typename T>
__global__ void max_abs_kernel(const T* u, long long n, typename FTraits<T>::Bits* slot) {
    typename FTraits<T>::Bits m = 0;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        typename FTraits<T>::Bits b = FTraits<T>::abs_bits(u[c]);
        m = b > m ? b : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
        typename FTraits<T>::Bits v = __shfl_xor_sync(0xffffffffu, m, o);
        m = v > m ? v : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(slot, m);
}

// out = the field with its axes reversed (A, B, C) -> (C, B, A): the
// first-axis-fastest byte order of the reference's field dumps
// (io.py:29-52, np.ravel(order="F")).  For each middle index j the (A x C)
// slab is transposed through a 32 x 33 shared tile so both the reads (along
// C) and the writes (along A) are coalesced.  2D / 1D fields are (1, n0, n1)
// / (1, 1, n0) here; reversing those dims gives the same bytes.
template <typename T>
__global__ void reverse_axes_kernel(const T* __restrict__ in, T* __restrict__ out, int A, int B,
                                    int C) {
    __shared__ T tile[32][33];
    const int j = blockIdx.z;
    const int k0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {   // rows i, columns k
        const int i = i0 + r, k = k0 + threadIdx.x;
        if (i < A && k < C) tile[r][threadIdx.x] = in[((long long)i * B + j) * C + k];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {   // rows k, columns i
        const int k = k0 + r, i = i0 + threadIdx.x;
        if (i < A && k < C) out[((long long)k * B + j) * A + i] = tile[threadIdx.x][r];
    }
}

// numpy's clip for floats: MIN(MAX(x, lo), hi) with NaN passed through and
// PyArray_MAX(a, b) = a > b ? a : b (npy_math / clip loops)
__device__ __forceinline__ double np_clip(double x, double lo, double hi) {
    if (x != x) return x;
    const double y = x > lo ? x : lo;
    return y < hi ? y : hi;
}

struct AdamScalars {
    double beta1, beta2, c1, c2;   // c1 = 1 - beta1, c2 = 1 - beta2 (host Python floats)
    double bc1, bc2;               // 1 - beta1**t, 1 - beta2**t
    double alpha, eps, lo, hi, frozen_value;
};

// One bias-corrected Adam step and bound clip per cell with numpy's fp64
// operation order (optim.py adam_step / clip_bounds, fwi.py:178-238):
//   g = double(acc) (0 on frozen cells when zero_frozen)
//   m = b1*m + (1-b1)*g ;  v = b2*v + ((1-b2)*g)*g
//   p = p - (alpha*(m/bc1)) / (sqrt(v/bc2) + eps) ; clip ; frozen -> value
// The new parameters are also cast to the field dtype (gamma.astype(T); FWI:
// the parameters ARE the material; TATO passes gamma = nullptr) and
// the block partial sums of g*g (fixed tree) give the logged gradient norm.
template <typename G, typename T>
__global__ void adam_clip_kernel(const G* __restrict__ acc, double* __restrict__ p,
                                 double* __restrict__ m, double* __restrict__ v,
                                 const unsigned char* __restrict__ frozen, int zero_frozen,
                                 AdamScalars s, long long n, T* __restrict__ gamma,
                                 double* __restrict__ partial) {
    __shared__ double red[256];
    double sq = 0.0;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const bool fz = frozen && frozen[c];
        double g = (double)acc[c];
        if (zero_frozen && fz) g = 0.0;
        sq = sq + g * g;
        const double mc = __dadd_rn(__dmul_rn(s.beta1, m[c]), __dmul_rn(s.c1, g));
        const double vc = __dadd_rn(__dmul_rn(s.beta2, v[c]), __dmul_rn(__dmul_rn(s.c2, g), g));
        m[c] = mc;
        v[c] = vc;
        const double mh = __ddiv_rn(mc, s.bc1), vh = __ddiv_rn(vc, s.bc2);
        const double step = __ddiv_rn(__dmul_rn(s.alpha, mh), __dadd_rn(__dsqrt_rn(vh), s.eps));
        double x = np_clip(__dsub_rn(p[c], step), s.lo, s.hi);
        if (fz) x = s.frozen_value;
        p[c] = x;
        if (gamma) gamma[c] = (T)x;
    }
    red[threadIdx.x] = sq;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

template <typename T>
__global__ void widen_kernel(const T* __restrict__ src, double* __restrict__ dst, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        dst[i] = (double)src[i];
}

}  // namespace wb
