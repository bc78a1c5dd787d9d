// Topology-optimisation design chain (tato.py:61-140) in fp64, the dtype the
// reference uses for it:
//   masked_correlate  scipy.ndimage.correlate(mode="constant", cval=0) of
//                     where(mask, v, 0) and of mask, restricted to the
//                     non-zero footprint of the linear-decay kernel, summed
//                     in C order of the footprint like ndimage's NI_Correlate
//   heaviside         (tanh(b*eta) + tanh(b*(g-eta))) / denom, clipped
//   chain             g * beta / (denom * cosh(b*(g-eta))^2) on the mask
// The correlation sums are bit-exact with the reference; tanh/cosh use the
// CUDA libm (<= 2 ulp), so the projection agrees to a few ulp, not bitwise.
#pragma once

#include <cstdint>

namespace wb {

struct Footprint {
    int n;
    const int* off;      // [n][3] kernel offsets (kernel space axes)
    const double* w;     // [n] weights
};

// out_num[c] = sum_f where(mask, v, 0)[c+off_f] * w_f ; out_den likewise for mask
__global__ void masked_correlate_kernel(int n0, int n1, int n2, const double* v,
                                        const unsigned char* mask, int use_mask_on_v,
                                        Footprint fp, double* out_num, double* out_den) {
    const long long N = (long long)n0 * n1 * n2;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
         c += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(c % n2);
        const int j = (int)((c / n2) % n1);
        const int i = (int)(c / ((long long)n1 * n2));
        double num = 0.0, den = 0.0;
        for (int f = 0; f < fp.n; ++f) {
            const int ii = i + fp.off[3 * f], jj = j + fp.off[3 * f + 1], kk = k + fp.off[3 * f + 2];
            const double w = fp.w[f];
            double x = 0.0, m = 0.0;
            if (ii >= 0 && ii < n0 && jj >= 0 && jj < n1 && kk >= 0 && kk < n2) {
                const long long q = ((long long)ii * n1 + jj) * n2 + kk;
                const bool in = mask ? mask[q] != 0 : true;
                x = (use_mask_on_v && !in) ? 0.0 : v[q];
                m = in ? 1.0 : 0.0;
            }
            num = num + x * w;
            den = den + m * w;
        }
        if (out_num) out_num[c] = num;
        if (out_den) out_den[c] = den;
    }
}

// density_filter epilogue (tato.py:90-94): out = mask ? num/den : gamma
__global__ void filter_finish_kernel(long long N, const double* gamma, const unsigned char* mask,
                                     const double* num, const double* den, double* out) {
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
         c += (long long)gridDim.x * blockDim.x) {
        const bool in = mask ? mask[c] != 0 : true;
        out[c] = in ? __ddiv_rn(num[c], den[c]) : gamma[c];
    }
}

// heaviside_project (tato.py:97-108) + design-region masking (tato.py:226)
__global__ void heaviside_kernel(long long N, const double* g, double beta, double eta,
                                 double t_be, double denom, const unsigned char* mask,
                                 double* out) {
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
         c += (long long)gridDim.x * blockDim.x) {
        double v = __ddiv_rn(t_be + tanh(beta * (g[c] - eta)), denom);
        v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        if (mask && !mask[c]) v = 0.0;
        out[c] = v;
    }
}

// chain_rule step 1 (tato.py:131): inner = mask ? g * beta/(denom*cosh^2) : 0
__global__ void chain_inner_kernel(long long N, const double* dcdbar, const double* g_tilde,
                                   double beta, double eta, double denom,
                                   const unsigned char* mask, double* inner) {
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
         c += (long long)gridDim.x * blockDim.x) {
        const bool in = mask ? mask[c] != 0 : true;
        double v = 0.0;
        if (in) {
            const double ch = cosh(beta * (g_tilde[c] - eta));
            v = dcdbar[c] * __ddiv_rn(beta, denom * (ch * ch));
        }
        inner[c] = v;
    }
}

// chain_rule step 2 (tato.py:133-134): ratio = mask ? inner/den : 0
__global__ void chain_ratio_kernel(long long N, const double* inner, const double* den,
                                   const unsigned char* mask, double* ratio) {
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
         c += (long long)gridDim.x * blockDim.x) {
        const bool in = mask ? mask[c] != 0 : true;
        ratio[c] = in ? __ddiv_rn(inner[c], den[c]) : 0.0;
    }
}

// chain_rule step 3 (tato.py:136-139): out = mask ? correlate(ratio) : 0
__global__ void mask_zero_kernel(long long N, const unsigned char* mask, double* out) {
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
         c += (long long)gridDim.x * blockDim.x)
        if (mask && !mask[c]) out[c] = 0.0;
}

}  // namespace wb
