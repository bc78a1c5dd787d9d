// Vectorised fused step: each thread owns a PAIR of adjacent cells along the
// contiguous axis 2 (8-byte float2 / 16-byte double2 accesses), a CTA a
// BY x 64-cell tile.  Same arithmetic, operation order and boundary
// treatment as step_kernel (step_kernel.cuh, whose header documents the
// reference mapping); what changes is the instruction budget per cell:
//   * one vector load/store per stream per pair;
//   * the face weight between the two cells of a pair lives in registers,
//     the pair's outer k-faces are computed from shared m, the j-faces are
//     shared through shared memory (computed once per face);
//   * loop control, address arithmetic and the barrier are paid once per
//     two cells.
// Requires an even row length n2 (pairs never straddle rows and stay
// aligned); the scalar kernel covers odd n2.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "step_kernel.cuh"

namespace wb {

constexpr int PBX = 64;           // cells per tile row (32 threads x 2)
constexpr int PW = PBX + 4;       // smem row: [pad][halo L][64 cells][halo R][pad]

template <typename T> struct Pair;
template <> struct Pair<float> { using V = float2; };
template <> struct Pair<double> { using V = double2; };

template <typename T, int FLAVOR, bool FAST, bool ACC, bool CHECK>
__global__ void __launch_bounds__(NTHREADS)
step_kernel_pair(const StepArgs<T> a) {
    using Tr = FTraits<T>;
    using MT = Mat<T, FLAVOR, FAST>;
    using V = typename Pair<T>::V;
    __shared__ __align__(16) T su[2][BY + 2][PW];
    __shared__ __align__(16) T sm[2][BY + 2][PW];
    __shared__ __align__(16) T sfj[2][BY + 1][PBX];   // j-face (j-1, j) per column
    __shared__ typename Tr::Bits smax[NTHREADS / 32];

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * 32 + tx;
    const int k0 = blockIdx.x * PBX, j0 = blockIdx.y * BY;
    const int kA = k0 + 2 * tx, j = j0 + ty;
    const int n1 = a.n1, n2 = a.n2;
    const bool oob = kA >= n2;                 // pair beyond the row: mirror of the last cell
    const bool inb = (j < n1) && !oob;
    const long long plane = (long long)n1 * n2;   // 64-bit plane offsets: grids of >= 2^31 cells
    const int i0 = a.c_lo + blockIdx.z * a.chunk;   // computed planes [c_lo, c_hi)
    const int i1 = min(i0 + a.chunk, a.c_hi);
    const MatScalars<T>& M = a.mat;
    const int cs = 2 + 2 * tx;                 // smem column of cell A

    const int jc = min(j, n1 - 1), kc = min(kA, n2 - 2);
    const int cofs = jc * n2 + kc;

    // halo roles: 16 scalar k-halo cells, 64 j-halo pairs (top/bottom rows)
    int hofs = 0, hsy = 0, hsx = 0;
    const bool hk_role = tid < 2 * BY;
    const bool hj_role = tid >= 2 * BY && tid < 2 * BY + 64;
    if (hk_role) {
        const int r = tid < BY ? tid : tid - BY;
        const int hk = tid < BY ? max(k0 - 1, 0) : min(k0 + PBX, n2 - 1);
        hofs = min(j0 + r, n1 - 1) * n2 + hk;
        hsy = r + 1;
        hsx = tid < BY ? 1 : PBX + 2;
    } else if (hj_role) {
        const int q = tid - 2 * BY;
        const int p = q & 31;
        const int hj = q < 32 ? max(j0 - 1, 0) : min(j0 + BY, n1 - 1);
        hofs = hj * n2 + min(k0 + 2 * p, n2 - 2);
        hsy = q < 32 ? 0 : BY + 1;
        hsx = 2 + 2 * p;
    }

    unsigned my_src = 0;
    for (int s = 0; s < a.n_src; ++s)
        if (a.src_i[s] >= i0 && a.src_i[s] < i1 && a.src_j[s] >= j0 && a.src_j[s] < j0 + BY &&
            a.src_k[s] >= k0 && a.src_k[s] < k0 + PBX)
            my_src |= 1u << s;

    auto pc = [&](int i) { return min(max(i, a.i_lo), a.i_hi - 1) * plane; };
    auto ldv = [&](const T* p) {
        V v = __ldg(reinterpret_cast<const V*>(p));
        if (oob) v.x = v.y;
        return v;
    };
    auto ldh = [&](const T* base, long long o) {       // halo load (scalar or pair role)
        V v;
        if (hk_role) { v.x = __ldg(base + o + hofs); v.y = v.x; }
        else v = __ldg(reinterpret_cast<const V*>(base + o + hofs));
        return v;
    };
    auto sth = [&](T (*buf)[PW], V v) {          // halo store
        if (hk_role) buf[hsy][hsx] = v.x;
        else *reinterpret_cast<V*>(&buf[hsy][hsx]) = v;
    };
    const bool hal = hk_role || hj_role;
    const int last = a.n0 - 1;

    // ---- prologue ----
    V u_0 = ldv(a.u_cur + i0 * plane + cofs);
    V u_m1 = ldv(a.u_cur + pc(i0 - 1) + cofs);
    V g_0 = ldv(a.gamma + i0 * plane + cofs);
    V u_p1 = ldv(a.u_cur + pc(i0 + 1) + cofs);
    V g_p1 = ldv(a.gamma + pc(i0 + 1) + cofs);
    V up = __ldg(reinterpret_cast<const V*>(a.u_prev + i0 * plane + cofs));
    V acc_old = ACC ? *reinterpret_cast<const V*>(a.acc + i0 * plane + cofs) : V{};
    V m_0 = {MT::m(M, g_0.x), MT::m(M, g_0.y)};
    V wf0_lo;
    {
        const V gm = ldv(a.gamma + pc(i0 - 1) + cofs);
        wf0_lo.x = MT::face(MT::m(M, gm.x), m_0.x);
        wf0_lo.y = MT::face(MT::m(M, gm.y), m_0.y);
    }
    V hu = {T(0), T(0)}, hg = {T(1), T(1)};
    *reinterpret_cast<V*>(&sm[0][ty + 1][cs]) = m_0;
    if (hal) {
        const V hg0 = ldh(a.gamma, i0 * plane);
        sth(sm[0], V{MT::m(M, hg0.x), MT::m(M, hg0.y)});
        hu = ldh(a.u_cur, i0 * plane);
        hg = ldh(a.gamma, pc(i0 + 1));
    }
    __syncthreads();
    // faces of plane i0: pair-outer k-faces + internal face in registers,
    // j lo-faces to smem (+ bottom row by warp 1)
    T fkL, fkI, fkR;
    V fj_lo;
    auto faces = [&](T (*smb)[PW], T (*sfb)[PBX], V m_c, T& oL, T& oI, T& oR, V& ojlo) {
        oL = MT::face(smb[ty + 1][cs - 1], m_c.x);
        oI = MT::face(m_c.x, m_c.y);
        oR = MT::face(m_c.y, smb[ty + 1][cs + 2]);
        const V mu = *reinterpret_cast<const V*>(&smb[ty][cs]);
        ojlo.x = MT::face(mu.x, m_c.x);
        ojlo.y = MT::face(mu.y, m_c.y);
        *reinterpret_cast<V*>(&sfb[ty][cs - 2]) = ojlo;
        if (tid >= 32 && tid < 64) {
            const int p = tid - 32;
            const V ma = *reinterpret_cast<const V*>(&smb[BY][2 + 2 * p]);
            const V mb = *reinterpret_cast<const V*>(&smb[BY + 1][2 + 2 * p]);
            *reinterpret_cast<V*>(&sfb[BY][2 * p]) = V{MT::face(ma.x, mb.x), MT::face(ma.y, mb.y)};
        }
    };
    faces(sm[0], sfj[0], m_0, fkL, fkI, fkR, fj_lo);

    typename Tr::Bits local_max = 0;

    auto body = [&](auto parity, int i) {
        constexpr int b = decltype(parity)::value, nb = b ^ 1;
        const bool next = i + 1 < i1;
        const long long oc = i * plane + cofs;

        // loads for the next iteration (clamped, always in bounds)
        const long long on = min(i + 1, last) * plane;
        const long long o2 = pc(i + 2);
        const V up_n = __ldg(reinterpret_cast<const V*>(a.u_prev + on + cofs));
        const V acc_n = ACC ? *reinterpret_cast<const V*>(a.acc + on + cofs) : V{};
        const V u_p2 = ldv(a.u_cur + o2 + cofs);
        const V g_p2 = ldv(a.gamma + o2 + cofs);
        V hu_n = hu, hg_n = hg;
        if (hal) {
            hu_n = ldh(a.u_cur, on);
            hg_n = ldh(a.gamma, o2);
        }

        // A: stage u(i) and m(i+1)
        *reinterpret_cast<V*>(&su[b][ty + 1][cs]) = u_0;
        if (hal) sth(su[b], hu);
        const V m_p1 = {MT::m(M, g_p1.x), MT::m(M, g_p1.y)};
        if (next) {
            *reinterpret_cast<V*>(&sm[nb][ty + 1][cs]) = m_p1;
            if (hal) sth(sm[nb], V{MT::m(M, hg.x), MT::m(M, hg.y)});
        }
        __syncthreads();

        // C: faces of plane i+1 (registers + smem)
        T nL = fkL, nI = fkI, nR = fkR;
        V njlo = fj_lo;
        if (next) faces(sm[nb], sfj[nb], m_p1, nL, nI, nR, njlo);

        // D: plane i
        const V uj_m = *reinterpret_cast<const V*>(&su[b][ty][cs]);
        const V uj_p = *reinterpret_cast<const V*>(&su[b][ty + 2][cs]);
        const T uL = su[b][ty + 1][cs - 1];
        const T uR = su[b][ty + 1][cs + 2];
        const V fj_hi = *reinterpret_cast<const V*>(&sfj[b][ty + 1][cs - 2]);
        const V wf0_hi = {MT::face(m_0.x, m_p1.x), MT::face(m_0.y, m_p1.y)};
        T kapA, kapB;
        const T coefA = MT::coef(M, g_0.x, kapA);
        const T coefB = MT::coef(M, g_0.y, kapB);
        // cell A, kernels.py:56-69 order: axis 0, axis 1 (j), axis 2 (k)
        T accA = u_0.x - u_0.x;
        accA += (u_p1.x - u_0.x) * wf0_hi.x;
        accA -= (u_0.x - u_m1.x) * wf0_lo.x;
        accA += (uj_p.x - u_0.x) * fj_hi.x;
        accA -= (u_0.x - uj_m.x) * fj_lo.x;
        accA += (u_0.y - u_0.x) * fkI;
        accA -= (u_0.x - uL) * fkL;
        // cell B
        T accB = u_0.y - u_0.y;
        accB += (u_p1.y - u_0.y) * wf0_hi.y;
        accB -= (u_0.y - u_m1.y) * wf0_lo.y;
        accB += (uj_p.y - u_0.y) * fj_hi.y;
        accB -= (u_0.y - uj_m.y) * fj_lo.y;
        accB += (uR - u_0.y) * fkR;
        accB -= (u_0.y - u_0.x) * fkI;
        V out;
        out.x = ((u_0.x + u_0.x) - up.x) + coefA * accA;
        out.y = ((u_0.y + u_0.y) - up.y) + coefB * accB;

        // nodal injections, solver.py:167-170 (sources first, then support)
        if (my_src) {
            for (int s = 0; s < a.n_src; ++s) {
                if (!((my_src >> s) & 1u) || i != a.src_i[s] || j != a.src_j[s]) continue;
                if (kA == a.src_k[s]) out.x = out.x + MT::fc(M, g_0.x, kapA) * a.src_val[s];
                if (kA + 1 == a.src_k[s]) out.y = out.y + MT::fc(M, g_0.y, kapB) * a.src_val[s];
            }
        }
        if (a.sup_mode != SUP_NONE && i >= a.sup_lo && i <= a.sup_hi && inb) {
            const unsigned long long flat = (unsigned long long)oc;       // even: A and B share a word
            const unsigned int w = __ldg(a.sup_mask + (flat >> 5));
            const unsigned int bit = (unsigned int)(flat & 31u);
            const unsigned int two = (w >> bit) & 3u;
            if (two) {
                const int s = __ldg(a.sup_prefix + (flat >> 5)) + __popc(w & ((1u << bit) - 1u));
                if (a.sup_mode == SUP_GATHER) {
                    if (two & 1u) a.trace_row[s] = u_0.x;
                    if (two & 2u) a.trace_row[s + (two & 1u)] = u_0.y;
                } else {
                    if (two & 1u) out.x = out.x + MT::fc(M, g_0.x, kapA) * ldg(a.adj_row + s);
                    if (two & 2u)
                        out.y = out.y + MT::fc(M, g_0.y, kapB) * ldg(a.adj_row + s + (two & 1u));
                }
            }
        }

        // self-kernel increments, kernels.py:105-128 (clamped differences)
        if (ACC) {
            const T vaA = a.backward ? (up.x - out.x) * a.inv2dt : (out.x - up.x) * a.inv2dt;
            const T vaB = a.backward ? (up.y - out.y) * a.inv2dt : (out.y - up.y) * a.inv2dt;
            const T g0A = (u_p1.x - u_m1.x) * a.inv2dx, g0B = (u_p1.y - u_m1.y) * a.inv2dx;
            const T g1A = (uj_p.x - uj_m.x) * a.inv2dx, g1B = (uj_p.y - uj_m.y) * a.inv2dx;
            const T g2A = (u_0.y - uL) * a.inv2dx, g2B = (uR - u_0.x) * a.inv2dx;
            V nacc;
            if (a.one_d) {
                nacc.x = acc_old.x + a.sdt * ((a.cv * vaA) * vaA + (a.cg * g2A) * g2A);
                nacc.y = acc_old.y + a.sdt * ((a.cv * vaB) * vaB + (a.cg * g2B) * g2B);
            } else {
                nacc.x = acc_old.x + a.sdt * ((a.cv * vaA) * vaA +
                                              a.cg * (((g0A * g0A) + (g1A * g1A)) + (g2A * g2A)));
                nacc.y = acc_old.y + a.sdt * ((a.cv * vaB) * vaB +
                                              a.cg * (((g0B * g0B) + (g1B * g1B)) + (g2B * g2B)));
            }
            if (inb) *reinterpret_cast<V*>(a.acc + oc) = nacc;
        }
        if (inb) {
            *reinterpret_cast<V*>(a.u_out + oc) = out;
            if (a.hist_out) *reinterpret_cast<V*>(a.hist_out + oc) = out;
            if (i < 2 && a.plo) *reinterpret_cast<V*>(a.plo + oc) = out;
            if (i >= a.n0 - 2 && a.phi) *reinterpret_cast<V*>(a.phi + oc) = out;
            if (CHECK) {
                typename Tr::Bits bx = Tr::abs_bits(out.x), by = Tr::abs_bits(out.y);
                bx = bx > by ? bx : by;
                local_max = bx > local_max ? bx : local_max;
            }
        }
        // advance the queue
        u_m1 = u_0; u_0 = u_p1; u_p1 = u_p2;
        g_0 = g_p1; g_p1 = g_p2;
        m_0 = m_p1; wf0_lo = wf0_hi;
        fkL = nL; fkI = nI; fkR = nR; fj_lo = njlo;
        up = up_n; acc_old = acc_n;
        hu = hu_n; hg = hg_n;
    };

    for (int i = i0; i < i1; i += 2) {
        body(std::integral_constant<int, 0>{}, i);
        if (i + 1 < i1) body(std::integral_constant<int, 1>{}, i + 1);
    }

    if (CHECK) {
        for (int o = 16; o > 0; o >>= 1) {
            typename Tr::Bits v = __shfl_xor_sync(0xffffffffu, local_max, o);
            local_max = v > local_max ? v : local_max;
        }
        const int lane = tid & 31, warp = tid >> 5;
        if (lane == 0) smax[warp] = local_max;
        __syncthreads();
        if (warp == 0) {
            typename Tr::Bits v = lane < (NTHREADS / 32) ? smax[lane] : 0;
            for (int o = 16; o > 0; o >>= 1) {
                typename Tr::Bits w = __shfl_xor_sync(0xffffffffu, v, o);
                v = w > v ? w : v;
            }
            if (lane == 0 && v) atomicMax(a.max_slot, v);
        }
    }
}

}  // namespace wb
