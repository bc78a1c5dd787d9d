// TMA-pipelined fused step, 2x2 cells per thread (production kernel on
// whole-tile grids).
//
// Data movement (tma_common.cuh): a 4-stage TMA ring of u^n / gamma halo
// boxes and u^{n-1} / acc tiles, one producer thread, mbarrier completion.
// Round 1's first TMA kernel (256 threads x 2 cells) was superseded by this
// layout, which cuts the per-cell instruction count:
//   * a thread owns a 2x2 block (rows j, j+1 x cells k, k+1): the k-face and
//     the j-face inside the block live in registers, the outer faces are
//     computed directly from the shared m-plane (no shared face arrays), and
//     loop control / addressing / barriers are paid once per four cells;
//   * the plane loop is unrolled by the stage count, so stage indices, mbarrier
//     parities and shared-memory buffer offsets are compile-time constants.
// Arithmetic, operation order and the mirrored-boundary argument are those of
// step_kernel.cuh (bit-identical to the reference).  Block 32 x 4 threads,
// tile 64 x 8 cells.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "step_kernel.cuh"
#include "tma_common.cuh"
#include "step_kernel_v2.cuh"

namespace wb {

constexpr int T4_THREADS = 128;
#ifndef WB_TMA_STAGES
#define WB_TMA_STAGES 4
#endif
constexpr int NS = WB_TMA_STAGES;        // ring stages (NS-1 planes in flight ahead)
constexpr int U = NS % 2 ? 2 * NS : NS;  // planes per unrolled group: lcm(NS, 2)

// body(q, plane) for q = 0..U-1 while the planes exist
template <typename B, int... Q>
__device__ __forceinline__ void unroll_planes(B& body, int i, int i1, unsigned gpar,
                                              std::integer_sequence<int, Q...>) {
    bool go = true;
    ((go = go && (i + Q < i1), go ? (body(std::integral_constant<int, Q>{}, i + Q, gpar), 0) : 0),
     ...);
}

template <typename T, int FLAVOR, bool FAST, bool ACC, bool CHECK, int SUP>
__global__ void __launch_bounds__(T4_THREADS, sizeof(T) == 4 ? 4 : 2)
step_kernel_tma4(const __grid_constant__ StepArgs<T> a, const __grid_constant__ TmaMaps maps) {
    using Tr = FTraits<T>;
    using MT = Mat<T, FLAVOR, FAST>;
    using V = typename Pair<T>::V;
    constexpr int W = th_w<T>(), HO = th_ho<T>();
    extern __shared__ __align__(128) unsigned char smem_dyn[];
    unsigned char* smem_raw =
        smem_dyn + ((128u - (static_cast<unsigned>(__cvta_generic_to_shared(smem_dyn)) & 127u)) & 127u);
    TmaStage<T>* st = reinterpret_cast<TmaStage<T>*>(smem_raw);
    T(*SM)[TH_H][W] = reinterpret_cast<T(*)[TH_H][W]>(smem_raw + NS * sizeof(TmaStage<T>));
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(
        smem_raw + NS * sizeof(TmaStage<T>) + 2 * sizeof(T) * TH_H * W);
    __shared__ typename Tr::Bits smax[T4_THREADS / 32];

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * 32 + tx;
    const int k0 = blockIdx.x * PBX, j0 = blockIdx.y * BY;
    const int kA = k0 + 2 * tx, ja = j0 + 2 * ty;
    const int n1 = a.n1, n2 = a.n2;
    const long long plane = (long long)n1 * n2;   // 64-bit plane offsets: grids of >= 2^31 cells
    const int i0 = a.c_lo + blockIdx.z * a.chunk;   // computed planes [c_lo, c_hi)
    const int i1 = min(i0 + a.chunk, a.c_hi);
    const int plast = a.i_hi - 1;
    const int pend = min(i1, plast);
    const MatScalars<T>& M = a.mat;

    // shared-memory coordinates: rows ra, rb = ra+1 of the block; clamped
    // (mirrored) outer neighbours
    const int ra = 2 * ty + 1, rb = ra + 1;
    const int rU = ja > 0 ? ra - 1 : ra, rD = ja + 2 < n1 ? rb + 1 : rb;
    const int cA = HO + 2 * tx;
    const int cL = kA > 0 ? cA - 1 : cA, cR = kA + 2 < n2 ? cA + 2 : cA + 1;
    // m-plane halo roles: 16 k-halo cells, 64 j-halo pairs
    const bool hk_role = tid < 2 * BY;
    const bool hj_role = tid >= 2 * BY && tid < 2 * BY + 64;
    int hr = 0, hc = 0;
    if (hk_role) { hr = (tid < BY ? tid : tid - BY) + 1; hc = tid < BY ? HO - 1 : HO + PBX; }
    else if (hj_role) { const int q = tid - 2 * BY; hr = q < 32 ? 0 : BY + 1; hc = HO + 2 * (q & 31); }

    unsigned my_src = 0;
    for (int s = 0; s < a.n_src; ++s)
        if (a.src_i[s] >= i0 && a.src_i[s] < i1 && a.src_j[s] >= j0 && a.src_j[s] < j0 + BY &&
            a.src_k[s] >= k0 && a.src_k[s] < k0 + PBX)
            my_src |= 1u << s;

    constexpr unsigned STAGE_BYTES =
        (unsigned)(sizeof(T) * (2 * TH_H * W + (ACC ? 2 : 1) * BY * PBX));
    const CUtensorMap* mU = pick_map(maps.u_halo, maps.cur);
    const CUtensorMap* mP = pick_map(maps.u_ctr, maps.prev);
    auto issue = [&](int p, int s) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[s], STAGE_BYTES);
        tma_load_3d(&st[s].U[0][0], mU, k0 - HO, j0 - 1, p + maps.lo, &bar[s]);
        tma_load_3d(&st[s].G[0][0], &maps.g_halo, k0 - HO, j0 - 1, p + maps.lo, &bar[s]);
        tma_load_3d(&st[s].P[0][0], mP, k0, j0, p + maps.lo, &bar[s]);
        if (ACC) tma_load_3d(&st[s].A[0][0], &maps.a_ctr, k0, j0, p, &bar[s]);
    };

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
#if WB_T2_PDL
    // programmatic dependent launch (as step2_kernel_tma): no global access above
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    if (tid == 0)
        for (int p = i0; p <= min(i0 + NS - 1, pend); ++p) issue(p, p - i0);

    auto ldv = [](const T* p) { return *reinterpret_cast<const V*>(p); };
    auto stv = [](T* p, V v) { *reinterpret_cast<V*>(p) = v; };

    // ---- prologue: plane i0 ----
    const int cofs = ja * n2 + kA;             // row a; row b is + n2
    const bool has_m0 = i0 > a.i_lo;
    V um_a = {T(0), T(0)}, um_b = um_a, gm_a = {T(1), T(1)}, gm_b = gm_a;
    if (has_m0) {
        um_a = __ldg(reinterpret_cast<const V*>(a.u_cur + (i0 - 1) * plane + cofs));
        um_b = __ldg(reinterpret_cast<const V*>(a.u_cur + (i0 - 1) * plane + cofs + n2));
        gm_a = __ldg(reinterpret_cast<const V*>(a.gamma + (i0 - 1) * plane + cofs));
        gm_b = __ldg(reinterpret_cast<const V*>(a.gamma + (i0 - 1) * plane + cofs + n2));
    }
    mbar_wait(&bar[0], 0);
    V u0_a = ldv(&st[0].U[ra][cA]), u0_b = ldv(&st[0].U[rb][cA]);
    V g0_a = ldv(&st[0].G[ra][cA]), g0_b = ldv(&st[0].G[rb][cA]);
    if (!has_m0) { um_a = u0_a; um_b = u0_b; gm_a = g0_a; gm_b = g0_b; }
    V m0_a = {MT::m(M, g0_a.x), MT::m(M, g0_a.y)};
    V m0_b = {MT::m(M, g0_b.x), MT::m(M, g0_b.y)};
    V w0_a = {MT::face(MT::m(M, gm_a.x), m0_a.x), MT::face(MT::m(M, gm_a.y), m0_a.y)};
    V w0_b = {MT::face(MT::m(M, gm_b.x), m0_b.x), MT::face(MT::m(M, gm_b.y), m0_b.y)};
    stv(&SM[0][ra][cA], m0_a);
    stv(&SM[0][rb][cA], m0_b);
    if (hk_role) SM[0][hr][hc] = MT::m(M, st[0].G[hr][hc]);
    else if (hj_role) {
        const V hg = ldv(&st[0].G[hr][hc]);
        stv(&SM[0][hr][hc], V{MT::m(M, hg.x), MT::m(M, hg.y)});
    }
    __syncthreads();

    // faces of a plane from its m-plane: k-faces (L, I, R) per row, j-faces
    // (row a lo, a-b inside, row b hi)
    struct Faces { T kLa, kIa, kRa, kLb, kIb, kRb; V jlo, jab, jhi; };
    auto faces = [&](T (*smb)[W], V ma, V mb) {
        Faces f;
        f.kLa = MT::face(smb[ra][cL], ma.x);
        f.kIa = MT::face(ma.x, ma.y);
        f.kRa = MT::face(ma.y, smb[ra][cR]);
        f.kLb = MT::face(smb[rb][cL], mb.x);
        f.kIb = MT::face(mb.x, mb.y);
        f.kRb = MT::face(mb.y, smb[rb][cR]);
        const V mu = ldv(&smb[rU][cA]);
        const V md = ldv(&smb[rD][cA]);
        f.jlo = V{MT::face(mu.x, ma.x), MT::face(mu.y, ma.y)};
        f.jab = V{MT::face(ma.x, mb.x), MT::face(ma.y, mb.y)};
        f.jhi = V{MT::face(mb.x, md.x), MT::face(mb.y, md.y)};
        return f;
    };
    Faces F = faces(SM[0], m0_a, m0_b);

    typename Tr::Bits local_max = 0;

    // one cell: face sum in the order of kernels.py:56-69, out, kernel increment
    auto cell = [&](T u0, T up1, T um1, T ujp, T ujm, T ukp, T ukm, T w0hi, T w0lo, T fjhi, T fjlo,
                    T fkhi, T fklo, T coef, T up, T& out) {
        T s = u0 - u0;
        s += (up1 - u0) * w0hi;
        s -= (u0 - um1) * w0lo;
        s += (ujp - u0) * fjhi;
        s -= (u0 - ujm) * fjlo;
        s += (ukp - u0) * fkhi;
        s -= (u0 - ukm) * fklo;
        out = ((u0 + u0) - up) + coef * s;
    };
    auto kinc = [&](T accv, T out, T up, T up1, T um1, T ujp, T ujm, T ukp, T ukm) {
        // (cv*va)*va is invariant under va -> -va: one form for both sweeps
        const T va = (out - up) * a.inv2dt;
        const T g0 = (up1 - um1) * a.inv2dx;
        const T g1 = (ujp - ujm) * a.inv2dx;
        const T g2 = (ukp - ukm) * a.inv2dx;
        return accv + a.sdt * ((a.cv * va) * va + a.cg * (((g0 * g0) + (g1 * g1)) + (g2 * g2)));
    };

    // body<q>: plane i = (group start) + q.  Stage of plane i is q % NS, the
    // m-plane buffer q & 1; the mbarrier parity of plane i+1 is static within
    // an unrolled group of U = lcm(NS, 2) planes up to the group parity gpar.
    auto body = [&](auto stage, int i, unsigned gpar) {
        constexpr int q = decltype(stage)::value;
        constexpr int s = q % NS, sn = (q + 1) % NS, sf = (q + NS - 1) % NS;
        constexpr int b = q & 1, nb = b ^ 1;
        constexpr unsigned pnext = (unsigned)(((q + 1) / NS) & 1);   // within-group parity
        constexpr unsigned gflip = (unsigned)((U / NS) & 1);          // parity step per group
        const bool next = i + 1 < i1;
        // ---- plane i+1 from its stage (mirror beyond the global end) ----
        V up1_a = u0_a, up1_b = u0_b, gp1_a = g0_a, gp1_b = g0_b;
        if (i + 1 <= plast) {
            mbar_wait(&bar[sn], (q + 1 == U) ? (gpar ^ gflip) : (gpar ^ pnext));
            up1_a = ldv(&st[sn].U[ra][cA]);
            up1_b = ldv(&st[sn].U[rb][cA]);
            gp1_a = ldv(&st[sn].G[ra][cA]);
            gp1_b = ldv(&st[sn].G[rb][cA]);
        }
        const V mp1_a = {MT::m(M, gp1_a.x), MT::m(M, gp1_a.y)};
        const V mp1_b = {MT::m(M, gp1_b.x), MT::m(M, gp1_b.y)};
        if (next) {
            stv(&SM[nb][ra][cA], mp1_a);
            stv(&SM[nb][rb][cA], mp1_b);
            if (hk_role) SM[nb][hr][hc] = MT::m(M, st[sn].G[hr][hc]);
            else if (hj_role) {
                const V hg = ldv(&st[sn].G[hr][hc]);
                stv(&SM[nb][hr][hc], V{MT::m(M, hg.x), MT::m(M, hg.y)});
            }
        }
        __syncthreads();
        if (tid == 0 && i > i0 && i - 1 + NS <= pend) issue(i - 1 + NS, sf);
        Faces Fn = F;
        if (next) Fn = faces(SM[nb], mp1_a, mp1_b);

        // ---- plane i ----
        const TmaStage<T>& S = st[s];
        const V uu = ldv(&S.U[rU][cA]);          // row above a
        const V ud = ldv(&S.U[rD][cA]);          // row below b
        const T uLa = S.U[ra][cL], uRa = S.U[ra][cR];
        const T uLb = S.U[rb][cL], uRb = S.U[rb][cR];
        const V pa = ldv(&S.P[2 * ty][2 * tx]), pb = ldv(&S.P[2 * ty + 1][2 * tx]);
        const V wh_a = {MT::face(m0_a.x, mp1_a.x), MT::face(m0_a.y, mp1_a.y)};
        const V wh_b = {MT::face(m0_b.x, mp1_b.x), MT::face(m0_b.y, mp1_b.y)};
        T kap[4];
        const T c0 = MT::coef(M, g0_a.x, kap[0]), c1 = MT::coef(M, g0_a.y, kap[1]);
        const T c2 = MT::coef(M, g0_b.x, kap[2]), c3 = MT::coef(M, g0_b.y, kap[3]);
        V oa, ob;
        cell(u0_a.x, up1_a.x, um_a.x, u0_b.x, uu.x, u0_a.y, uLa, wh_a.x, w0_a.x, F.jab.x, F.jlo.x,
             F.kIa, F.kLa, c0, pa.x, oa.x);
        cell(u0_a.y, up1_a.y, um_a.y, u0_b.y, uu.y, uRa, u0_a.x, wh_a.y, w0_a.y, F.jab.y, F.jlo.y,
             F.kRa, F.kIa, c1, pa.y, oa.y);
        cell(u0_b.x, up1_b.x, um_b.x, ud.x, u0_a.x, u0_b.y, uLb, wh_b.x, w0_b.x, F.jhi.x, F.jab.x,
             F.kIb, F.kLb, c2, pb.x, ob.x);
        cell(u0_b.y, up1_b.y, um_b.y, ud.y, u0_a.y, uRb, u0_b.x, wh_b.y, w0_b.y, F.jhi.y, F.jab.y,
             F.kRb, F.kIb, c3, pb.y, ob.y);

        // nodal injections, solver.py:167-170 (sources first, then support)
        if (my_src) {
            for (int q = 0; q < a.n_src; ++q) {
                if (!((my_src >> q) & 1u) || i != a.src_i[q]) continue;
                const int dj = a.src_j[q] - ja, dk = a.src_k[q] - kA;
                if (dj == 0 && dk == 0) oa.x = oa.x + MT::fc(M, g0_a.x, kap[0]) * a.src_val[q];
                if (dj == 0 && dk == 1) oa.y = oa.y + MT::fc(M, g0_a.y, kap[1]) * a.src_val[q];
                if (dj == 1 && dk == 0) ob.x = ob.x + MT::fc(M, g0_b.x, kap[2]) * a.src_val[q];
                if (dj == 1 && dk == 1) ob.y = ob.y + MT::fc(M, g0_b.y, kap[3]) * a.src_val[q];
            }
        }
        const long long oc = i * plane + cofs;
        if (SUP != SUP_NONE && i >= a.sup_lo && i <= a.sup_hi) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const unsigned long long flat = (unsigned long long)(oc + r * n2);
                const unsigned int w = __ldg(a.sup_mask + (flat >> 5));
                const unsigned int bit = (unsigned int)(flat & 31u);
                const unsigned int two = (w >> bit) & 3u;
                if (two) {
                    V& o = r ? ob : oa;
                    const V u = r ? u0_b : u0_a;
                    const V g = r ? g0_b : g0_a;
                    const int q = __ldg(a.sup_prefix + (flat >> 5)) +
                                  __popc(w & ((1u << bit) - 1u));
                    if (SUP == SUP_GATHER) {
                        if (two & 1u) a.trace_row[q] = u.x;
                        if (two & 2u) a.trace_row[q + (two & 1u)] = u.y;
                    } else {
                        if (two & 1u) o.x = o.x + MT::fc(M, g.x, kap[2 * r]) * ldg(a.adj_row + q);
                        if (two & 2u)
                            o.y = o.y + MT::fc(M, g.y, kap[2 * r + 1]) * ldg(a.adj_row + q + (two & 1u));
                    }
                }
            }
        }
        if (ACC) {
            const V aa = ldv(&S.A[2 * ty][2 * tx]), ab = ldv(&S.A[2 * ty + 1][2 * tx]);
            V na, nbv;
            na.x = kinc(aa.x, oa.x, pa.x, up1_a.x, um_a.x, u0_b.x, uu.x, u0_a.y, uLa);
            na.y = kinc(aa.y, oa.y, pa.y, up1_a.y, um_a.y, u0_b.y, uu.y, uRa, u0_a.x);
            nbv.x = kinc(ab.x, ob.x, pb.x, up1_b.x, um_b.x, ud.x, u0_a.x, u0_b.y, uLb);
            nbv.y = kinc(ab.y, ob.y, pb.y, up1_b.y, um_b.y, ud.y, u0_a.y, uRb, u0_b.x);
            stv(a.acc + oc, na);
            stv(a.acc + oc + n2, nbv);
        }
        stv(a.u_out + oc, oa);
        stv(a.u_out + oc + n2, ob);
        if (i < 2 && a.plo) { stv(a.plo + oc, oa); stv(a.plo + oc + n2, ob); }
        if (i >= a.n0 - 2 && a.phi) { stv(a.phi + oc, oa); stv(a.phi + oc + n2, ob); }
        if (CHECK) {
            typename Tr::Bits m1 = Tr::abs_bits(oa.x), m2 = Tr::abs_bits(oa.y);
            typename Tr::Bits m3 = Tr::abs_bits(ob.x), m4 = Tr::abs_bits(ob.y);
            m1 = m1 > m2 ? m1 : m2;
            m3 = m3 > m4 ? m3 : m4;
            m1 = m1 > m3 ? m1 : m3;
            local_max = m1 > local_max ? m1 : local_max;
        }
        // advance the queue
        um_a = u0_a; um_b = u0_b; u0_a = up1_a; u0_b = up1_b;
        g0_a = gp1_a; g0_b = gp1_b;
        m0_a = mp1_a; m0_b = mp1_b;
        w0_a = wh_a; w0_b = wh_b;
        F = Fn;
    };

    unsigned gpar = 0;
    for (int i = i0; i < i1; i += U) {
        unroll_planes(body, i, i1, gpar, std::make_integer_sequence<int, U>{});
        gpar ^= (unsigned)((U / NS) & 1);
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
            typename Tr::Bits v = lane < (T4_THREADS / 32) ? smax[lane] : 0;
            for (int o = 16; o > 0; o >>= 1) {
                typename Tr::Bits w = __shfl_xor_sync(0xffffffffu, v, o);
                v = w > v ? w : v;
            }
            if (lane == 0 && v) atomicMax(a.max_slot, v);
        }
    }
}

template <typename T>
constexpr size_t tma4_smem_bytes() {
    return NS * sizeof(TmaStage<T>) + 2 * sizeof(T) * TH_H * th_w<T>() +
           NS * sizeof(unsigned long long) + 128;
}

}  // namespace wb
