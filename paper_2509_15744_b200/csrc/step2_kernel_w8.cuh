// Two-step pass, 8-warp layout: the same algorithm, shared-memory ring and
// arithmetic as step2_kernel_tma (step2_kernel.cuh, read that first), with
// 256 threads per 64 x 8 tile — one row and two cells per thread instead of
// a 2 x 2 block.  Half the per-thread state, so more resident warps per SM to
// cover the TMA latency of the one-plane-ahead ring; each ring cell has its
// own thread (148 of 256).
#pragma once

#include "step2_kernel.cuh"

namespace wb {

#ifndef WB_T8_MINB
#define WB_T8_MINB 3
#endif
constexpr int T8_THREADS = 256;

template <typename T, int FLAVOR, bool ACC, int SUP>
__global__ void __launch_bounds__(T8_THREADS, sizeof(T) == 4 ? WB_T8_MINB : 1)
step2_kernel_w8(const __grid_constant__ Step2Args<T> a, const __grid_constant__ Tma2Maps maps) {
    using Tr = FTraits<T>;
    using MP = Mat<T, FLAVOR, false>;   // sparse force coefficients only
    using V = typename Pair<T>::V;
    using Bits = typename Tr::Bits;
    constexpr int W = th_w<T>(), HO = th_ho<T>();
    constexpr int PL = R2_H * W;
    extern __shared__ __align__(128) unsigned char smem_dyn[];
    unsigned char* smem_raw =
        smem_dyn + ((128u - (static_cast<unsigned>(__cvta_generic_to_shared(smem_dyn)) & 127u)) & 127u);
    Tma2Stage<T>* st = reinterpret_cast<Tma2Stage<T>*>(smem_raw);
    T* Xb = reinterpret_cast<T*>(smem_raw + T2_NS * sizeof(Tma2Stage<T>));   // X[2][PL]
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(Xb + T2_NX * PL);
    __shared__ Bits smax[2][T8_THREADS / 32];

    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    const int tid = ty * 32 + tx;
    const int k0 = blockIdx.x * PBX, j0 = blockIdx.y * BY;
    const int kA = k0 + 2 * tx, ja = j0 + ty;
    const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
    const int plane = n1 * n2;
    const int i0 = blockIdx.z * a.chunk;
    const int i1 = min(i0 + a.chunk, n0);
    const int pbeg = max(i0 - 1, 0);
    const int pfin = min(i1, n0 - 1);

    // offsets in the R2 frame; clamped (mirrored) neighbours at the grid edge
    const int ra = ty + 2, cA = HO + 2 * tx;
    const int rU = min(max(ja - 1, 0), n1 - 1) - j0 + 2;
    const int rD = min(max(ja + 1, 0), n1 - 1) - j0 + 2;
    const int dL = kA > 0 ? 1 : 0, dR = kA + 2 < n2 ? 1 : 0;
    const int oA = ra * W + cA;
    const int oU = rU * W + cA, oD = rD * W + cA;
    // ring cell of this thread (tid < NRING)
    int oR, rnb;
    bool rg_ok;
    {
        const int q = tid;
        int jj = j0, kk = k0;
        if (q < PBX + 2) { jj = j0 - 1; kk = k0 - 1 + q; }
        else if (q < 2 * (PBX + 2)) { jj = j0 + BY; kk = k0 - 1 + (q - (PBX + 2)); }
        else if (q < 2 * (PBX + 2) + BY) { jj = j0 + (q - 2 * (PBX + 2)); kk = k0 - 1; }
        else if (q < NRING) { jj = j0 + (q - 2 * (PBX + 2) - BY); kk = k0 + PBX; }
        rg_ok = q < NRING && jj >= 0 && jj < n1 && kk >= 0 && kk < n2;
        oR = rg_ok ? (jj - j0 + 2) * W + (kk - k0 + HO) : oA;
        rnb = (kk > 0 ? 1 : 0) | (kk < n2 - 1 ? 2 : 0) | (jj > 0 ? 4 : 0) | (jj < n1 - 1 ? 8 : 0);
    }
    const int rl = oR - (rnb & 1), rr = oR + ((rnb >> 1) & 1);
    const int ru = oR - W * ((rnb >> 2) & 1), rd = oR + W * ((rnb >> 3) & 1);

    unsigned my_src = 0;
    for (int s = 0; s < a.n_src; ++s)
        if (a.src_i[s] >= pbeg && a.src_i[s] <= pfin && a.src_j[s] >= j0 - 1 &&
            a.src_j[s] <= j0 + BY && a.src_k[s] >= k0 - 1 && a.src_k[s] <= k0 + PBX)
            my_src |= 1u << s;

    constexpr unsigned STAGE_BYTES =
        (unsigned)(sizeof(T) * ((2 * R2_H + 4 * R1_H) * W + (ACC ? BY * PBX : 0)));
    const CUtensorMap* mU = pick_map(maps.u_r2, maps.cur);
    const CUtensorMap* mP = pick_map(maps.u_r1, maps.prev);
    auto prefetch = [&](int p) {
        auto pf = [&](const CUtensorMap* m, int c0, int c1) {
            asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
                         ::"l"(reinterpret_cast<unsigned long long>(m)), "r"(c0), "r"(c1), "r"(p)
                         : "memory");
        };
        pf(mU, k0 - HO, j0 - 2);
        pf(&maps.fj_r2, k0 - HO, j0 - 2);
        pf(mP, k0 - HO, j0 - 1);
        pf(&maps.c_r1, k0 - HO, j0 - 1);
        pf(&maps.fk_r1, k0 - HO, j0 - 1);
        pf(&maps.fi_r1, k0 - HO, j0 - 1);
        if (ACC) pf(&maps.a_ctr, k0, j0);
    };
    auto issue = [&](int p, int s) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[s], STAGE_BYTES);
        tma_load_3d(&st[s].U[0][0], mU, k0 - HO, j0 - 2, p, &bar[s]);
        tma_load_3d(&st[s].FJ[0][0], &maps.fj_r2, k0 - HO, j0 - 2, p, &bar[s]);
        tma_load_3d(&st[s].P[0][0], mP, k0 - HO, j0 - 1, p, &bar[s]);
        tma_load_3d(&st[s].C[0][0], &maps.c_r1, k0 - HO, j0 - 1, p, &bar[s]);
        tma_load_3d(&st[s].FK[0][0], &maps.fk_r1, k0 - HO, j0 - 1, p, &bar[s]);
        tma_load_3d(&st[s].FI[0][0], &maps.fi_r1, k0 - HO, j0 - 1, p, &bar[s]);
        if (ACC) tma_load_3d(&st[s].A[0][0], &maps.a_ctr, k0, j0, p, &bar[s]);
    };
    constexpr int PRODUCER = 7 * 32;   // last warp: no ring cells
    if (tid == 0) {
        for (int s = 0; s < T2_NS; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == PRODUCER) {
        for (int s = 0; s < T2_NS && pbeg + s <= pfin; ++s) issue(pbeg + s, s);
        for (int d = 0; d < T2_PF && pbeg + T2_NS + d <= pfin; ++d) prefetch(pbeg + T2_NS + d);
    }

    auto ldv = [](const T* p) { return *reinterpret_cast<const V*>(p); };
    auto stv = [](T* p, V v) { *reinterpret_cast<V*>(p) = v; };
    auto cell = [&](T u0, T up1, T um1, T ujp, T ujm, T ukp, T ukm, T w0hi, T w0lo, T fjhi, T fjlo,
                    T fkhi, T fklo, T coef, T up) {
        T s = u0 - u0;
        s += (up1 - u0) * w0hi;
        s -= (u0 - um1) * w0lo;
        s += (ujp - u0) * fjhi;
        s -= (u0 - ujm) * fjlo;
        s += (ukp - u0) * fkhi;
        s -= (u0 - ukm) * fklo;
        return ((u0 + u0) - up) + coef * s;
    };
    auto kinc = [&](T accv, T out, T up, T up1, T um1, T ujp, T ujm, T ukp, T ukm) {
        const T va = (out - up) * a.inv2dt;
        const T g0 = (up1 - um1) * a.inv2dx;
        const T g1 = (ujp - ujm) * a.inv2dx;
        const T g2 = (ukp - ukm) * a.inv2dx;
        return accv + a.sdt * ((a.cv * va) * va + a.cg * (((g0 * g0) + (g1 * g1)) + (g2 * g2)));
    };
    auto fcoef = [&](int flat) {
        const T g = __ldg(a.gamma + flat);
        T kap;
        (void)MP::coef(a.mat, g, kap);
        return MP::fc(a.mat, g, kap);
    };
    auto inject_src = [&](int p, int jj, int kk, const T* val, T& o) {
        for (int q = 0; q < a.n_src; ++q)
            if (((my_src >> q) & 1u) && p == a.src_i[q] && jj == a.src_j[q] && kk == a.src_k[q])
                o = o + fcoef(p * plane + jj * n2 + kk) * val[q];
    };
    auto sup_index = [&](int p, int jj, int kk) -> int {
        if (SUP == SUP_NONE || p < a.sup_lo || p > a.sup_hi) return -1;
        const unsigned flat = (unsigned)(p * plane + jj * n2 + kk);
        const unsigned w = __ldg(a.sup_mask + (flat >> 5));
        const unsigned bit = flat & 31u;
        if (!((w >> bit) & 1u)) return -1;
        return __ldg(a.sup_prefix + (flat >> 5)) + __popc(w & ((1u << bit) - 1u));
    };
    auto tile_inject = [&](int p, V& o, V u, const T* val, T* row, bool gather_ok) {
        if (my_src) {
            inject_src(p, ja, kA, val, o.x);
            inject_src(p, ja, kA + 1, val, o.y);
        }
        if (SUP != SUP_NONE && p >= a.sup_lo && p <= a.sup_hi) {
            const T uo[2] = {u.x, u.y};
            T* oo[2] = {&o.x, &o.y};
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int kk = kA + c;
                const int qi = sup_index(p, ja, kk);
                if (qi >= 0) {
                    if (SUP == SUP_GATHER) { if (gather_ok) row[qi] = uo[c]; }
                    else *oo[c] = *oo[c] + fcoef(p * plane + ja * n2 + kk) * ldg(row + qi);
                }
            }
        }
    };

    // ---------------- prologue: plane pbeg ----------------
    const int cofs = ja * n2 + kA;
    const bool has_m0 = pbeg > 0;
    const int rgofs = [&] {
        const int r = oR / W, c = oR - r * W;
        return (r + j0 - 2) * n2 + (c + k0 - HO);
    }();
    V unm, w0 = {T(0), T(0)};
    T rum = T(0), rw0 = T(0);
    if (has_m0) {
        const int gm = (pbeg - 1) * plane;
        unm = __ldg(reinterpret_cast<const V*>(a.u_cur + gm + cofs));
        w0 = __ldg(reinterpret_cast<const V*>(a.fi + gm + cofs));
        if (rg_ok) {
            rum = __ldg(a.u_cur + gm + rgofs);
            rw0 = __ldg(a.fi + gm + rgofs);
        }
    }
    mbar_wait(&bar[0], 0u);
    V un0 = ldv(&st[0].U[0][0] + oA);
    T run0 = (&st[0].U[0][0])[oR];
    if (!has_m0) { unm = un0; rum = run0; }

    T f1_kL = T(0), f1_kI = T(0), f1_kR = T(0);
    V f1_jlo = {T(0), T(0)}, f1_jhi = f1_jlo, w1lo = f1_jlo, w1hi = f1_jlo, c1 = f1_jlo;
    V x_m1 = un0, x_0 = un0, un1 = unm, acc1 = {T(0), T(0)};
    Bits lmax1 = 0, lmax2 = 0;

    auto step2_tile = [&](int q1, const T* Xq, V xp) {
        const V xu = ldv(Xq + oU), xd = ldv(Xq + oD);
        const T xL = Xq[oA - dL], xR = Xq[oA + 1 + dR];
        V o2;
        o2.x = cell(x_0.x, xp.x, x_m1.x, xd.x, xu.x, x_0.y, xL, w1hi.x, w1lo.x, f1_jhi.x, f1_jlo.x,
                    f1_kI, f1_kL, c1.x, un1.x);
        o2.y = cell(x_0.y, xp.y, x_m1.y, xd.y, xu.y, xR, x_0.x, w1hi.y, w1lo.y, f1_jhi.y, f1_jlo.y,
                    f1_kR, f1_kI, c1.y, un1.y);
        tile_inject(q1, o2, x_0, a.src_val2, a.row2, true);
        const int oc = q1 * plane + cofs;
        if (ACC) {
            V f;
            f.x = kinc(acc1.x, o2.x, un1.x, xp.x, x_m1.x, xd.x, xu.x, x_0.y, xL);
            f.y = kinc(acc1.y, o2.y, un1.y, xp.y, x_m1.y, xd.y, xu.y, xR, x_0.x);
            stv(a.acc + oc, f);
        }
        stv(a.out1 + oc, x_0);
        stv(a.out2 + oc, o2);
        if (a.check2) {
            Bits m1 = Tr::abs_bits(o2.x), m2 = Tr::abs_bits(o2.y);
            m1 = m1 > m2 ? m1 : m2;
            lmax2 = m1 > lmax2 ? m1 : lmax2;
        }
    };

    auto body = [&](int q, int p, unsigned gpar) {
        const int sn = q + 1 == T2_NS ? 0 : q + 1, sf = q == 0 ? T2_NS - 1 : q - 1;
        const int b = (p - pbeg) & 1;
        const unsigned pn = (q + 1 == T2_NS) ? 1u : 0u;
        T* Xc = Xb + b * PL;
        const T* Xp = Xb + (b ^ 1) * PL;
        const Tma2Stage<T>& S = st[q];
        const T* SU = &S.U[0][0];
        const T* SFJ = &S.FJ[0][0];
        const T* SP = &S.P[0][0] - W;
        const T* SC = &S.C[0][0] - W;
        const T* SFK = &S.FK[0][0] - W;
        const T* SFI = &S.FI[0][0] - W;
        // ---- a: u^n of plane p+1 ----
        V unp = un0;
        T runp = run0;
        if (p + 1 <= pfin) {
            mbar_wait(&bar[sn], gpar ^ pn);
            const T* NU = &st[sn].U[0][0];
            unp = ldv(NU + oA);
            runp = NU[oR];
        } else if (p + 1 <= n0 - 1) {
            const int gp = (p + 1) * plane;
            unp = __ldg(reinterpret_cast<const V*>(a.u_cur + gp + cofs));
            if (rg_ok) runp = __ldg(a.u_cur + gp + rgofs);
        }
        __syncthreads();
        if (tid == PRODUCER && p > pbeg && p + T2_NS - 1 <= pfin) {
            issue(p + T2_NS - 1, sf);
            if (p + T2_NS - 1 + T2_PF <= pfin) prefetch(p + T2_NS - 1 + T2_PF);
        }

        // ---- d: step n at plane p (tile + ring) -> X[b] ----
        const V wh = ldv(SFI + oA), cf = ldv(SC + oA), fk = ldv(SFK + oA);
        const T kL = SFK[oA - dL];
        const V jlo = ldv(SFJ + oU), jhi = ldv(SFJ + oA);
        const V uu = ldv(SU + oU), ud = ldv(SU + oD);
        const T uL = SU[oA - dL], uR = SU[oA + 1 + dR];
        const V pa = ldv(SP + oA);
        V o;
        o.x = cell(un0.x, unp.x, unm.x, ud.x, uu.x, un0.y, uL, wh.x, w0.x, jhi.x, jlo.x, fk.x, kL,
                   cf.x, pa.x);
        o.y = cell(un0.y, unp.y, unm.y, ud.y, uu.y, uR, un0.x, wh.y, w0.y, jhi.y, jlo.y, fk.y, fk.x,
                   cf.y, pa.y);
        const bool own_plane = p >= i0 && p < i1;
        tile_inject(p, o, un0, a.src_val1, a.row1, own_plane);
        stv(Xc + oA, o);
        V nacc = acc1;
        if (own_plane) {
            if (ACC) {
                const V av = ldv(&S.A[ty][2 * tx]);
                nacc.x = kinc(av.x, o.x, pa.x, unp.x, unm.x, ud.x, uu.x, un0.y, uL);
                nacc.y = kinc(av.y, o.y, pa.y, unp.y, unm.y, ud.y, uu.y, uR, un0.x);
            }
            if (a.check1) {
                Bits m1 = Tr::abs_bits(o.x), m2 = Tr::abs_bits(o.y);
                m1 = m1 > m2 ? m1 : m2;
                lmax1 = m1 > lmax1 ? m1 : lmax1;
            }
        }
        // ring cell (step n only)
        T rwh = rw0;
        if (rg_ok) {
            rwh = SFI[oR];
            T v = cell(run0, runp, rum, SU[rd], SU[ru], SU[rr], SU[rl], rwh, rw0, SFJ[oR], SFJ[ru],
                       SFK[oR], SFK[rl], SC[oR], SP[oR]);
            if (my_src || SUP == SUP_INJECT) {
                const int r = oR / W;
                const int jj = r + j0 - 2, kk = oR - r * W + k0 - HO;
                if (my_src) inject_src(p, jj, kk, a.src_val1, v);
                if (SUP == SUP_INJECT) {
                    const int qi = sup_index(p, jj, kk);
                    if (qi >= 0) v = v + fcoef(p * plane + jj * n2 + kk) * ldg(a.row1 + qi);
                }
            }
            Xc[oR] = v;
        }

        // ---- c: step n+1 at plane p-1 ----
        if (p - 1 >= i0 && p - 1 < i1) step2_tile(p - 1, Xp, o);

        // ---- rotate ----
        f1_kL = kL; f1_kI = fk.x; f1_kR = fk.y;
        f1_jlo = jlo; f1_jhi = jhi;
        w1lo = w0; w1hi = wh; c1 = cf;
        acc1 = nacc;
        un1 = un0;
        x_m1 = p == 0 ? o : x_0;
        x_0 = o;
        unm = un0; un0 = unp;
        w0 = wh;
        rw0 = rwh; rum = run0; run0 = runp;
    };

    unsigned gpar = 0;
    for (int p = pbeg, q = 0; p <= pfin; ++p) {
        body(q, p, gpar);
        if (++q == T2_NS) { q = 0; gpar ^= 1u; }
    }
    __syncthreads();
    if (pfin == i1 - 1) step2_tile(pfin, Xb + ((pfin - pbeg) & 1) * PL, x_0);

    if (a.check1 || a.check2) {
        for (int o = 16; o > 0; o >>= 1) {
            Bits v1 = __shfl_xor_sync(0xffffffffu, lmax1, o);
            Bits v2 = __shfl_xor_sync(0xffffffffu, lmax2, o);
            lmax1 = v1 > lmax1 ? v1 : lmax1;
            lmax2 = v2 > lmax2 ? v2 : lmax2;
        }
        const int lane = tid & 31, warp = tid >> 5;
        if (lane == 0) { smax[0][warp] = lmax1; smax[1][warp] = lmax2; }
        __syncthreads();
        if (warp == 0) {
            Bits v1 = lane < (T8_THREADS / 32) ? smax[0][lane] : 0;
            Bits v2 = lane < (T8_THREADS / 32) ? smax[1][lane] : 0;
            for (int o = 16; o > 0; o >>= 1) {
                Bits w1 = __shfl_xor_sync(0xffffffffu, v1, o);
                Bits w2 = __shfl_xor_sync(0xffffffffu, v2, o);
                v1 = w1 > v1 ? w1 : v1;
                v2 = w2 > v2 ? w2 : v2;
            }
            if (lane == 0) {
                if (a.check1 && v1) atomicMax(a.max1, v1);
                if (a.check2 && v2) atomicMax(a.max2, v2);
            }
        }
    }
}

}  // namespace wb
