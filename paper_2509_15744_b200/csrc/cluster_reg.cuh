// Register-resident whole sweeps of small 2D grids: one thread-block cluster
// of up to 16 CTAs runs all N steps of a sweep in ONE launch, every field in
// registers.
//
// The first cluster engine (cluster_sweep.cuh) kept the window, coef, the
// faces and the accumulator in shared memory: ~14 shared-memory accesses and
// a scalar, branchy stencil per cell left it at ~4.7 us per step for C1
// (2D 256^2, N = 3200), slower than 148-SM two-step launches.
// Here thread t of CTA r owns a 2 x 2PC block of cells (rows r0, r0+1 of the
// CTA's R rows; PC packed pairs of columns, PC = 2 by default: 512 threads)
// and keeps u^{n-1}, u^n and the accumulator of its cells in registers as
// packed pairs (fp32: one f32x2 register per pair, FADD2 / FFMA2; fp64: two
// doubles), coef and the face weights in registers (fp32) or in a
// thread-major shared-memory table (fp64).  Per step:
//   1. publish u^n of the own block into the exchange plane X[n & 1] (the
//      grid-edge threads also write their mirror copies into the pad / halo
//      slots); the CTA's first / last row-pair pushes its boundary row into
//      the neighbour CTA's halo row with st.async (complete_tx on the
//      receiver's mbarrier); source amplitudes and adjoint forces are
//      prefetched with cp.async
//   2. one __syncthreads; the boundary row-pairs wait on the halo mbarrier.
//      X is double-buffered, so a plane is rewritten two steps later, after
//      every reader has published the step in between (no cluster barrier)
//   3. per packed pair: neighbours from registers / X, stencil, sources,
//      adjoint injection, self-kernel increment; trace gather and the
//      stability max — in the reference's per-cell operation order
//      (kernels.py:30-44, solver.py:154-186, gradients.py:237, 268,
//      kernels.py:86-102), so results are bit-identical to the step kernels.
//      A face leading out of the grid has weight 0 and its neighbour is
//      mirrored (u - u = +0), bit-identical to skipping the term
//      (step_kernel.cuh).
// The window and the accumulator go back to global memory at the end.
#pragma once

#include "cluster_sweep.cuh"
#include "tma_common.cuh"

namespace wb {

constexpr int CR_THREADS = 1024;

// Packed pairs: the two cells of a block row run the same IEEE sequence.
template <typename T> struct CR2;
template <> struct CR2<float> {
    using V = unsigned long long;
    __device__ static __forceinline__ V mk(float lo, float hi) {
        V r;
        asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
        return r;
    }
    __device__ static __forceinline__ float lo(V v) {
        float a;
        asm("{\n.reg .f32 t;\nmov.b64 {%0, t}, %1;\n}" : "=f"(a) : "l"(v));
        return a;
    }
    __device__ static __forceinline__ float hi(V v) {
        float b;
        asm("{\n.reg .f32 t;\nmov.b64 {t, %0}, %1;\n}" : "=f"(b) : "l"(v));
        return b;
    }
    __device__ static __forceinline__ V add(V a, V b) {
        V r;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
        return r;
    }
    __device__ static __forceinline__ V sub(V a, V b) {
        V r;
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
        return r;
    }
    // exact product: fma with a (-0, -0) addend from a kernel argument
    // (ptxas would contract mul.rn.f32x2 + add.rn.f32x2, see step2_kernel.cuh)
    __device__ static __forceinline__ V mul(V a, V b, V negz) {
        V r;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(negz));
        return r;
    }
    __device__ static __forceinline__ V lds(unsigned addr) {
        V r;
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(r) : "r"(addr) : "memory");
        return r;
    }
    __device__ static __forceinline__ float lds1(unsigned addr) {
        float r;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(addr) : "memory");
        return r;
    }
    __device__ static __forceinline__ void sts(unsigned addr, V v) {
        asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
    }
    __device__ static __forceinline__ void sts1(unsigned addr, float v) {
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
    }
    // store into a cluster peer's shared memory, completing bytes on its mbarrier
    __device__ static __forceinline__ void push(unsigned addr, V v, unsigned mbar) {
        asm volatile(
            "st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr),
            "l"(v), "r"(mbar)
            : "memory");
    }
};
template <> struct CR2<double> {
    struct V {
        double x, y;
    };
    __device__ static __forceinline__ V mk(double lo, double hi) { return V{lo, hi}; }
    __device__ static __forceinline__ double lo(V v) { return v.x; }
    __device__ static __forceinline__ double hi(V v) { return v.y; }
    __device__ static __forceinline__ V add(V a, V b) { return V{a.x + b.x, a.y + b.y}; }
    __device__ static __forceinline__ V sub(V a, V b) { return V{a.x - b.x, a.y - b.y}; }
    __device__ static __forceinline__ V mul(V a, V b, V) { return V{a.x * b.x, a.y * b.y}; }
    __device__ static __forceinline__ V lds(unsigned addr) {
        V r;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(addr) : "memory");
        return r;
    }
    __device__ static __forceinline__ double lds1(unsigned addr) {
        double r;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(addr) : "memory");
        return r;
    }
    __device__ static __forceinline__ void sts(unsigned addr, V v) {
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
    }
    __device__ static __forceinline__ void sts1(unsigned addr, double v) {
        asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
    }
    __device__ static __forceinline__ void push(unsigned addr, V v, unsigned mbar) {
        asm volatile(
            "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                addr),
            "d"(v.x), "d"(v.y), "r"(mbar)
            : "memory");
    }
};

// one element global -> shared, asynchronous (LDGSTS)
template <typename E> __device__ __forceinline__ void cp_async_el(E* dst, const E* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d), "l"(src), "n"(sizeof(E))
                 : "memory");
}

// Thread block of PC packed pairs per row: 2 x 2*PC cells, CR_THREADS / PC
// threads per CTA.  rows per CTA must be even; threads = ceil(n2 / (2 PC)) *
// rows / 2 <= CR_THREADS / PC.
template <int PC> __host__ __device__ constexpr int cr_threads() { return CR_THREADS / PC; }
__host__ __device__ constexpr int cr_txn(int n2, int pc) { return (n2 + 2 * pc - 1) / (2 * pc); }
template <typename T> __host__ __device__ constexpr bool cluster_reg_mreg() {
    return sizeof(T) == 4;   // fp32: material in registers
}
template <typename T>
__host__ __device__ constexpr size_t cluster_reg_smem(int rows, int n2, long long sup_cap, int pc) {
    const size_t W = (size_t)cr_txn(n2, pc) * 2 * pc + 4;   // exchange row stride (2 pad columns each side)
    const size_t nthr = (size_t)cr_txn(n2, pc) * (rows / 2);
    return 16 + sizeof(T) * 2 * (size_t)(rows + 2) * W                  // mbarriers, X[2][R+2][W]
           + (cluster_reg_mreg<T>() ? 0 : 9 * pc * nthr * 2 * sizeof(T))   // fp64 material table
           + (size_t)sup_cap * (sizeof(int) + 2 * sizeof(T))               // support slots, forces
           + MAX_SRC * (sizeof(T) + sizeof(double)) + 16;                  // source fc / amp, counter
}

template <typename T, int FLAVOR, bool ACC, int PC, bool FULL>
__global__ void __launch_bounds__(CR_THREADS / PC, 1) cluster_reg_kernel(const ClusterSweepArgs<T> a) {
    using P = Mat<T, FLAVOR, false>;
    using O = CR2<T>;
    using V = typename O::V;
    using Bits = typename FTraits<T>::Bits;
    constexpr bool MREG = cluster_reg_mreg<T>();
    constexpr int CW = 2 * PC;                            // columns per thread
    extern __shared__ __align__(16) unsigned char cr_smem[];
    const int n1 = a.n1, n2 = a.n2, R = a.rows;
    const int TXN = cr_txn(n2, PC), W = CW * TXN;
    // exchange row: 2 pad columns each side (mirror copies of the edge
    // columns at columns 1 and W + 2), own columns from column 2 (V-aligned)
    const int XW = W + 4;
    const int nthr = TXN * (R / 2);
    const unsigned rank = cs_rank(), nranks = cs_nranks();
    const int j0 = (int)rank * R;
    const int tid = threadIdx.x;
    const bool live = tid < nthr;
    const int ty = live ? tid / TXN : 0, tx = live ? tid - ty * TXN : 0;
    const int r0 = 2 * ty, c0 = CW * tx;
    const int mtid = live ? tid : 0;                      // material table row (fp64)
    const int ja = j0 + r0, jb = ja + 1;                 // grid rows of the block
    const bool acta = live && ja < n1, actb = live && jb < n1;
    // X[2][R + 2][W]: own rows 0..R-1 at rows 1..R, the neighbours' boundary
    // rows (pushed by them) at rows 0 and R + 1
    unsigned long long* MB = reinterpret_cast<unsigned long long*>(cr_smem);   // [2]
    T* X0 = reinterpret_cast<T*>(cr_smem + 16);
    const int XS = (R + 2) * XW;                          // one exchange buffer
    V* MT = reinterpret_cast<V*>(X0 + 2 * XS);            // fp64: [9 PC][nthr]
    int* SQ = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(MT) +
                                     (MREG ? 0 : 9 * PC * (size_t)nthr * sizeof(V)));
    T* SFC = reinterpret_cast<T*>(SQ + a.sup_cap);
    // sup_cap ints then sup_cap T: T-aligned because sup_cap is rounded to even
    T* SFV = SFC + a.sup_cap;                             // this step's adjoint forces
    double* SAMP = reinterpret_cast<double*>(SFV + a.sup_cap);   // this step's amplitudes
    T* SRCFC = reinterpret_cast<T*>(SAMP + MAX_SRC);
    int* counter = reinterpret_cast<int*>(SRCFC + MAX_SRC);
    const V nz = *reinterpret_cast<const V*>(&a.negz2);

    if (tid == 0) {
        *counter = 0;
        mbar_init(MB, 1);
        mbar_init(MB + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // ---- prologue: material (the operations of solver.py:89-119), window ----
    auto mg = [&](int j, int k) { return P::m(a.mat, __ldg(a.gamma + (long long)j * n2 + k)); };
    auto face = [&](bool in, int jl, int kl, int jh, int kh) {
        return in ? P::face(mg(jl, kl), mg(jh, kh)) : T(0);
    };
    // material fields (MT index): co[i][p] i*PC+p, wkl 2PC+.., wkr 4PC+.., wj[k][p] 6PC+k*PC+p
    V co[2][PC], wkl[2][PC], wkr[2][PC], wj[3][PC];   // wj: above row a, between a and b, below b
    V up[2][PC], uc[2][PC], ac[2][PC];
#pragma unroll
    for (int p = 0; p < PC; ++p) {
        const int cp = c0 + 2 * p;
        const bool cx = cp < n2, cy = cp + 1 < n2;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int j = ja + i;
            const bool in = i == 0 ? acta : actb;
            T kx = 0, ky = 0;
            if (in) {
                T kap;
                if (cx) kx = P::coef(a.mat, __ldg(a.gamma + (long long)j * n2 + cp), kap);
                if (cy) ky = P::coef(a.mat, __ldg(a.gamma + (long long)j * n2 + cp + 1), kap);
            }
            co[i][p] = O::mk(kx, ky);
            wkl[i][p] = O::mk(face(in && cx && cp > 0, j, cp - 1, j, cp), face(in && cy, j, cp, j, cp + 1));
            wkr[i][p] = O::mk(face(in && cy, j, cp, j, cp + 1),
                              face(in && cp + 2 < n2, j, cp + 1, j, cp + 2));
            const long long g = (long long)j * n2 + cp;
            up[i][p] = O::mk(in && cx ? a.u_prev_in[g] : T(0), in && cy ? a.u_prev_in[g + 1] : T(0));
            uc[i][p] = O::mk(in && cx ? a.u_cur_in[g] : T(0), in && cy ? a.u_cur_in[g + 1] : T(0));
            ac[i][p] = O::mk(ACC && in && cx ? a.acc[g] : T(0), ACC && in && cy ? a.acc[g + 1] : T(0));
        }
        wj[0][p] = O::mk(face(acta && cx && ja > 0, ja - 1, cp, ja, cp),
                         face(acta && cy && ja > 0, ja - 1, cp + 1, ja, cp + 1));
        wj[1][p] = O::mk(face(actb && cx, ja, cp, jb, cp), face(actb && cy, ja, cp + 1, jb, cp + 1));
        wj[2][p] = O::mk(face(actb && cx && jb + 1 < n1, jb, cp, jb + 1, cp),
                         face(actb && cy && jb + 1 < n1, jb, cp + 1, jb + 1, cp + 1));
        if (!MREG && live) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                MT[(i * PC + p) * nthr + tid] = co[i][p];
                MT[(2 * PC + i * PC + p) * nthr + tid] = wkl[i][p];
                MT[(4 * PC + i * PC + p) * nthr + tid] = wkr[i][p];
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) MT[(6 * PC + k * PC + p) * nthr + tid] = wj[k][p];
        }
    }
    __syncthreads();   // slot counter initialised

    // support cells of the block: bit i * CW + c (row i, column c0 + c), slots sbase..
    const bool has_sup = a.sup_mode != SUP_NONE && a.n_sup > 0;
    unsigned smask = 0;
    int sbase = 0;
    if (has_sup && live) {
        int nb = 0;
        for (int e = 0; e < 2 * CW; ++e) {
            const int j = ja + e / CW, k = c0 + e % CW;
            if (j < n1 && k < n2) {
                const long long g = (long long)j * n2 + k;
                if ((__ldg(a.sup_mask + (g >> 5)) >> (g & 31)) & 1u) {
                    smask |= 1u << e;
                    ++nb;
                }
            }
        }
        if (smask) {
            sbase = atomicAdd(counter, nb);
            int s = sbase;
            for (int e = 0; e < 2 * CW; ++e)
                if ((smask >> e) & 1u) {
                    const long long g = (long long)(ja + e / CW) * n2 + c0 + e % CW;
                    const unsigned w = __ldg(a.sup_mask + (g >> 5)), bit = (unsigned)(g & 31);
                    const T gam = __ldg(a.gamma + g);
                    T kap;
                    (void)P::coef(a.mat, gam, kap);
                    SQ[s] = __ldg(a.sup_prefix + (g >> 5)) + __popc(w & ((1u << bit) - 1u));
                    SFC[s] = P::fc(a.mat, gam, kap);
                    ++s;
                }
        }
    }
    // sources in the block (bit q), their force coefficients
    unsigned tsrc = 0;
    for (int s = 0; s < a.n_src; ++s) {
        const int dj = a.src_j[s] - ja, dk = a.src_k[s] - c0;
        if (live && dj >= 0 && dj < 2 && dk >= 0 && dk < CW && a.src_j[s] < n1 && a.src_k[s] < n2) {
            tsrc |= 1u << s;
            const T gam = __ldg(a.gamma + (long long)a.src_j[s] * n2 + a.src_k[s]);
            T kap;
            (void)P::coef(a.mat, gam, kap);
            SRCFC[s] = P::fc(a.mat, gam, kap);
        }
    }

    // boundary rows: the first row-pair pushes its row a into the upper
    // neighbour's row R + 1, the last one its row b into the lower
    // neighbour's row 0 (st.async + complete_tx on the receiver's mbarrier).
    // A CTA's shared window is contiguous in the cluster window, so buffer 1
    // of a remote X is buffer 0 plus XS elements.
    const bool send_up = live && ty == 0 && rank > 0;
    const bool send_dn = live && ty == R / 2 - 1 && rank + 1 < nranks;
    const unsigned rx_up = send_up ? cs_remote(X0 + (R + 1) * XW + 2 + c0, rank - 1) : 0u;
    const unsigned rb_up = send_up ? cs_remote(MB, rank - 1) : 0u;
    const unsigned rx_dn = send_dn ? cs_remote(X0 + 2 + c0, rank + 1) : 0u;
    const unsigned rb_dn = send_dn ? cs_remote(MB, rank + 1) : 0u;
    const unsigned xs_bytes = (unsigned)(XS * sizeof(T));
    const unsigned rx_bytes =
        (unsigned)(((rank > 0) + (rank + 1 < nranks)) * W * sizeof(T));   // pushed to me per step
    const bool recv = live && ((ty == 0 && rank > 0) || (ty == R / 2 - 1 && rank + 1 < nranks));
    const int oa = (r0 + 1) * XW + 2 + c0, ob = oa + XW;
    cs_cluster_sync();   // every mbarrier initialised before the first push

    // pairs (bit i * PC + p) with an injection (a source, or an adjoint
    // support cell): injected right after their stencil, before the kernel
    // increment; support cells of a gathering sweep only store their u^n
    const bool inject = a.sup_mode == SUP_INJECT;
    const unsigned gmask = inject ? 0u : smask;
    unsigned pmask = 0;
#pragma unroll
    for (int e = 0; e < 2 * CW; ++e)
        if (inject && ((smask >> e) & 1u)) pmask |= 1u << (e / CW * PC + (e % CW) / 2);
    for (unsigned bb = tsrc; bb; bb &= bb - 1) {
        const int q = __ffs(bb) - 1;
        pmask |= 1u << ((a.src_j[q] - ja) * PC + (a.src_k[q] - c0) / 2);
    }
    const bool special = (pmask | gmask) != 0;
    // opaque to the compiler, so it stays in a register instead of being
    // rematerialised (S2R SR_CgaCtaId + LEA) at every use
    unsigned xs0, mt0;
    asm volatile("mov.u32 %0, %1;" : "=r"(xs0) : "r"(smem_addr(X0)));
    asm volatile("mov.u32 %0, %1;" : "=r"(mt0) : "r"(smem_addr(MT)));
    const bool top = acta && ja == 0, bot = actb && jb + 1 == n1;   // mirror rows to publish
    const bool medge = live && c0 == 0, pedge = live && FULL && c0 + CW == n2;
    const int nlast = a.backward ? 1 : (int)a.N - 1;      // stability check positions
    const V i2t = O::mk(a.inv2dt, a.inv2dt), i2x = O::mk(a.inv2dx, a.inv2dx);
    const V cvv = O::mk(a.cv, a.cv), cgv = O::mk(a.cg, a.cg), sdv = O::mk(a.sdt, a.sdt);
    Bits lmax = 0;
    for (int it = 0; it < a.n_count; ++it) {
        const int n = a.backward ? a.n_first - it : a.n_first + it;
        const int b = it & 1;
        const unsigned xb = xs0 + b * xs_bytes;          // X[b], shared-space address
        auto xa = [&](int off) { return xb + off * (unsigned)sizeof(T); };
        // ---- 1: publish u^n (own plane, neighbours' halo rows); prefetch
        //      this step's forces / amplitudes ----
        // rows beyond the grid publish nothing: the slot below the grid's
        // last row holds that row's mirror copy (a partial last CTA)
        if (acta) {
#pragma unroll
            for (int p = 0; p < PC; ++p) {
                O::sts(xa(oa + 2 * p), uc[0][p]);
                // mirrored neighbours of the grid's edge cells (u - u = +0)
                if (top) O::sts(xa(oa - XW + 2 * p), uc[0][p]);
            }
            if (medge) O::sts1(xa(oa - 1), O::lo(uc[0][0]));
            if (pedge) O::sts1(xa(oa + CW), O::hi(uc[0][PC - 1]));
        }
        if (actb) {
#pragma unroll
            for (int p = 0; p < PC; ++p) {
                O::sts(xa(ob + 2 * p), uc[1][p]);
                if (bot) O::sts(xa(ob + XW + 2 * p), uc[1][p]);
            }
            if (medge) O::sts1(xa(ob - 1), O::lo(uc[1][0]));
            if (pedge) O::sts1(xa(ob + CW), O::hi(uc[1][PC - 1]));
        }
#pragma unroll
        for (int p = 0; p < PC; ++p) {
            if (send_up) O::push(rx_up + b * xs_bytes + 2 * p * sizeof(T), uc[0][p], rb_up + b * 8);
            if (send_dn) O::push(rx_dn + b * xs_bytes + 2 * p * sizeof(T), uc[1][p], rb_dn + b * 8);
        }
        if (tid == 0) mbar_expect_tx(MB + b, rx_bytes);
        if (special) {   // asynchronous copies into shared memory, latency hidden by the barrier
            const T* srow = a.store + (long long)n * a.n_sup;
            if (a.sup_mode == SUP_INJECT)
                for (int s = sbase; s < sbase + __popc(smask); ++s) cp_async_el(SFV + s, srow + SQ[s]);
            for (unsigned bb = tsrc; bb; bb &= bb - 1) {
                const int q = __ffs(bb) - 1;
                cp_async_el(SAMP + q, a.src_amp + (long long)q * a.N + n);
            }
        }
        // ---- 2: plane n visible in the CTA, the neighbours' rows arrived ----
        __syncthreads();
        if (recv) mbar_wait(MB + b, (it >> 1) & 1);
        if (special) {
            asm volatile("cp.async.wait_all;" ::: "memory");
            if (gmask) {   // trace entries n = u^n (gradients.py:237)
                T* srow = a.store + (long long)n * a.n_sup;
                int s0 = sbase;
#pragma unroll
                for (int e = 0; e < 2 * CW; ++e)
                    if ((gmask >> e) & 1u) {
                        const V u = uc[e / CW][(e % CW) / 2];
                        srow[SQ[s0++]] = (e & 1) ? O::hi(u) : O::lo(u);
                    }
            }
        }
        // neighbours of pair p in row i: rows from registers / X, columns
        // from registers / X, mirrored at the grid edge
        auto nbrs = [&](int i, int p, V& ujm, V& ujp, V& ukm, V& ukp) {
            const int cp = c0 + 2 * p;
            const V u = uc[i][p];
            if (i == 0) {
                ujm = O::lds(xa(oa - XW + 2 * p));
                ujp = actb ? uc[1][p] : u;
            } else {
                ujm = uc[0][p];
                ujp = O::lds(xa(ob + XW + 2 * p));
            }
            const int o = i == 0 ? oa : ob;
            const T xl = p > 0 ? O::hi(uc[i][p - 1]) : O::lds1(xa(o - 1));
            T yr;
            if (FULL)
                yr = p + 1 < PC ? O::lo(uc[i][p + 1]) : O::lds1(xa(o + CW));
            else
                yr = cp + 2 < n2 ? (p + 1 < PC ? O::lo(uc[i][p + 1]) : O::lds1(xa(o + CW))) : O::hi(u);
            ukm = O::mk(xl, O::lo(u));
            ukp = O::mk(FULL || cp + 1 < n2 ? O::hi(u) : O::lo(u), yr);
        };
        // self-kernel increment (kernels.py:86-102); the absent axis 0
        // contributes (0*0) + ... = the 2D sum exactly
        auto kinc = [&](int i, int p, V unew, V ujm, V ujp, V ukm, V ukp) {
            const V va = O::mul(O::sub(unew, up[i][p]), i2t, nz);
            const V gj = O::mul(O::sub(ujp, ujm), i2x, nz);
            const V gk = O::mul(O::sub(ukp, ukm), i2x, nz);
            const V inc = O::add(O::mul(O::mul(cvv, va, nz), va, nz),
                                 O::mul(cgv, O::add(O::mul(gj, gj, nz), O::mul(gk, gk, nz)), nz));
            ac[i][p] = O::add(ac[i][p], O::mul(sdv, inc, nz));
        };
        // ---- 3: stencil of the 2 x CW cells (kernels.py:30-44), injections,
        //      kernel increment ----
        V nu[2][PC];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int p = 0; p < PC; ++p) {
                V ujm, ujp, ukm, ukp;
                nbrs(i, p, ujm, ujp, ukm, ukp);
                const V u = uc[i][p];
                // fp64: the material comes from the shared table right where it is used
                auto mt = [&](int f, const V& r) {
                    return MREG ? r : O::lds(mt0 + (unsigned)((f * nthr + mtid) * sizeof(V)));
                };
                const V wa = mt(6 * PC + i * PC + p, wj[i][p]);            // face above
                const V wb = mt(6 * PC + (i + 1) * PC + p, wj[i + 1][p]);  // face below
                V s = O::sub(u, u);
                s = O::add(s, O::mul(O::sub(ujp, u), wb, nz));
                s = O::sub(s, O::mul(O::sub(u, ujm), wa, nz));
                s = O::add(s, O::mul(O::sub(ukp, u), mt(4 * PC + i * PC + p, wkr[i][p]), nz));
                s = O::sub(s, O::mul(O::sub(u, ukm), mt(2 * PC + i * PC + p, wkl[i][p]), nz));
                nu[i][p] = O::add(O::sub(O::add(u, u), up[i][p]), O::mul(mt(i * PC + p, co[i][p]), s, nz));
                if ((pmask >> (i * PC + p)) & 1u) {
                    // nodal sources, then the support (solver.py:167-170), per cell
                    T v[2] = {O::lo(nu[i][p]), O::hi(nu[i][p])};
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int j = ja + i, k = c0 + 2 * p + h, e = i * CW + 2 * p + h;
                        for (unsigned bb = tsrc; bb; bb &= bb - 1) {
                            const int q = __ffs(bb) - 1;
                            if (a.src_j[q] == j && a.src_k[q] == k) v[h] = v[h] + SRCFC[q] * (T)SAMP[q];
                        }
                        if (inject && ((smask >> e) & 1u)) {   // adjoint force (gradients.py:268)
                            const int s0 = sbase + __popc(smask & ((1u << e) - 1u));
                            v[h] = v[h] + SFC[s0] * SFV[s0];
                        }
                    }
                    nu[i][p] = O::mk(v[0], v[1]);
                }
                if (ACC) kinc(i, p, nu[i][p], ujm, ujp, ukm, ukp);
            }
        if (n % 50 == 0 || n == nlast) {   // stability max (solver.py:180-186), block-uniform
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int p = 0; p < PC; ++p) {
                    const bool in = i == 0 ? acta : actb;
                    const int cp = c0 + 2 * p;
                    if (in && cp < n2) lmax = max(lmax, FTraits<T>::abs_bits(O::lo(nu[i][p])));
                    if (in && cp + 1 < n2) lmax = max(lmax, FTraits<T>::abs_bits(O::hi(nu[i][p])));
                }
            for (int d = 16; d > 0; d >>= 1) {
                const Bits v = __shfl_xor_sync(0xffffffffu, lmax, d);
                lmax = v > lmax ? v : lmax;
            }
            if ((tid & 31) == 0 && lmax) atomicMax(a.maxslots + n, lmax);
            lmax = 0;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int p = 0; p < PC; ++p) {
                up[i][p] = uc[i][p];
                uc[i][p] = nu[i][p];
            }
    }
    cs_cluster_sync();   // no CTA leaves with a push into it in flight

    // ---- epilogue: window (prev, cur) and the accumulator to global ----
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const bool in = i == 0 ? acta : actb;
        if (!in) continue;
#pragma unroll
        for (int p = 0; p < PC; ++p) {
            const int cp = c0 + 2 * p;
            const long long g = (long long)(ja + i) * n2 + cp;
            if (cp < n2) {
                a.u_prev_out[g] = O::lo(up[i][p]);
                a.u_cur_out[g] = O::lo(uc[i][p]);
                if (ACC) a.acc[g] = O::lo(ac[i][p]);
            }
            if (cp + 1 < n2) {
                a.u_prev_out[g + 1] = O::hi(up[i][p]);
                a.u_cur_out[g + 1] = O::hi(uc[i][p]);
                if (ACC) a.acc[g + 1] = O::hi(ac[i][p]);
            }
        }
    }
}

}  // namespace wb
