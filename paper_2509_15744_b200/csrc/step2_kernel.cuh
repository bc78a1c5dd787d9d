// Two time steps per HBM pass (temporal blocking) on whole-tile grids.
//
// One launch advances the window by TWO steps, n and n+1 (forward: n, n+1;
// backward: n, n-1), each with the exact per-cell arithmetic of step_kernel
// (stencil, injections, support gather/inject, self-kernel increment,
// stability max — see step_kernel.cuh for the reference mapping and the
// mirrored-boundary argument).
//
// Material: the face weights and coef are time-invariant, so a one-off pass
// (material4_kernel) stores them — coef, the +k, +j and +i face weights of
// every cell, computed with the same operations the single-step kernel
// applies to gamma (solver.py:93-119) — and this kernel streams them instead
// of recomputing reciprocals: its dense arithmetic is only the face sum and
// the kernel increment.  A face leading out of the grid is stored as 0; it
// only ever multiplies a mirrored difference (u - u) = 0.
//
// Per plane p of the 2.5D march (TMA ring of T2_NS stages, one barrier):
//   a  wait for plane p+1; u^n(p+1) of the tile + ring (registers)
//   d  step n at plane p on the tile AND a one-cell ring around it (the ring
//      is recomputed redundantly so step n+1 never needs another CTA's data);
//      u^{n+1}(p) goes to a shared-memory plane X
//   b  __syncthreads; refill the stage of plane p with plane p+T2_NS
//   c  step n+1 at plane p-1 on the tile, from X(p-1), the register queue of
//      u^{n+1}, and plane p-1's material kept in registers
// HBM traffic per fp32 cell and pass: read u^{n-1}, u^n, acc, coef and three
// face arrays, write u^{n+1}, u^{n+2}, acc = 40 B for two cell-updates
// (20 B each, against 24 B for a single step).  u^{n+1} and u^{n+2} go to two
// fresh buffers (other CTAs still read u^{n-1} / u^n rings), so the window
// rotates through four level buffers.  Single-domain contexts only (a slab
// would need ghost planes two deep).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "step_kernel.cuh"
#include "tma_common.cuh"
#include "step_kernel_v2.cuh"

namespace wb {

#ifndef WB_T2_STAGES
#define WB_T2_STAGES 3
#endif
#ifndef WB_T2_PREFETCH
#define WB_T2_PREFETCH 2
#endif
#ifndef WB_T2_STREAM_STORES
#define WB_T2_STREAM_STORES 0
#endif
#ifndef WB_T2_NEXT_PREFETCH
// L2 prefetch of the next block's first planes (round 1, +1% then); with
// dataflow-chained passes it costs 1-2% (256^3 / 512^3 / 1024^3 / C5 slab,
// profiles/dev/cycle53.sh): off
#define WB_T2_NEXT_PREFETCH 0
#endif
#ifndef WB_T2_TIMELINE
#define WB_T2_TIMELINE 0   // dev: per-CTA start / first data / end times (launch_pair dump)
#endif
#ifndef WB_T2_PACKED
#define WB_T2_PACKED 1
#endif
#ifndef WB_T2_POLL_NS
#define WB_T2_POLL_NS 128   // back-off between polls of a neighbour's completion flag
#endif
#ifndef WB_T2_PDL
#define WB_T2_PDL 1   // programmatic dependent launch: overlap the next pass's start with this tail
#endif
#ifndef WB_T2_CTAS
#define WB_T2_CTAS 3
#endif
constexpr int T2_THREADS = 128;
constexpr int T2_CTAS_F32 = WB_T2_CTAS;   // resident fp32 CTAs per SM
#ifndef WB_T2_CTAS_F64
#define WB_T2_CTAS_F64 2
#endif
#ifndef WB_T2_STAGES_F64
#define WB_T2_STAGES_F64 2   // fp64: two ring stages -> two CTAs per SM (98 KB each)
#endif
constexpr int T2_CTAS_F64 = WB_T2_CTAS_F64;
constexpr int T2_MAXZ = 64;          // z layers (chunks along axis 0) per launch

// Feature level of a two-step launch (template parameter MODE): the launch-
// latency-bound grids (2D, one plane per pass) lose 7% to code they never run
// (C1 24.9 vs 26.6 Gcell-upd/s), so each level compiles only what it needs:
//   T2_BASE   32-bit cell offsets, whole-grid dependency (griddepcontrol.wait)
//   T2_CHAIN  + dataflow-chained passes (completion flags, Step2Args::chain)
//   T2_FULL   + 64-bit offsets (grids of >= 2^31 cells) and peer ghost
//             stores (peer-store slabs)
enum T2Mode : int { T2_BASE = 0, T2_CHAIN = 1, T2_FULL = 2 };

// Packed fp32 pairs (sm_100a FADD2 / FFMA2): the two cells of a thread's row
// run the same IEEE operation sequence, so one f32x2 instruction computes
// both with the bits of two scalar ones.  Products are fma(a, b, z) with z =
// (-0, -0) from a kernel argument: exact a*b (one rounding, signed zeros and
// subnormals as mul.rn) that ptxas cannot contract with the following add
// (it does contract a mul.rn.f32x2 + add.rn.f32x2 pair, unlike scalar mul.rn).
using f2x = unsigned long long;
__device__ __forceinline__ f2x pk2(float lo, float hi) {
    f2x r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ f2x pk2(float2 v) { return pk2(v.x, v.y); }
__device__ __forceinline__ float2 upk2(f2x r) {
    float2 o;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
    return o;
}
__device__ __forceinline__ f2x add2(f2x a, f2x b) {
    f2x r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2x sub2(f2x a, f2x b) {
    f2x r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b, f2x negz) {
    f2x r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(negz));
    return r;
}
constexpr int T2_NS = WB_T2_STAGES;  // TMA ring stages (fp32)
template <typename T> __host__ __device__ constexpr int t2_ns() {
    return sizeof(T) == 8 ? WB_T2_STAGES_F64 : T2_NS;
}
constexpr int T2_PF = WB_T2_PREFETCH;   // L2 prefetch distance beyond the ring (planes)
constexpr int T2_PRODUCER = 32;      // thread issuing TMA (warp 0 carries the extra ring cells)

// Tile geometry of a two-step CTA: TBX x TBY cells (axis 2 x axis 1), 128
// threads of 2 x 2 cells.  Wide = 64 x 8 (ring of 148 cells: two ring slots
// for warp 0); Tall = 32 x 16 (ring of 100 cells: one slot, balanced warps,
// less halo per cell).
template <int TBX_, int TBY_> struct Geo2 {
    static constexpr int TBX = TBX_, TBY = TBY_;
    static constexpr int TX = TBX / 2, TY = TBY / 2;       // threads
    static constexpr int R2 = TBY + 4;                      // rows j0-2 .. j0+TBY+1
    static constexpr int R1 = TBY + 2;                      // rows j0-1 .. j0+TBY
    static constexpr int NRING = 2 * (TBX + 2) + 2 * TBY;   // one-cell ring
    template <typename T> __host__ __device__ static constexpr int W() {
        return TBX + 2 * th_ho<T>();
    }
    static_assert(TX * TY == 128, "two-step CTAs have 128 threads");
};
using GeoWide = Geo2<64, 8>;
using GeoTall = Geo2<32, 16>;

template <typename T> struct Step2Args {
    const T* gamma;    // sparse use only (nodal force coefficient)
    const T* u_prev;   // u^{n-1}
    const T* u_cur;    // u^n
    const T* fi;       // +i face weights (plane below the chunk)
    T* out1;           // u^{n+1}
    T* out2;           // u^{n+2}
    T* acc;
    int n0, n1, n2, chunk;
    int zb[T2_MAXZ + 1];   // plane boundaries of the z layers (blockIdx.z); chunk = longest
    int resident;      // CTAs resident at once (3 per SM; 0: no next-block prefetch)
    MatScalars<T> mat;
    T cv, cg, inv2dt, inv2dx, sdt;
    int n_src;
    int src_i[MAX_SRC], src_j[MAX_SRC], src_k[MAX_SRC];
    T src_val1[MAX_SRC], src_val2[MAX_SRC];   // amplitudes of the two steps
    int sup_lo, sup_hi;
    const unsigned int* sup_mask;
    const int* sup_prefix;
    const T* sup_fc;   // fc(gamma) per support node, compact order (SUP_INJECT)
    T* row1;           // store row of step 1 (gather: u^n; inject: adj of step 1)
    T* row2;           // store row of step 2 (gather: u^{n+1}; inject: adj of step 2)
    int check1, check2;
    typename FTraits<T>::Bits* max1;
    typename FTraits<T>::Bits* max2;
    unsigned long long negz;   // (-0.0f, -0.0f) bits, opaque to ptxas (packed fp32 products)
    // slab contexts: neighbours below / above (two ghost planes each side in
    // the level buffers and the material; TMA plane coordinate = p + zo) and
    // the peer ghost stores of the results (see StepArgs::plo / phi)
    int lo_open, hi_open, zo;
    // dataflow chaining of consecutive passes (WB_T2_CHAIN): every CTA
    // publishes seq in tflags[block] when done; with chain = 1 a CTA waits
    // only for its 3 x 3 x 3 neighbour blocks of the previous pass (seq - 1:
    // everything it reads, and every block still reading what it overwrites)
    // instead of the whole previous grid (griddepcontrol.wait)
    unsigned int* tflags;
    unsigned int seq;
    int chain;
    int zrev;          // z layers in reverse dispatch order (logical layer = nz-1-blockIdx.z)
    T* plo1;
    T* phi1;
    T* plo2;
    T* phi2;
    unsigned long long* timeline;   // WB_T2_TIMELINE builds only: 4 words per CTA
};

__device__ __forceinline__ unsigned long long wb_globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct Tma2Maps {
    CUtensorMap u_r2[4];   // level buffers, (W, R2) boxes at (k0-HO, j0-2)
    CUtensorMap u_r1[4];   // level buffers, (W, R1) boxes at (k0-HO, j0-1)
    CUtensorMap fj_r2;     // +j faces, (W, R2)
    CUtensorMap c_r1;      // coef, (W, R1)
    CUtensorMap fk_r1;     // +k faces, (W, R1)
    CUtensorMap fi_r1;     // +i faces, (W, R1)
    CUtensorMap a_ctr;     // accumulator, (TBX, TBY)
    int prev, cur;         // buffer indices of u^{n-1}, u^n
};

template <typename T, typename G> struct Tma2Stage {
    alignas(128) T U[G::R2][G::template W<T>()];
    alignas(128) T FJ[G::R2][G::template W<T>()];
    alignas(128) T P[G::R1][G::template W<T>()];
    alignas(128) T C[G::R1][G::template W<T>()];
    alignas(128) T FK[G::R1][G::template W<T>()];
    alignas(128) T FI[G::R1][G::template W<T>()];
    alignas(128) T A[G::TBY][G::TBX];
};

constexpr int T2_NX = 3;             // u^{n+1} plane buffers (X)

template <typename T, typename G>
constexpr size_t step2_smem_bytes() {
    return t2_ns<T>() * sizeof(Tma2Stage<T, G>) +
           T2_NX * sizeof(T) * G::R2 * G::template W<T>() /* X planes */ +
           t2_ns<T>() * sizeof(unsigned long long) + 128;
}

// coef and the +k / +j / +i face weights of every cell (0 across the grid
// edge), with the operations of Mat (solver.py:93-119) — the intrinsic
// divisions, which the fast path is verified against.
template <typename T, int FLAVOR>
__global__ void material4_kernel(const T* __restrict__ gamma, MatScalars<T> M, int n0, int n1,
                                 int n2, T* __restrict__ coef, T* __restrict__ fk,
                                 T* __restrict__ fj, T* __restrict__ fi) {
    using P = Mat<T, FLAVOR, false>;
    const long long pl = (long long)n1 * n2, N = pl * n0;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
         c += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(c % n2), j = (int)((c / n2) % n1), i = (int)(c / pl);
        const T g = gamma[c];
        const T m = P::m(M, g);
        T kap;
        coef[c] = P::coef(M, g, kap);
        fk[c] = k + 1 < n2 ? P::face(m, P::m(M, gamma[c + 1])) : T(0);
        fj[c] = j + 1 < n1 ? P::face(m, P::m(M, gamma[c + n2])) : T(0);
        fi[c] = i + 1 < n0 ? P::face(m, P::m(M, gamma[c + pl])) : T(0);
    }
}

template <typename T, typename G, int FLAVOR, bool ACC, int SUP, int MODE>
__global__ void __launch_bounds__(T2_THREADS, sizeof(T) == 4 ? T2_CTAS_F32 : T2_CTAS_F64)
step2_kernel_tma(const __grid_constant__ Step2Args<T> a, const __grid_constant__ Tma2Maps maps) {
    using Tr = FTraits<T>;
    using MP = Mat<T, FLAVOR, false>;   // sparse force coefficients only
    using V = typename Pair<T>::V;
    using Bits = typename Tr::Bits;
    using Off = typename std::conditional<MODE == T2_FULL, long long, int>::type;   // cell offsets
    using UOff = typename std::make_unsigned<Off>::type;
    constexpr bool CHAIN = MODE != T2_BASE, PEER = MODE == T2_FULL;
    constexpr int W = G::template W<T>(), HO = th_ho<T>();
    constexpr int TBX = G::TBX, TBY = G::TBY, R2_H = G::R2, R1_H = G::R1, NRING = G::NRING;
    constexpr int PL = R2_H * W;                       // elements of one R2 plane
    extern __shared__ __align__(128) unsigned char smem_dyn[];
    unsigned char* smem_raw =
        smem_dyn + ((128u - (static_cast<unsigned>(__cvta_generic_to_shared(smem_dyn)) & 127u)) & 127u);
    Tma2Stage<T, G>* st = reinterpret_cast<Tma2Stage<T, G>*>(smem_raw);
    constexpr int T2_NS = t2_ns<T>();   // ring stages of this dtype (shadows the fp32 default)
    T* Xb = reinterpret_cast<T*>(smem_raw + T2_NS * sizeof(Tma2Stage<T, G>));   // X[T2_NX][PL]
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(Xb + T2_NX * PL);
    __shared__ Bits smax[2][T2_THREADS / 32];

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * G::TX + tx;
#if WB_T2_TIMELINE
    const unsigned long long tl_start = wb_globaltimer();
#endif
    // blocks: tiles fastest, then chunks (a chunk-fastest order measured 4%
    // slower: neighbouring tiles at the same planes share halos through L2)
    const int k0 = blockIdx.x * TBX, j0 = blockIdx.y * TBY;
    const int kA = k0 + 2 * tx, ja = j0 + 2 * ty;
    const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
    const Off plane = (Off)n1 * n2;   // 64-bit in T2_FULL: grids of >= 2^31 cells
    // logical z layer: consecutive passes may dispatch the layers in opposite
    // orders (zrev), so a pass starts where the previous one ended (its
    // outputs still in L2)
    const int lz = a.zrev ? (int)gridDim.z - 1 - (int)blockIdx.z : (int)blockIdx.z;
    const int i0 = a.zb[lz];
    const int i1 = a.zb[lz + 1];
    // step-n planes of this chunk: one recomputed plane beyond each end
    // (a ghost plane at a slab boundary; none at the global ends)
    const int pbeg = (i0 > 0 || a.lo_open) ? i0 - 1 : 0;
    const int pfin = (i1 < n0 || a.hi_open) ? i1 : n0 - 1;
    // planes streamed through the ring: pbeg .. pfin, plus pfin+1 (u^n of the
    // chunk end's upper neighbour) so no chunk stalls on a global load
    const int plast = min(pfin + 1, a.hi_open ? n0 + 1 : n0 - 1);
    const int zo = a.zo;

    // ---- per-thread offsets in the R2 frame (rows j0-2.., cols k0-HO..) ----
    // tile rows a, b; clamped (mirrored) outer neighbours at the grid edge.
    // The R1-frame arrays are addressed through bases shifted by one row.
    const int ra = 2 * ty + 2, cA = HO + 2 * tx;
    const int rU = min(max(ja - 1, 0), n1 - 1) - j0 + 2;
    const int rD = min(max(ja + 2, 0), n1 - 1) - j0 + 2;
    const int dL = kA > 0 ? 1 : 0, dR = kA + 2 < n2 ? 1 : 0;   // k-1 / k+2 inside
    const int oA = ra * W + cA, oB = oA + W;
    const int oU = rU * W + cA, oD = rD * W + cA;
    // ring cells: slot 0 = tid, slot 1 = tid + 128 (only the wide tile: warp
    // 0, lanes < NRING-128);
    // rnb packs which neighbours lie inside the grid (bit 0 k-1, 1 k+1, 2 j-1,
    // 3 j+1) — outside ones mirror to the cell itself
    int oR[2], rnb[2];
    bool rg_ok[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int q = tid + t * T2_THREADS;
        int jj = j0, kk = k0;
        if (q < TBX + 2) { jj = j0 - 1; kk = k0 - 1 + q; }
        else if (q < 2 * (TBX + 2)) { jj = j0 + TBY; kk = k0 - 1 + (q - (TBX + 2)); }
        else if (q < 2 * (TBX + 2) + TBY) { jj = j0 + (q - 2 * (TBX + 2)); kk = k0 - 1; }
        else if (q < NRING) { jj = j0 + (q - 2 * (TBX + 2) - TBY); kk = k0 + TBX; }
        rg_ok[t] = q < NRING && jj >= 0 && jj < n1 && kk >= 0 && kk < n2;
        oR[t] = rg_ok[t] ? (jj - j0 + 2) * W + (kk - k0 + HO) : oA;
        rnb[t] = (kk > 0 ? 1 : 0) | (kk < n2 - 1 ? 2 : 0) | (jj > 0 ? 4 : 0) | (jj < n1 - 1 ? 8 : 0);
    }
    const bool ring1 = NRING > T2_THREADS && tid < NRING - T2_THREADS;   // warp 0 only

    unsigned my_src = 0;   // sources in tile + ring and the step-n plane range
    for (int s = 0; s < a.n_src; ++s)
        if (a.src_i[s] >= pbeg && a.src_i[s] <= pfin && a.src_j[s] >= j0 - 1 &&
            a.src_j[s] <= j0 + TBY && a.src_k[s] >= k0 - 1 && a.src_k[s] <= k0 + TBX)
            my_src |= 1u << s;

    constexpr unsigned STAGE_BYTES =
        (unsigned)(sizeof(T) * ((2 * R2_H + 4 * R1_H) * W + (ACC ? TBY * TBX : 0)));
    const CUtensorMap* mU = pick_map(maps.u_r2, maps.cur);
    const CUtensorMap* mP = pick_map(maps.u_r1, maps.prev);
    // L2 prefetch of a later plane's boxes (no shared memory; hides DRAM
    // latency beyond the T2_NS-stage ring)
    auto prefetch_at = [&](int kk0, int jj0, int p) {
        auto pf = [&](const CUtensorMap* m, int c0, int c1, int c2) {
            asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
                         ::"l"(reinterpret_cast<unsigned long long>(m)), "r"(c0), "r"(c1), "r"(c2)
                         : "memory");
        };
        pf(mU, kk0 - HO, jj0 - 2, p + zo);
        pf(&maps.fj_r2, kk0 - HO, jj0 - 2, p + zo);
        pf(mP, kk0 - HO, jj0 - 1, p + zo);
        pf(&maps.c_r1, kk0 - HO, jj0 - 1, p + zo);
        pf(&maps.fk_r1, kk0 - HO, jj0 - 1, p + zo);
        pf(&maps.fi_r1, kk0 - HO, jj0 - 1, p + zo);
        if (ACC) pf(&maps.a_ctr, kk0, jj0, p);
    };
    auto prefetch = [&](int p) { prefetch_at(k0, j0, p); };
    // the block that will most likely take this block's slot when it ends
    // (blocks start in index order, a.resident at a time): its first planes
    // are pulled into L2 during this block's last planes (WB_T2_NEXT_PREFETCH)
    const int nblk = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z) + a.resident;
    const bool has_next = WB_T2_NEXT_PREFETCH && a.resident > 0 &&
                          nblk < (int)(gridDim.x * gridDim.y * gridDim.z);
    int nk0 = 0, nj0 = 0, npb = 0;
    if (has_next) {
        nk0 = (nblk % gridDim.x) * TBX;
        nj0 = ((nblk / gridDim.x) % gridDim.y) * TBY;
        const int nbz = nblk / (gridDim.x * gridDim.y);
        const int nz0 = a.zb[a.zrev ? (int)gridDim.z - 1 - nbz : nbz];
        npb = (nz0 > 0 || a.lo_open) ? nz0 - 1 : 0;
    }
    auto issue = [&](int p, int s) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[s], STAGE_BYTES);
        tma_load_3d(&st[s].U[0][0], mU, k0 - HO, j0 - 2, p + zo, &bar[s]);
        tma_load_3d(&st[s].FJ[0][0], &maps.fj_r2, k0 - HO, j0 - 2, p + zo, &bar[s]);
        tma_load_3d(&st[s].P[0][0], mP, k0 - HO, j0 - 1, p + zo, &bar[s]);
        tma_load_3d(&st[s].C[0][0], &maps.c_r1, k0 - HO, j0 - 1, p + zo, &bar[s]);
        tma_load_3d(&st[s].FK[0][0], &maps.fk_r1, k0 - HO, j0 - 1, p + zo, &bar[s]);
        tma_load_3d(&st[s].FI[0][0], &maps.fi_r1, k0 - HO, j0 - 1, p + zo, &bar[s]);
        // acc holds the own planes only (a ghost plane's box reads as zeros
        // and is never used)
        if (ACC) tma_load_3d(&st[s].A[0][0], &maps.a_ctr, k0, j0, p, &bar[s]);
    };
    if (tid == 0) {
        for (int s = 0; s < T2_NS; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
#if WB_T2_PDL
    // launched with programmatic stream serialisation: this CTA may start
    // while the previous pass drains; nothing above touched global memory.
    // Wait for the previous grid (and its memory) before the first load, and
    // let the next pass start its prologue once every CTA of this one runs.
    if (CHAIN && a.chain) {
        // the next pass may dispatch as soon as all our CTAs run; ours only
        // depend on the previous pass's blocks around this one
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        if (tid < 27) {
            const int bx = (int)blockIdx.x + tid % 3 - 1, by = (int)blockIdx.y + (tid / 3) % 3 - 1;
            const int bz = lz + tid / 9 - 1;
            if (bx >= 0 && bx < (int)gridDim.x && by >= 0 && by < (int)gridDim.y && bz >= 0 &&
                bz < (int)gridDim.z) {
                const unsigned int* f = a.tflags + ((size_t)bz * gridDim.y + by) * gridDim.x + bx;
                unsigned int v;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                    if (v + 1u >= a.seq) break;
                    __nanosleep(WB_T2_POLL_NS);
                }
            }
        }
        __syncthreads();
        // generic-proxy writes of the previous pass -> our TMA (async proxy) reads
        asm volatile("fence.proxy.async.global;" ::: "memory");
    } else {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
#endif
    if (tid == T2_PRODUCER) {
        for (int s = 0; s < T2_NS && pbeg + s <= plast; ++s) issue(pbeg + s, s);
        for (int d = 0; d < T2_PF && pbeg + T2_NS + d <= plast; ++d) prefetch(pbeg + T2_NS + d);
    }

    auto ldv = [](const T* p) { return *reinterpret_cast<const V*>(p); };
    auto stv = [](T* p, V v) { *reinterpret_cast<V*>(p) = v; };
    // global results (u^{n+1}, u^{n+2}, acc) are next read a whole pass later:
    // optionally stream them past L2 (evict-first) so the halo rows shared by
    // neighbouring tiles stay resident (WB_T2_STREAM_STORES)
    auto stg = [](T* p, V v) {
#if WB_T2_STREAM_STORES
        __stcs(reinterpret_cast<V*>(p), v);
#else
        *reinterpret_cast<V*>(p) = v;
#endif
    };
    auto ring_nb = [&](int t, int& l, int& r, int& u, int& d) {
        const int o = oR[t], f = rnb[t];
        l = o - (f & 1); r = o + ((f >> 1) & 1); u = o - W * ((f >> 2) & 1); d = o + W * ((f >> 3) & 1);
    };

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
        const T va = (out - up) * a.inv2dt;    // sign-invariant: (cv*va)*va
        const T g0 = (up1 - um1) * a.inv2dx;
        const T g1 = (ujp - ujm) * a.inv2dx;
        const T g2 = (ukp - ukm) * a.inv2dx;
        return accv + a.sdt * ((a.cv * va) * va + a.cg * (((g0 * g0) + (g1 * g1)) + (g2 * g2)));
    };
    // the same two sequences on packed fp32 pairs (cells k, k+1 of a row)
    constexpr bool PK = WB_T2_PACKED && std::is_same<T, float>::value;
    const f2x NZ = a.negz;
    auto cell2 = [&](f2x u0, f2x up1, f2x um1, f2x ujp, f2x ujm, f2x ukp, f2x ukm, f2x w0hi,
                     f2x w0lo, f2x fjhi, f2x fjlo, f2x fkhi, f2x fklo, f2x coef, f2x up) {
        f2x s = sub2(u0, u0);
        s = add2(s, mul2(sub2(up1, u0), w0hi, NZ));
        s = sub2(s, mul2(sub2(u0, um1), w0lo, NZ));
        s = add2(s, mul2(sub2(ujp, u0), fjhi, NZ));
        s = sub2(s, mul2(sub2(u0, ujm), fjlo, NZ));
        s = add2(s, mul2(sub2(ukp, u0), fkhi, NZ));
        s = sub2(s, mul2(sub2(u0, ukm), fklo, NZ));
        return add2(sub2(add2(u0, u0), up), mul2(coef, s, NZ));
    };
    auto kinc2 = [&](f2x accv, f2x out, f2x up, f2x up1, f2x um1, f2x ujp, f2x ujm, f2x ukp,
                     f2x ukm) {
        const f2x i2dt = pk2((float)a.inv2dt, (float)a.inv2dt);
        const f2x i2dx = pk2((float)a.inv2dx, (float)a.inv2dx);
        const f2x va = mul2(sub2(out, up), i2dt, NZ);
        const f2x g0 = mul2(sub2(up1, um1), i2dx, NZ);
        const f2x g1 = mul2(sub2(ujp, ujm), i2dx, NZ);
        const f2x g2 = mul2(sub2(ukp, ukm), i2dx, NZ);
        const f2x cv = pk2((float)a.cv, (float)a.cv), cg = pk2((float)a.cg, (float)a.cg);
        const f2x sdt = pk2((float)a.sdt, (float)a.sdt);
        const f2x gg = add2(add2(mul2(g0, g0, NZ), mul2(g1, g1, NZ)), mul2(g2, g2, NZ));
        return add2(accv, mul2(sdt, add2(mul2(mul2(cv, va, NZ), va, NZ), mul2(cg, gg, NZ)), NZ));
    };
    // nodal force coefficient of a cell from its gamma (sparse; solver.py:98,110)
    auto fcoef = [&](Off flat) {
        const T g = __ldg(a.gamma + flat);
        T kap;
        (void)MP::coef(a.mat, g, kap);
        return MP::fc(a.mat, g, kap);
    };
    // nodal sources at (plane, j, k) for the step's amplitudes
    auto inject_src = [&](int p, int jj, int kk, const T* val, T& o) {
        for (int q = 0; q < a.n_src; ++q)
            if (((my_src >> q) & 1u) && p == a.src_i[q] && jj == a.src_j[q] && kk == a.src_k[q])
                o = o + fcoef(p * plane + jj * n2 + kk) * val[q];
    };
    // support bit / compact index of cell (p, jj, kk)
    auto sup_index = [&](int p, int jj, int kk) -> int {
        if (SUP == SUP_NONE || p < a.sup_lo || p > a.sup_hi) return -1;
        const UOff flat = (UOff)(p * plane + jj * n2 + kk);
        const unsigned w = __ldg(a.sup_mask + (flat >> 5));
        const unsigned bit = (unsigned)(flat & 31u);
        if (!((w >> bit) & 1u)) return -1;
        return __ldg(a.sup_prefix + (flat >> 5)) + __popc(w & ((1u << bit) - 1u));
    };
    // injections of one step into a tile 2x2 block at plane p: sources, then
    // the support (solver.py:167-170); gather records the pre-step level
    auto tile_inject = [&](int p, V& oa, V& ob, V ua, V ub, const T* val, T* row, bool gather_ok) {
        if (my_src) {
            inject_src(p, ja, kA, val, oa.x);
            inject_src(p, ja, kA + 1, val, oa.y);
            inject_src(p, ja + 1, kA, val, ob.x);
            inject_src(p, ja + 1, kA + 1, val, ob.y);
        }
        if (SUP != SUP_NONE && p >= a.sup_lo && p <= a.sup_hi) {
            const T uo[4] = {ua.x, ua.y, ub.x, ub.y};
            T* oo[4] = {&oa.x, &oa.y, &ob.x, &ob.y};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int jj = ja + (c >> 1), kk = kA + (c & 1);
                const int qi = sup_index(p, jj, kk);
                if (qi >= 0) {
                    if (SUP == SUP_GATHER) { if (gather_ok) row[qi] = uo[c]; }
                    else *oo[c] = *oo[c] + ldg(a.sup_fc + qi) * ldg(row + qi);
                }
            }
        }
    };

    // ---------------- prologue: plane pbeg ----------------
    const int cofs = ja * n2 + kA;
    const bool has_m0 = pbeg - 1 >= (a.lo_open ? -2 : 0);   // plane pbeg-1 (ghost or real)
    auto ring_gofs = [&](int t) {   // global offset (in plane) of ring slot t
        const int r = oR[t] / W, c = oR[t] - r * W;
        return (r + j0 - 2) * n2 + (c + k0 - HO);
    };
    V unm_a, unm_b, w0_a = {T(0), T(0)}, w0_b = {T(0), T(0)};   // plane pbeg-1 (mirror at 0)
    T rum[2] = {T(0), T(0)}, rw0[2] = {T(0), T(0)};
    if (has_m0) {
        const Off gm = (pbeg - 1) * plane;
        unm_a = __ldg(reinterpret_cast<const V*>(a.u_cur + gm + cofs));
        unm_b = __ldg(reinterpret_cast<const V*>(a.u_cur + gm + cofs + n2));
        w0_a = __ldg(reinterpret_cast<const V*>(a.fi + gm + cofs));
        w0_b = __ldg(reinterpret_cast<const V*>(a.fi + gm + cofs + n2));
#pragma unroll
        for (int t = 0; t < 2; ++t)
            if (rg_ok[t]) {
                rum[t] = __ldg(a.u_cur + gm + ring_gofs(t));
                rw0[t] = __ldg(a.fi + gm + ring_gofs(t));
            }
    }
    mbar_wait(&bar[0], 0u);
#if WB_T2_TIMELINE
    const unsigned long long tl_data = wb_globaltimer();
#endif
    V un0_a = ldv(&st[0].U[0][0] + oA), un0_b = ldv(&st[0].U[0][0] + oB);
    T run0[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) run0[t] = (&st[0].U[0][0])[oR[t]];
    if (!has_m0) {
        unm_a = un0_a; unm_b = un0_b;
        rum[0] = run0[0]; rum[1] = run0[1];
    }

    // step n+1 state: material of the previous step-n plane, u^{n+1} queue
    T f1_kLa = T(0), f1_kIa = T(0), f1_kRa = T(0), f1_kLb = T(0), f1_kIb = T(0), f1_kRb = T(0);
    V f1_jlo = {T(0), T(0)}, f1_jab = f1_jlo, f1_jhi = f1_jlo;
    V w1lo_a = f1_jlo, w1lo_b = f1_jlo, w1hi_a = f1_jlo, w1hi_b = f1_jlo;
    V c1_a = f1_jlo, c1_b = f1_jlo;
    V x_m1a = un0_a, x_m1b = un0_b, x_0a = un0_a, x_0b = un0_b;   // u^{n+1}(p-2), (p-1)
    V un1_a = unm_a, un1_b = unm_b;                                // u^n(p-1)
    V acc1_a = {T(0), T(0)}, acc1_b = acc1_a;                      // acc after step n at p-1
    Bits lmax1 = 0, lmax2 = 0;

    // step n+1 at plane q1 for the tile: xp = u^{n+1}(q1+1) (registers)
    auto step2_tile = [&](int q1, const T* Xq, V xp_a, V xp_b) {
        const V xu = ldv(Xq + oU), xd = ldv(Xq + oD);
        const T xLa = Xq[oA - dL], xRa = Xq[oA + 1 + dR], xLb = Xq[oB - dL], xRb = Xq[oB + 1 + dR];
        V o2a, o2b;
        if constexpr (PK) {
            const f2x kpa = pk2(x_0a.y, xRa), kma = pk2(xLa, x_0a.x);
            const f2x kpb = pk2(x_0b.y, xRb), kmb = pk2(xLb, x_0b.x);
            const f2x ra = cell2(pk2(x_0a), pk2(xp_a), pk2(x_m1a), pk2(x_0b), pk2(xu), kpa, kma,
                                 pk2(w1hi_a), pk2(w1lo_a), pk2(f1_jab), pk2(f1_jlo),
                                 pk2(f1_kIa, f1_kRa), pk2(f1_kLa, f1_kIa), pk2(c1_a), pk2(un1_a));
            const f2x rb = cell2(pk2(x_0b), pk2(xp_b), pk2(x_m1b), pk2(xd), pk2(x_0a), kpb, kmb,
                                 pk2(w1hi_b), pk2(w1lo_b), pk2(f1_jhi), pk2(f1_jab),
                                 pk2(f1_kIb, f1_kRb), pk2(f1_kLb, f1_kIb), pk2(c1_b), pk2(un1_b));
            o2a = upk2(ra);
            o2b = upk2(rb);
            tile_inject(q1, o2a, o2b, x_0a, x_0b, a.src_val2, a.row2, true);
            const Off oc = q1 * plane + cofs;
            if (ACC) {
                const f2x fa = kinc2(pk2(acc1_a), pk2(o2a), pk2(un1_a), pk2(xp_a), pk2(x_m1a),
                                     pk2(x_0b), pk2(xu), kpa, kma);
                const f2x fb = kinc2(pk2(acc1_b), pk2(o2b), pk2(un1_b), pk2(xp_b), pk2(x_m1b),
                                     pk2(xd), pk2(x_0a), kpb, kmb);
                stg(a.acc + oc, upk2(fa));
                stg(a.acc + oc + n2, upk2(fb));
            }
            stg(a.out1 + oc, x_0a);
            stg(a.out1 + oc + n2, x_0b);
            stg(a.out2 + oc, o2a);
            stg(a.out2 + oc + n2, o2b);
        } else {
        o2a.x = cell(x_0a.x, xp_a.x, x_m1a.x, x_0b.x, xu.x, x_0a.y, xLa, w1hi_a.x, w1lo_a.x,
                     f1_jab.x, f1_jlo.x, f1_kIa, f1_kLa, c1_a.x, un1_a.x);
        o2a.y = cell(x_0a.y, xp_a.y, x_m1a.y, x_0b.y, xu.y, xRa, x_0a.x, w1hi_a.y, w1lo_a.y,
                     f1_jab.y, f1_jlo.y, f1_kRa, f1_kIa, c1_a.y, un1_a.y);
        o2b.x = cell(x_0b.x, xp_b.x, x_m1b.x, xd.x, x_0a.x, x_0b.y, xLb, w1hi_b.x, w1lo_b.x,
                     f1_jhi.x, f1_jab.x, f1_kIb, f1_kLb, c1_b.x, un1_b.x);
        o2b.y = cell(x_0b.y, xp_b.y, x_m1b.y, xd.y, x_0a.y, xRb, x_0b.x, w1hi_b.y, w1lo_b.y,
                     f1_jhi.y, f1_jab.y, f1_kRb, f1_kIb, c1_b.y, un1_b.y);
        tile_inject(q1, o2a, o2b, x_0a, x_0b, a.src_val2, a.row2, true);
        const Off oc = q1 * plane + cofs;
        if (ACC) {
            V fa, fb;
            fa.x = kinc(acc1_a.x, o2a.x, un1_a.x, xp_a.x, x_m1a.x, x_0b.x, xu.x, x_0a.y, xLa);
            fa.y = kinc(acc1_a.y, o2a.y, un1_a.y, xp_a.y, x_m1a.y, x_0b.y, xu.y, xRa, x_0a.x);
            fb.x = kinc(acc1_b.x, o2b.x, un1_b.x, xp_b.x, x_m1b.x, xd.x, x_0a.x, x_0b.y, xLb);
            fb.y = kinc(acc1_b.y, o2b.y, un1_b.y, xp_b.y, x_m1b.y, xd.y, x_0a.y, xRb, x_0b.x);
            stg(a.acc + oc, fa);
            stg(a.acc + oc + n2, fb);
        }
        stg(a.out1 + oc, x_0a);
        stg(a.out1 + oc + n2, x_0b);
        stg(a.out2 + oc, o2a);
        stg(a.out2 + oc + n2, o2b);
        }
        // slab boundary planes: both new levels also go straight into the
        // neighbour's ghost planes (NVLink stores across GPUs)
        if (PEER && q1 < 2 && a.plo1) {
            const Off oc = q1 * plane + cofs;
            stg(a.plo1 + oc, x_0a); stg(a.plo1 + oc + n2, x_0b);
            stg(a.plo2 + oc, o2a); stg(a.plo2 + oc + n2, o2b);
        }
        if (PEER && q1 >= n0 - 2 && a.phi1) {
            const Off oc = q1 * plane + cofs;
            stg(a.phi1 + oc, x_0a); stg(a.phi1 + oc + n2, x_0b);
            stg(a.phi2 + oc, o2a); stg(a.phi2 + oc + n2, o2b);
        }
        if (a.check2) {
            Bits m1 = Tr::abs_bits(o2a.x), m2 = Tr::abs_bits(o2a.y);
            Bits m3 = Tr::abs_bits(o2b.x), m4 = Tr::abs_bits(o2b.y);
            m1 = m1 > m2 ? m1 : m2; m3 = m3 > m4 ? m3 : m4; m1 = m1 > m3 ? m1 : m3;
            lmax2 = m1 > lmax2 ? m1 : lmax2;
        }
    };

    // one plane; q = stage of plane p, gpar = its mbarrier parity, xq = its X
    // buffer (rolled loop: unrolled copies of this body overflow the
    // instruction cache).  One barrier per plane, after step n: it publishes
    // X(p) and frees stage(p), which is refilled at once (T2_NS planes ahead);
    // three X buffers keep X(p) from overwriting X(p-3) before (c) read it.
    auto body = [&](int q, int xq, int p, unsigned gpar) {
        const int sn = q + 1 == T2_NS ? 0 : q + 1;
        const unsigned pn = (q + 1 == T2_NS) ? 1u : 0u;   // parity flip for plane p+1
        T* Xc = Xb + xq * PL;
        const T* Xp = Xb + (xq == 0 ? T2_NX - 1 : xq - 1) * PL;
        const Tma2Stage<T, G>& S = st[q];
        const T* SU = &S.U[0][0];
        const T* SFJ = &S.FJ[0][0];
        const T* SP = &S.P[0][0] - W;     // R1 frame = R2 frame shifted one row
        const T* SC = &S.C[0][0] - W;
        const T* SFK = &S.FK[0][0] - W;
        const T* SFI = &S.FI[0][0] - W;
        // ---- a: u^n of plane p+1 ----
        V unp_a = un0_a, unp_b = un0_b;
        T runp[2] = {run0[0], run0[1]};
        if (p + 1 <= plast) {            // else: plane n0 mirrors plane n0-1
            mbar_wait(&bar[sn], gpar ^ pn);
            const T* NU = &st[sn].U[0][0];
            unp_a = ldv(NU + oA); unp_b = ldv(NU + oB);
#pragma unroll
            for (int t = 0; t < 2; ++t) runp[t] = NU[oR[t]];
        }

        // ---- d: step n at plane p (tile + ring) -> X[b] ----
        const V wh_a = ldv(SFI + oA), wh_b = ldv(SFI + oB);
        const V cf_a = ldv(SC + oA), cf_b = ldv(SC + oB);
        const V fka = ldv(SFK + oA), fkb = ldv(SFK + oB);        // (kI, kR) of rows a, b
        const T kLa = SFK[oA - dL], kLb = SFK[oB - dL];
        const V jlo = ldv(SFJ + oU), jab = ldv(SFJ + oA), jhi = ldv(SFJ + oB);
        const V uu = ldv(SU + oU), ud = ldv(SU + oD);
        const T uLa = SU[oA - dL], uRa = SU[oA + 1 + dR], uLb = SU[oB - dL], uRb = SU[oB + 1 + dR];
        const V pa = ldv(SP + oA), pb = ldv(SP + oB);
        V oa, ob;
        f2x kpa = 0, kma = 0, kpb = 0, kmb = 0;
        if constexpr (PK) {
            kpa = pk2(un0_a.y, uRa); kma = pk2(uLa, un0_a.x);
            kpb = pk2(un0_b.y, uRb); kmb = pk2(uLb, un0_b.x);
            oa = upk2(cell2(pk2(un0_a), pk2(unp_a), pk2(unm_a), pk2(un0_b), pk2(uu), kpa, kma,
                            pk2(wh_a), pk2(w0_a), pk2(jab), pk2(jlo), pk2(fka), pk2(kLa, fka.x),
                            pk2(cf_a), pk2(pa)));
            ob = upk2(cell2(pk2(un0_b), pk2(unp_b), pk2(unm_b), pk2(ud), pk2(un0_a), kpb, kmb,
                            pk2(wh_b), pk2(w0_b), pk2(jhi), pk2(jab), pk2(fkb), pk2(kLb, fkb.x),
                            pk2(cf_b), pk2(pb)));
        } else {
        oa.x = cell(un0_a.x, unp_a.x, unm_a.x, un0_b.x, uu.x, un0_a.y, uLa, wh_a.x, w0_a.x,
                    jab.x, jlo.x, fka.x, kLa, cf_a.x, pa.x);
        oa.y = cell(un0_a.y, unp_a.y, unm_a.y, un0_b.y, uu.y, uRa, un0_a.x, wh_a.y, w0_a.y,
                    jab.y, jlo.y, fka.y, fka.x, cf_a.y, pa.y);
        ob.x = cell(un0_b.x, unp_b.x, unm_b.x, ud.x, un0_a.x, un0_b.y, uLb, wh_b.x, w0_b.x,
                    jhi.x, jab.x, fkb.x, kLb, cf_b.x, pb.x);
        ob.y = cell(un0_b.y, unp_b.y, unm_b.y, ud.y, un0_a.y, uRb, un0_b.x, wh_b.y, w0_b.y,
                    jhi.y, jab.y, fkb.y, fkb.x, cf_b.y, pb.y);
        }
        const bool own_plane = p >= i0 && p < i1;
        tile_inject(p, oa, ob, un0_a, un0_b, a.src_val1, a.row1, own_plane);
        stv(Xc + oA, oa);
        stv(Xc + oB, ob);
        V nacc_a = acc1_a, nacc_b = acc1_b;
        if (own_plane) {
            if (ACC) {
                const V aa = ldv(&S.A[2 * ty][2 * tx]), ab = ldv(&S.A[2 * ty + 1][2 * tx]);
                if constexpr (PK) {
                    nacc_a = upk2(kinc2(pk2(aa), pk2(oa), pk2(pa), pk2(unp_a), pk2(unm_a),
                                        pk2(un0_b), pk2(uu), kpa, kma));
                    nacc_b = upk2(kinc2(pk2(ab), pk2(ob), pk2(pb), pk2(unp_b), pk2(unm_b),
                                        pk2(ud), pk2(un0_a), kpb, kmb));
                } else {
                nacc_a.x = kinc(aa.x, oa.x, pa.x, unp_a.x, unm_a.x, un0_b.x, uu.x, un0_a.y, uLa);
                nacc_a.y = kinc(aa.y, oa.y, pa.y, unp_a.y, unm_a.y, un0_b.y, uu.y, uRa, un0_a.x);
                nacc_b.x = kinc(ab.x, ob.x, pb.x, unp_b.x, unm_b.x, ud.x, un0_a.x, un0_b.y, uLb);
                nacc_b.y = kinc(ab.y, ob.y, pb.y, unp_b.y, unm_b.y, ud.y, un0_a.y, uRb, un0_b.x);
                }
            }
            if (a.check1) {
                Bits m1 = Tr::abs_bits(oa.x), m2 = Tr::abs_bits(oa.y);
                Bits m3 = Tr::abs_bits(ob.x), m4 = Tr::abs_bits(ob.y);
                m1 = m1 > m2 ? m1 : m2; m3 = m3 > m4 ? m3 : m4; m1 = m1 > m3 ? m1 : m3;
                lmax1 = m1 > lmax1 ? m1 : lmax1;
            }
        }
        // ring cells (step n only, no accumulation / gather)
        T rwh[2] = {rw0[0], rw0[1]};
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            if (t == 1 && !ring1) continue;
            if (!rg_ok[t]) continue;
            const int o = oR[t];
            int nl, nr, nu, nd;
            ring_nb(t, nl, nr, nu, nd);
            rwh[t] = SFI[o];
            T v = cell(run0[t], runp[t], rum[t], SU[nd], SU[nu], SU[nr], SU[nl], rwh[t], rw0[t],
                       SFJ[o], SFJ[nu], SFK[o], SFK[nl], SC[o], SP[o]);
            if (my_src || SUP == SUP_INJECT) {
                const int r = o / W;
                const int jj = r + j0 - 2, kk = o - r * W + k0 - HO;
                if (my_src) inject_src(p, jj, kk, a.src_val1, v);
                if (SUP == SUP_INJECT) {
                    const int qi = sup_index(p, jj, kk);
                    if (qi >= 0) v = v + ldg(a.sup_fc + qi) * ldg(a.row1 + qi);
                }
            }
            Xc[o] = v;
        }
        __syncthreads();
        if (tid == T2_PRODUCER && p + T2_NS <= plast) {
            issue(p + T2_NS, q);
            if (p + T2_NS + T2_PF <= plast) prefetch(p + T2_NS + T2_PF);
        } else if (tid == T2_PRODUCER && has_next) {   // one plane of the next block per body
            const int d = p + T2_NS - plast - 1;
            if (d >= 0 && d < T2_NS && npb + d < n0) prefetch_at(nk0, nj0, npb + d);
        }

        // ---- c: step n+1 at plane p-1 (tile) ----
        if (p - 1 >= i0 && p - 1 < i1) step2_tile(p - 1, Xp, oa, ob);

        // ---- rotate: plane p's material serves step n+1 at the next plane ----
        f1_kLa = kLa; f1_kIa = fka.x; f1_kRa = fka.y;
        f1_kLb = kLb; f1_kIb = fkb.x; f1_kRb = fkb.y;
        f1_jlo = jlo; f1_jab = jab; f1_jhi = jhi;
        w1lo_a = w0_a; w1lo_b = w0_b; w1hi_a = wh_a; w1hi_b = wh_b;
        c1_a = cf_a; c1_b = cf_b;
        acc1_a = nacc_a; acc1_b = nacc_b;
        un1_a = un0_a; un1_b = un0_b;
        // u^{n+1} queue; at the global bottom plane the "previous" plane is
        // the mirror (the plane itself)
        const bool gbot = p == 0 && !a.lo_open;
        x_m1a = gbot ? oa : x_0a; x_m1b = gbot ? ob : x_0b;
        x_0a = oa; x_0b = ob;
        // step-n queue
        unm_a = un0_a; unm_b = un0_b; un0_a = unp_a; un0_b = unp_b;
        w0_a = wh_a; w0_b = wh_b;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            rw0[t] = rwh[t];
            rum[t] = run0[t]; run0[t] = runp[t];
        }
    };

    unsigned gpar = 0;
    int xq = 0;
    for (int p = pbeg, q = 0; p <= pfin; ++p) {
        body(q, xq, p, gpar);
        if (++q == T2_NS) { q = 0; gpar ^= 1u; }
        if (++xq == T2_NX) xq = 0;
    }

    // ---- step n+1 at the last plane of the grid (mirror above) ----
    // interior chunks finish inside the loop (pfin = i1); at the global end
    // pfin = n0-1 = i1-1 and plane n0 mirrors the plane itself (X(pfin) was
    // published by the last plane's barrier)
    if (pfin == i1 - 1) step2_tile(pfin, Xb + ((pfin - pbeg) % T2_NX) * PL, x_0a, x_0b);
#if WB_T2_TIMELINE
    if (tid == 0 && a.timeline) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        unsigned long long* t = a.timeline +
            4ull * (blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z));
        t[0] = tl_start; t[1] = tl_data; t[2] = wb_globaltimer(); t[3] = smid;
    }
#endif

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
            Bits v1 = lane < (T2_THREADS / 32) ? smax[0][lane] : 0;
            Bits v2 = lane < (T2_THREADS / 32) ? smax[1][lane] : 0;
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
    if (CHAIN && a.tflags) {   // publish this block's completion (release: all its writes first)
        __syncthreads();
        if (tid == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __threadfence();
            unsigned int* f = a.tflags + ((size_t)lz * gridDim.y + blockIdx.y) * gridDim.x +
                              blockIdx.x;
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(a.seq) : "memory");
        }
    }
}

}  // namespace wb
