// waveb200 C ABI implementation (include/waveb200.h).
//
// Host-side driver of the fused sweeps: owns the device buffers of one grid,
// builds the per-step launch arguments (pointer rotation of the 3-level
// window, source values, support rows, check slots) and evaluates the
// stability checks after each sweep in the reference's order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/waveb200.h"
#include "aux_kernels.cuh"
#include "common.cuh"
#include "design_kernels.cuh"
#include "dropin_kernels.cuh"
#include "launchers.cuh"

#include <cudaTypedefs.h>

using namespace wb;

namespace wb {
thread_local bool t_no_pdl = false;
}

namespace {

constexpr int STABILITY_CHECK_INTERVAL = 50;     // solver.py:29
constexpr double STABILITY_GROWTH_FACTOR = 1e6;  // solver.py:30
thread_local std::string g_create_error;

// cluster-resident sweeps of small 2D grids (cluster_reg.cuh): default of
// WO_OPT_CLUSTER for new contexts, 2 = the default (on: C1 fp32 27.6 -> 42.3,
// fp64 24.1 -> 26.7 Gcell-upd/s against two-step passes); WB_CLUSTER=0/1/2
// overrides (A/B runs)
constexpr int CLUSTER_DEFAULT = 2;
int cluster_default() {
    static const int on = [] {
        const char* e = getenv("WB_CLUSTER");
        return e ? atoi(e) : CLUSTER_DEFAULT;
    }();
    return on;
}
// which cluster engine: the register-resident one (cluster_reg.cuh) unless
// WB_CLUSTER_ENGINE=smem asks for the shared-memory one (cluster_sweep.cuh)
bool cluster_smem_engine() {
    static const bool smem = [] {
        const char* e = getenv("WB_CLUSTER_ENGINE");
        return e && strcmp(e, "smem") == 0;
    }();
    return smem;
}
// packed pairs per thread row of the register-resident engine (WB_CR_PC=1|2)
int cluster_reg_pc() {
    static const int pc = [] {
        const char* e = getenv("WB_CR_PC");
        return e && atoi(e) == 1 ? 1 : 2;
    }();
    return pc;
}

}  // namespace

struct wo_ctx {
    int device = 0;
    int ndim = 0;
    int64_t shape[3] = {1, 1, 1};      // caller's shape (local for slabs)
    int kn0 = 1, kn1 = 1, kn2 = 1;     // kernel-space local extents
    int i_off = 0, n0g = 1;            // slab placement along axis 0
    int has_lo = 0, has_hi = 0;        // neighbour slab below / above
    int gl = 0, gh = 0;                // ghost planes below / above (2 if room, global end: 0)
    int itemsize = 8;
    double dx = 0.0;
    cudaStream_t stream = nullptr;

    char* gamma = nullptr;             // allocation bases (ghost planes first)
    char* u[4] = {nullptr, nullptr, nullptr, nullptr};  // level buffers (2-3 only for two-step passes)
    char* acc = nullptr;
    int cur = 0, prv = 1;              // u[cur] = u^n, u[prv] = u^{n-1}

    bool material_set = false;
    bool fast_div = false;             // verify_material_kernel passed for this material
    int allow_fast_div = 1;            // wo_set_option(WO_OPT_FAST_DIV)
    int use_pair = 1;                  // wo_set_option(WO_OPT_PAIR_KERNEL)
    int use_tma = 1;                   // wo_set_option(WO_OPT_TMA_KERNEL)
    int use_two_step = 1;              // wo_set_option(WO_OPT_TWO_STEP)
    int num_sms = 148;                 // of the context's device
    int part = 0;                      // WO_OPT_PLANE_PART: 0 whole steps, 1 boundary, 2 interior
    // peer ghost stores (wo_slab_peers): every launch also stores its own
    // planes 0, 1 / n0-2, n0-1 of the level(s) it writes into the neighbours'
    // two ghost planes of the same level buffer (slabs step in lockstep), then
    // bumps the neighbours' flags; the next launch waits for both neighbours'
    // flags (p2p_wait / p2p_signal, one epoch per sweep)
    char* peer_lo[4] = {nullptr, nullptr, nullptr, nullptr};   // lower's top ghost planes
    char* peer_hi[4] = {nullptr, nullptr, nullptr, nullptr};   // upper's bottom ghost planes
    unsigned int* peer_lo_flag = nullptr;   // lower's in_flags + 1 (its "from upper" word)
    unsigned int* peer_hi_flag = nullptr;   // upper's in_flags + 0 (its "from lower" word)
    unsigned int* in_flags = nullptr;       // [parity][from lower, from upper]
    unsigned int p2p_seq = 0;               // signals sent in this epoch
    int p2p_epoch = 0;                      // sweeps begun (flag slot = epoch parity)
    bool p2p = false;
    // neighbours' allocations mapped through CUDA IPC (wo_ipc_open): handle
    // bytes -> mapped base, closed by wo_destroy
    std::vector<std::pair<std::string, char*>> ipc_maps;
    // CUDA graphs of whole sweeps (WO_OPT_GRAPHS): a sweep whose launch
    // sequence repeats (same key: range, sources, amplitudes, window indices
    // and the state generation) is captured on its second sighting and
    // replayed from then on.  The key hashes the parameter buffers' addresses
    // and gen, which changes with every setting that enters a kernel's
    // parameters (material scalars, coefficients, support, options, maps).
    struct SweepGraph {
        uint64_t key = 0, seen = 0;
        cudaGraphExec_t exec = nullptr;
        int cur = 0, prv = 0;
        int64_t d_launches = 0, d_steps = 0, d_pairs = 0;
    } graph[2];                        // forward, backward
    int use_graphs = 1;
    uint64_t gen = 1;
    int t2_geo = GEO_NONE;             // two-step tile geometry (set when its maps are built)
    int t2_state = 0;                  // two-step tensor maps: 0 not built, 1 ready, -1 no
    Tma2Maps t2maps;
    char* mat4 = nullptr;              // coef | +k | +j | +i faces (two-step passes)
    unsigned int* tflags = nullptr;    // per-block completion of the last two-step pass
    size_t tflags_bytes = 0;
    unsigned int t2_seq = 0;           // two-step passes of the current sweep (flag values)
    bool t2_chain_next = false;        // the next pass directly follows one of this sweep
    bool t2_oom = false;               // two-step buffers did not fit: single steps only
    int use_cluster = cluster_default();   // wo_set_option(WO_OPT_CLUSTER)
    int cl_state = 0;                  // cluster sweep engine: 0 unknown, 1 ready, -1 no
    int cl_size = 0, cl_rows = 0;      // CTAs per cluster, rows per CTA
    int cr_state = 0, cr_size = 0, cr_rows = 0;   // register-resident engine (cluster_reg.cuh)
    double* amp_dev = nullptr;         // source amplitude table of a cluster sweep
    size_t amp_cap = 0;
    char* stage = nullptr;             // fp64 upload staging (persistent)
    char* hstage = nullptr;            // pinned host staging for field downloads (2 halves)
    char* scratch = nullptr;           // one field (wo_get_field axis reversal)
    double* opt = nullptr;             // wo_opt_*: params | m | v (fp64 fields)
    unsigned char* opt_frozen = nullptr;
    double* opt_partial = nullptr;     // 592 block sums
    AdamScalars adam{};
    int opt_zero_frozen = 0;
    double* dsn = nullptr;             // design loop: g_tilde | g_bar | grad | 3 temporaries (fp64)
    unsigned char* dmask = nullptr;    // design mask (nullptr: everywhere)
    int* dfp_off = nullptr;            // filter footprint [n][3]
    double* dfp_w = nullptr;
    int dfp_n = 0;
    int design_active = 0;             // wo_opt_step takes the chain-rule gradient
    size_t scratch_bytes = 0;
    char* snap = nullptr;              // wo_snapshot: window levels | acc | store
    size_t snap_bytes = 0;
    int64_t snap_store = -1;           // store bytes held by the snapshot (-1: none)
    cudaEvent_t hev[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;
    char* flag = nullptr;              // device int scratch (verification flag)
    size_t flag_bytes = 0;
    bool mat4_valid = false;           // computed for the current material
    int64_t pair_launches = 0;
    int tma_state = 0;                 // 0 not built, 1 maps ready, -1 not eligible
    TmaMaps tmaps;                     // tensor maps of gamma, u[0], u[1], acc
    int sup_lo = 0, sup_hi = -1;       // local planes holding support nodes
    int flavor = 0;
    double rho0 = 0, rho1 = 0, kappa1 = 0, rho2 = 0, kappa2 = 0, dt_mat = 0, ratio2 = 0;
    double cv = 0, cg = 0, inv2dt = 0, inv2dx = 0;

    int64_t n_sup = 0;
    unsigned int* mask = nullptr;
    int* prefix = nullptr;
    // per-support-node force coefficients fc(gamma), compact order
    // (sup_fc_kernel; the two-step kernel's adjoint injection)
    long long* sup_flat = nullptr;     // device copy of the support indices
    size_t sup_flat_bytes = 0;
    char* sup_fc = nullptr;
    size_t sup_fc_bytes = 0;
    bool sup_fc_valid = false;
    char* store = nullptr;
    size_t store_bytes = 0;
    double* measured = nullptr;
    size_t measured_bytes = 0;
    double* partial = nullptr;
    size_t partial_bytes = 0;
    double* cost = nullptr;
    char* maxslots = nullptr;
    size_t maxslot_bytes = 0;
    long long* f_idx = nullptr;
    size_t f_idx_cap = 0;
    char* f_vals = nullptr;
    size_t f_vals_cap = 0;
    double* f_dense = nullptr;
    size_t f_dense_cap = 0;
    char* hist = nullptr;              // full forward history (reference engine)
    size_t hist_bytes = 0;
    char* u3 = nullptr;                // third adjoint level (reference engine)
    size_t u3_bytes = 0;

    bool prof = false;                 // any step-launch profiling
    int prof_every = 0;                // bracket every prof_every-th step launch with events
    int64_t prof_tick = 0;
    bool prof_open = false;            // the current launch is bracketed
    cudaEvent_t marks[8] = {};
    std::vector<cudaEvent_t> ev_free, ev_used;
    std::vector<char> ev_kind;         // per bracketed launch: 1 two-step pass, 0 single step
    int64_t launches = 0, step_launches = 0;
    double step_ms = 0.0;
    double prof_ms[2] = {0.0, 0.0};    // summed bracketed time: [single, pair]
    int64_t prof_n[2] = {0, 0};
    int64_t dev_bytes = 0;
    std::string err;

    int64_t plane() const { return (int64_t)kn1 * kn2; }
    int64_t cells() const { return (int64_t)kn0 * plane(); }
    int alloc_planes() const { return kn0 + gl + gh; }
    int64_t alloc_cells() const { return (int64_t)alloc_planes() * plane(); }
    size_t field_bytes() const { return (size_t)cells() * itemsize; }
    char* base0(char* p) const { return p + (size_t)gl * plane() * itemsize; }
    char* ucur() const { return base0(u[cur]); }
    char* uprev() const { return base0(u[prv]); }
};

#define CK(call)                                                                     \
    do {                                                                             \
        cudaError_t e_ = (call);                                                     \
        if (e_ != cudaSuccess) {                                                     \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);           \
            return WO_ERR_CUDA;                                                      \
        }                                                                            \
    } while (0)

#define REQUIRE(cond, msg)                   \
    do {                                     \
        if (!(cond)) {                       \
            ctx->err = (msg);                \
            return WO_ERR_CONFIG;            \
        }                                    \
    } while (0)

namespace {

int dev_alloc(wo_ctx* ctx, void** p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();   // not sticky: later launch checks must not see it
        *p = nullptr;
        ctx->err = std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e);
        return e == cudaErrorMemoryAllocation ? WO_ERR_BUDGET : WO_ERR_CUDA;
    }
    ctx->dev_bytes += (int64_t)bytes;
    return WO_OK;
}

template <typename P>
int ensure(wo_ctx* ctx, P** p, size_t* cap, size_t bytes) {
    if (*cap >= bytes && *p) return WO_OK;
    if (*p) {
        cudaFree(*p);
        ctx->dev_bytes -= (int64_t)*cap;
    }
    *p = nullptr;
    *cap = 0;
    int rc = dev_alloc(ctx, (void**)p, bytes);
    if (rc == WO_OK) *cap = bytes;
    return rc;
}

template <typename T>
MatScalars<T> mat_scalars(const wo_ctx* ctx) {
    MatScalars<T> M{};
    M.flavor = ctx->flavor;
    const double dt = ctx->dt_mat;
    if (ctx->flavor == RHO_SCALED) {
        const T r2 = (T)ctx->ratio2;          // dtype.type((c0*dt/dx)**2), solver.py:96
        M.two_r2 = T(2) * r2;                 // dtype.type(2.0) * r2, solver.py:97
        M.rho0 = (T)ctx->rho0;
    } else {
        M.irho1 = (T)(1.0 / ctx->rho1);       // grids.py:252 (python floats, then weak cast)
        M.drho = (T)(1.0 / ctx->rho2 - 1.0 / ctx->rho1);
        M.ikap1 = (T)(1.0 / ctx->kappa1);
        M.dkap = (T)(1.0 / ctx->kappa2 - 1.0 / ctx->kappa1);
        M.s2 = (T)ctx->ratio2;                // dtype.type((dt/dx)**2), solver.py:108
    }
    M.dt2 = (T)(dt * dt);
    return M;
}

// WB_T2_CHAIN (default 1): consecutive two-step passes of a sweep wait only
// for their neighbour blocks of the previous pass (Step2Args::chain)
bool t2_chain_enabled() {
    static const bool on = [] {
        const char* e = getenv("WB_T2_CHAIN");
        return !e || atoi(e) != 0;
    }();
    return on;
}

// planes per CTA of a single-step launch (tile width tw, per_sm resident
// CTAs): the same model as choose_chunk2 — about two waves or more so CTAs
// do not run in lockstep (fp64 256^3: 148 us/step at 4.8 waves vs 185 at
// one), then the fewest waves x (planes + 1).  WB_T1_CHUNK overrides.
int choose_chunk(const wo_ctx* ctx, int tw, int per_sm) {
    static const int forced = [] {   // WB_T1_CHUNK: tuning runs
        const char* e = getenv("WB_T1_CHUNK");
        return e ? atoi(e) : 0;
    }();
    if (forced > 0) return std::min(forced, std::max(ctx->kn0, 1));
    const int tiles = ((ctx->kn2 + tw - 1) / tw) * ((ctx->kn1 + BY - 1) / BY);
    const int slots = ctx->num_sms * per_sm;
    const int nz_max = std::min(ctx->kn0, 128);
    const double min_work = 1.9 * slots;
    const bool can_stagger = (double)tiles * nz_max >= min_work;
    int best_nz = 1;
    double best = 1e30;
    for (int nz = 1; nz <= nz_max; ++nz) {
        if (can_stagger && (double)tiles * nz < min_work) continue;
        const int chunk = (ctx->kn0 + nz - 1) / nz;
        const int waves = (int)(((int64_t)tiles * nz + slots - 1) / slots);
        const double cost = (double)waves * (chunk + 1);
        if (cost < best - 1e-9) { best = cost; best_nz = nz; }
    }
    return std::max(1, (ctx->kn0 + best_nz - 1) / best_nz);
}

cudaEvent_t take_event(wo_ctx* ctx) {
    cudaEvent_t e;
    if (!ctx->ev_free.empty()) {
        e = ctx->ev_free.back();
        ctx->ev_free.pop_back();
    } else {
        cudaEventCreate(&e);
    }
    ctx->ev_used.push_back(e);
    return e;
}

// bracket a step launch with events when it is one of the sampled launches
void prof_begin(wo_ctx* ctx, int kind) {
    ctx->prof_open = ctx->prof && (ctx->prof_tick++ % ctx->prof_every) == 0;
    if (!ctx->prof_open) return;
    cudaEventRecord(take_event(ctx), ctx->stream);
    ctx->ev_kind.push_back((char)kind);
}
void prof_end(wo_ctx* ctx) {
    if (ctx->prof_open) cudaEventRecord(take_event(ctx), ctx->stream);
    ctx->prof_open = false;
}

// after a stream sync: fold the bracketed step-kernel times into the stats
void harvest_events(wo_ctx* ctx) {
    for (size_t i = 0; i + 1 < ctx->ev_used.size(); i += 2) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, ctx->ev_used[i], ctx->ev_used[i + 1]) == cudaSuccess) {
            const int kind = ctx->ev_kind[i / 2] ? 1 : 0;
            ctx->step_ms += ms;
            ctx->prof_ms[kind] += ms;
            ctx->prof_n[kind] += 1;
        }
    }
    for (auto e : ctx->ev_used) ctx->ev_free.push_back(e);
    ctx->ev_used.clear();
    ctx->ev_kind.clear();
}

// ---- TMA tensor maps (driver entry point; no libcuda link dependency) ----
PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// programmatic dependent launch between peer-store launches (which stream
// memory operations separate): off unless WB_P2P_PDL=1
bool p2p_pdl() {
    static const bool on = [] {
        const char* e = getenv("WB_P2P_PDL");
        return e && atoi(e) == 1;
    }();
    return on;
}

int cu_fail(wo_ctx* ctx, const char* msg) {
    ctx->err = msg;
    return WO_ERR_CUDA;
}

// stream memory operations (flag wait / write between slab neighbours)
typedef CUresult (*PfnStreamValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PfnStreamValue32 stream_value_fn(const char* name) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        return reinterpret_cast<PfnStreamValue32>(p);
    return nullptr;
}
PfnStreamValue32 wait_value32() {
    static PfnStreamValue32 fn = stream_value_fn("cuStreamWaitValue32");
    return fn;
}
PfnStreamValue32 write_value32() {
    static PfnStreamValue32 fn = stream_value_fn("cuStreamWriteValue32");
    return fn;
}

bool make_map(CUtensorMap* m, void* base, int itemsize, uint64_t n2, uint64_t n1, uint64_t np,
              uint32_t bw, uint32_t bh) {
    auto enc = tma_encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {n2, n1, np};
    const cuuint64_t strides[2] = {n2 * (cuuint64_t)itemsize, n1 * n2 * (cuuint64_t)itemsize};
    const cuuint32_t box[3] = {bw, bh, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(m, itemsize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                            : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                           3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// whole 64 x 8 tiles and 16-byte pitches: the TMA kernel applies
bool tma_ready(wo_ctx* ctx) {
    if (ctx->tma_state == 0) {
        ctx->tma_state = -1;
        if (ctx->kn2 % PBX == 0 && ctx->kn1 % BY == 0) {
            const uint64_t np = (uint64_t)ctx->alloc_planes();
            const uint32_t hw = ctx->itemsize == 4 ? th_w<float>() : th_w<double>();
            bool ok = true;
            for (int b = 0; b < 4; ++b) {
                if (!ctx->u[b]) continue;   // buffers 2/3 exist only after a two-step pass
                ok &= make_map(&ctx->tmaps.u_halo[b], ctx->u[b], ctx->itemsize, ctx->kn2, ctx->kn1,
                               np, hw, TH_H);
                ok &= make_map(&ctx->tmaps.u_ctr[b], ctx->u[b], ctx->itemsize, ctx->kn2, ctx->kn1,
                               np, PBX, BY);
            }
            ok &= make_map(&ctx->tmaps.g_halo, ctx->gamma, ctx->itemsize, ctx->kn2, ctx->kn1, np,
                           hw, TH_H);
            ok &= make_map(&ctx->tmaps.a_ctr, ctx->acc, ctx->itemsize, ctx->kn2, ctx->kn1,
                           (uint64_t)ctx->kn0, PBX, BY);
            ctx->tmaps.lo = ctx->gl;
            if (ok) ctx->tma_state = 1;
            ++ctx->gen;
        }
    }
    return ctx->tma_state == 1;
}

struct StepSpec {
    bool acc = false;
    bool check = false;
    int backward = 0;
    double sdt = 0.0;
    int n_src = 0;
    const long long* src_flat = nullptr;
    const double* src_val = nullptr;   // fp64 values, cast to T here
    int sup_mode = SUP_NONE;
    int64_t row = 0;                   // store row (trace entry / adjoint step)
    int64_t slot = 0;                  // max slot index
    char* prev = nullptr;              // overrides of the window pointers
    char* cur = nullptr;
    char* out = nullptr;
    char* hist = nullptr;              // history row receiving a copy of out
    int c_lo = 0, c_hi = -1;           // computed planes [c_lo, c_hi) (c_hi < 0: all)
    bool peer = false;                 // peer ghost stores of the written level (p2p sweeps)
};

template <typename T>
int launch_step(wo_ctx* ctx, const StepSpec& sp) {
    StepArgs<T> a{};
    a.gamma = reinterpret_cast<const T*>(ctx->base0(ctx->gamma));
    a.u_prev = reinterpret_cast<const T*>(sp.prev ? sp.prev : ctx->uprev());
    a.u_cur = reinterpret_cast<const T*>(sp.cur ? sp.cur : ctx->ucur());
    a.u_out = reinterpret_cast<T*>(sp.out ? sp.out : ctx->uprev());
    a.hist_out = reinterpret_cast<T*>(sp.hist);
    a.acc = reinterpret_cast<T*>(ctx->acc);
    a.n0 = ctx->kn0;
    a.n1 = ctx->kn1;
    a.n2 = ctx->kn2;
    a.i_lo = ctx->has_lo ? -1 : 0;
    a.i_hi = ctx->kn0 + ctx->has_hi;
    a.c_lo = sp.c_lo;
    a.c_hi = sp.c_hi < 0 ? ctx->kn0 : std::min(sp.c_hi, ctx->kn0);
    if (a.c_hi <= a.c_lo) return WO_OK;   // empty part
    a.mat = mat_scalars<T>(ctx);
    a.cv = (T)ctx->cv;
    a.cg = (T)ctx->cg;
    a.inv2dt = (T)ctx->inv2dt;
    a.inv2dx = (T)ctx->inv2dx;
    a.sdt = (T)sp.sdt;
    a.backward = sp.backward;
    a.one_d = ctx->ndim == 1;
    a.n_src = 0;
    for (int s = 0; s < sp.n_src; ++s) {
        // local kernel-space (i, j, k) of the node; skip nodes outside the slab
        const long long f = sp.src_flat[s];
        const long long pl = ctx->plane();
        if (f < 0 || f >= ctx->cells()) continue;
        a.src_i[a.n_src] = (int)(f / pl);
        a.src_j[a.n_src] = (int)((f % pl) / ctx->kn2);
        a.src_k[a.n_src] = (int)(f % ctx->kn2);
        a.src_val[a.n_src] = (T)sp.src_val[s];
        a.n_src++;
    }
    a.sup_mode = ctx->n_sup > 0 ? sp.sup_mode : SUP_NONE;
    a.sup_lo = ctx->sup_lo;
    a.sup_hi = ctx->sup_hi;
    a.sup_mask = ctx->mask;
    a.sup_prefix = ctx->prefix;
    if (sp.sup_mode != SUP_NONE) {
        T* st = reinterpret_cast<T*>(ctx->store) + sp.row * ctx->n_sup;
        a.trace_row = st;
        a.adj_row = st;
    }
    a.max_slot = reinterpret_cast<typename FTraits<T>::Bits*>(ctx->maxslots) + sp.slot;
    if (sp.peer) {   // the written level is buffer prv (in place over u^{n-1})
        const size_t up = (size_t)(ctx->kn0 - 2) * ctx->plane() * ctx->itemsize;
        a.plo = reinterpret_cast<T*>(ctx->peer_lo[ctx->prv]);
        a.phi = ctx->peer_hi[ctx->prv] ? reinterpret_cast<T*>(ctx->peer_hi[ctx->prv] - up) : nullptr;
    }

    // whole 64x8 tiles on the default window: TMA pipeline; even rows: the
    // pair-vectorised kernel; otherwise the scalar kernel
    const bool tma = ctx->use_tma && ctx->use_pair && !sp.prev && !sp.cur && !sp.out &&
                     !sp.hist && tma_ready(ctx);
    const bool pair = tma || ((ctx->kn2 % 2 == 0) && ctx->use_pair);
    a.chunk = choose_chunk(ctx, pair ? PBX : BX, tma ? (ctx->itemsize == 4 ? 4 : 2) : 8);
    dim3 block(pair ? 32 : BX, BY, 1);
    dim3 grid(pair ? (ctx->kn2 + PBX - 1) / PBX : (ctx->kn2 + BX - 1) / BX,
              (ctx->kn1 + BY - 1) / BY, (a.c_hi - a.c_lo + a.chunk - 1) / a.chunk);
    if (tma) {
        ctx->tmaps.cur = ctx->cur;
        ctx->tmaps.prev = ctx->prv;
    }
    prof_begin(ctx, 0);
    const StepSel sel{ctx->flavor, ctx->fast_div, sp.acc, sp.check, a.sup_mode};
    const int engine = tma ? ENGINE_TMA4 : (pair ? ENGINE_PAIR : ENGINE_SCALAR);
    t_no_pdl = sp.peer && !p2p_pdl();
    ctx->t2_chain_next = false;   // the next two-step pass waits for this whole grid
    launch_step_engine<T>(engine, sel, grid, block, ctx->stream, a, ctx->tmaps);
    t_no_pdl = false;
    prof_end(ctx);
    ctx->launches++;
    ctx->step_launches++;
    CK(cudaGetLastError());
    return WO_OK;
}

// Peer ghost stores between slabs (wo_slab_peers): no exchange step.  Every
// launch stores its own planes 0, 1 / n0-2, n0-1 of the level(s) it writes
// straight into the neighbours' two ghost planes of the same level buffer
// (NVLink stores when the neighbour is another GPU; slabs rotate their buffers
// in lockstep), then bumps the neighbours' flag (cuStreamWriteValue32: its
// memory barrier makes the plane stores visible first).  Launch i of a sweep
// first waits (cuStreamWaitValue32 GEQ, on the stream: no SM spins) until both
// neighbours completed their launch i-1: their stores into our ghost planes
// are then complete, and they no longer read the ghost planes our launch i
// overwrites (it writes buffers their launch i-1 was reading).  Each sweep is
// one epoch with its own flag slot (parity): the epoch's first signal comes
// after the context's window reset (so no neighbour store can precede it) and
// the slot of the previous epoch is cleared for the next one; every epoch is
// separated from the next by a host synchronisation on all slabs (the
// stability / cost reductions), which orders those clears.
int p2p_signal(wo_ctx* ctx) {
    auto write = write_value32();
    REQUIRE(write, "stream memory operations unavailable");
    const int par = ctx->p2p_epoch & 1;
    ++ctx->p2p_seq;
    for (unsigned int* f : {ctx->peer_lo_flag, ctx->peer_hi_flag})
        if (f && write((CUstream)ctx->stream, (CUdeviceptr)(f + 2 * par), ctx->p2p_seq,
                       CU_STREAM_WRITE_VALUE_DEFAULT))
            return cu_fail(ctx, "cuStreamWriteValue32 failed");
    return WO_OK;
}

// where the device supports it, a satisfied wait also flushes the remote
// (peer / NVLink) writes that arrived before the flag, so the next launch
// sees the neighbour's ghost-plane stores
unsigned wait_flags(int device) {
    static int cached[64];
    static bool known[64] = {};
    const int d = device & 63;
    if (!known[d]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, (cudaDeviceAttr)CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES,
                               device);
        (void)cudaGetLastError();
        cached[d] = v;
        known[d] = true;
    }
    return CU_STREAM_WAIT_VALUE_GEQ | (cached[d] ? CU_STREAM_WAIT_VALUE_FLUSH : 0u);
}

int p2p_wait(wo_ctx* ctx) {
    auto wait = wait_value32();
    REQUIRE(wait, "stream memory operations unavailable");
    const int par = ctx->p2p_epoch & 1;
    const unsigned wf = wait_flags(ctx->device);
    if (ctx->peer_lo_flag &&
        wait((CUstream)ctx->stream, (CUdeviceptr)(ctx->in_flags + 2 * par), ctx->p2p_seq, wf))
        return cu_fail(ctx, "cuStreamWaitValue32 failed");
    if (ctx->peer_hi_flag &&
        wait((CUstream)ctx->stream, (CUdeviceptr)(ctx->in_flags + 2 * par + 1), ctx->p2p_seq, wf))
        return cu_fail(ctx, "cuStreamWaitValue32 failed");
    return WO_OK;
}

int p2p_epoch_begin(wo_ctx* ctx) {
    if (!ctx->p2p) return WO_OK;
    ++ctx->p2p_epoch;
    const int par = ctx->p2p_epoch & 1;
    CK(cudaMemsetAsync(ctx->in_flags + 2 * (par ^ 1), 0, 2 * sizeof(unsigned int), ctx->stream));
    ctx->p2p_seq = 0;
    return p2p_signal(ctx);   // sends 1: everything enqueued before (window reset) is done
}

// one step of a slab split for halo overlap (wo_set_option WO_OPT_PLANE_PART):
// part 1 computes the boundary planes 0 and n0-1 (whose new values the
// neighbours need), part 2 the interior; part 0 everything
template <typename T>
int launch_step_part(wo_ctx* ctx, StepSpec sp) {
    if (ctx->p2p) {   // whole step between the neighbours' flags
        REQUIRE(ctx->part == 0, "peer ghost stores run whole steps (WO_OPT_PLANE_PART 0)");
        int rc = p2p_wait(ctx);
        if (rc) return rc;
        sp.peer = true;
        rc = launch_step<T>(ctx, sp);
        if (rc) return rc;
        return p2p_signal(ctx);
    }
    if (ctx->part == 0) return launch_step<T>(ctx, sp);
    if (ctx->part == 2) {
        sp.c_lo = 1;
        sp.c_hi = ctx->kn0 - 1;
        return launch_step<T>(ctx, sp);
    }
    sp.c_lo = 0;
    sp.c_hi = 1;
    int rc = launch_step<T>(ctx, sp);
    if (rc || ctx->kn0 < 2) return rc;
    sp.c_lo = ctx->kn0 - 1;
    sp.c_hi = ctx->kn0;
    return launch_step<T>(ctx, sp);
}

// ---- CUDA graphs of repeated sweeps (see wo_ctx::SweepGraph) ----
struct KeyHash {
    uint64_t h = 1469598103934665603ull;   // FNV-1a
    void bytes(const void* p, size_t n) {
        const unsigned char* c = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
    }
    template <typename V> void val(const V& v) { bytes(&v, sizeof(v)); }
};

// the device buffers a sweep's kernel parameters point into
void hash_param_buffers(KeyHash& kh, const wo_ctx* ctx) {
    for (auto* b : ctx->u) kh.val(b);
    kh.val(ctx->gamma); kh.val(ctx->acc); kh.val(ctx->mat4); kh.val(ctx->store);
    kh.val(ctx->maxslots); kh.val(ctx->mask); kh.val(ctx->prefix); kh.val(ctx->sup_fc);
}

// true: the sweep was replayed from its graph (the caller skips its loop)
bool graph_replay(wo_ctx* ctx, int dir, uint64_t key) {
    auto& g = ctx->graph[dir];
    if (!g.exec || g.key != key) return false;
    if (cudaGraphLaunch(g.exec, ctx->stream) != cudaSuccess) return false;
    ctx->cur = g.cur;
    ctx->prv = g.prv;
    ctx->launches += g.d_launches;
    ctx->step_launches += g.d_steps;
    ctx->pair_launches += g.d_pairs;
    return true;
}

// second sighting of a key: capture this sweep's launches
bool graph_capture_begin(wo_ctx* ctx, int dir, uint64_t key) {
    auto& g = ctx->graph[dir];
    if (g.seen != key) {
        g.seen = key;
        return false;
    }
    return cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
}

int graph_capture_end(wo_ctx* ctx, int dir, uint64_t key, int64_t l0, int64_t s0, int64_t p0) {
    auto& g = ctx->graph[dir];
    cudaGraph_t graph = nullptr;
    CK(cudaStreamEndCapture(ctx->stream, &graph));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    CK(e);
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = exec;
    g.key = key;
    g.cur = ctx->cur;
    g.prv = ctx->prv;
    g.d_launches = ctx->launches - l0;
    g.d_steps = ctx->step_launches - s0;
    g.d_pairs = ctx->pair_launches - p0;
    CK(cudaGraphLaunch(exec, ctx->stream));   // the captured work has not run yet
    return WO_OK;
}

template <typename T>
double slot_value(const char* host_slots, int64_t idx) {
    using Bits = typename FTraits<T>::Bits;
    Bits b;
    std::memcpy(&b, host_slots + idx * sizeof(Bits), sizeof(Bits));
    T v;
    std::memcpy(&v, &b, sizeof(T));
    return (double)v;
}

// deduplicate nodal injections, keeping the LAST occurrence of a node
// (numpy fancy-index += semantics, solver.py:170)
void dedupe_last(int n, const int64_t* idx, std::vector<long long>& out_idx,
                 std::vector<int>& out_pos) {
    out_idx.clear();
    out_pos.clear();
    for (int s = 0; s < n; ++s) {
        bool later = false;
        for (int t = s + 1; t < n; ++t)
            if (idx[t] == idx[s]) { later = true; break; }
        if (!later) {
            out_idx.push_back((long long)idx[s]);
            out_pos.push_back(s);
        }
    }
}

int check_ctx(wo_ctx* ctx) {
    if (!ctx) return WO_ERR_CONFIG;
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) {
        ctx->err = cudaGetErrorString(e);
        return WO_ERR_CUDA;
    }
    return WO_OK;
}

int ensure_slots(wo_ctx* ctx, int64_t n) {
    return ensure(ctx, &ctx->maxslots, &ctx->maxslot_bytes, (size_t)(n + 2) * 8);
}

// ---- two-step passes (step2_kernel.cuh) ----
int ensure_four(wo_ctx* ctx) {
    const size_t ab = (size_t)ctx->alloc_cells() * ctx->itemsize;
    for (int b = 2; b < 4; ++b) {
        if (ctx->u[b]) continue;
        int rc = dev_alloc(ctx, (void**)&ctx->u[b], ab);
        if (rc) return rc;
        CK(cudaMemsetAsync(ctx->u[b], 0, ab, ctx->stream));
        ctx->tma_state = 0;   // single-step maps must cover the new buffers
        ctx->t2_state = 0;
    }
    return WO_OK;
}

// coef and face arrays of the current material for the two-step kernel, over
// the whole allocation (a slab's ghost planes included: its passes recompute
// one plane beyond each boundary; the top allocated plane's +i face is 0 and
// never used there)
int ensure_mat4(wo_ctx* ctx) {
    const size_t fb = (size_t)ctx->alloc_cells() * ctx->itemsize;
    if (!ctx->mat4) {
        int rc = dev_alloc(ctx, (void**)&ctx->mat4, 4 * fb);
        if (rc) return rc;
        ctx->t2_state = 0;
        ctx->mat4_valid = false;
    }
    if (!ctx->mat4_valid) {
        char* g = ctx->gamma;
        const int np = ctx->alloc_planes();
        if (ctx->itemsize == 4)
            launch_material4<float>(ctx->flavor, ctx->stream, reinterpret_cast<const float*>(g),
                                    mat_scalars<float>(ctx), np, ctx->kn1, ctx->kn2,
                                    reinterpret_cast<float*>(ctx->mat4));
        else
            launch_material4<double>(ctx->flavor, ctx->stream, reinterpret_cast<const double*>(g),
                                     mat_scalars<double>(ctx), np, ctx->kn1, ctx->kn2,
                                     reinterpret_cast<double*>(ctx->mat4));
        ctx->launches++;
        CK(cudaGetLastError());
        ctx->mat4_valid = true;
    }
    return WO_OK;
}

// fc(gamma) of every support node for the two-step kernel's adjoint
// injection (sup_fc_kernel), rebuilt when gamma or the support changes;
// called from pair_ready, i.e. before a sweep's graph capture
int ensure_sup_fc(wo_ctx* ctx) {
    if (ctx->sup_fc_valid || ctx->n_sup == 0) return WO_OK;
    int rc = ensure(ctx, &ctx->sup_fc, &ctx->sup_fc_bytes, (size_t)ctx->n_sup * ctx->itemsize);
    if (rc) return rc;
    const char* g = ctx->base0(ctx->gamma);
    const long long n = ctx->n_sup;
    const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 592);
    if (ctx->itemsize == 4) {
        const MatScalars<float> M = mat_scalars<float>(ctx);
        const float* gf = reinterpret_cast<const float*>(g);
        float* o = reinterpret_cast<float*>(ctx->sup_fc);
        if (ctx->flavor == RHO_SCALED)
            sup_fc_kernel<float, RHO_SCALED><<<blocks, 256, 0, ctx->stream>>>(gf, M, ctx->sup_flat, n, o);
        else
            sup_fc_kernel<float, ACOUSTIC><<<blocks, 256, 0, ctx->stream>>>(gf, M, ctx->sup_flat, n, o);
    } else {
        const MatScalars<double> M = mat_scalars<double>(ctx);
        const double* gd = reinterpret_cast<const double*>(g);
        double* o = reinterpret_cast<double*>(ctx->sup_fc);
        if (ctx->flavor == RHO_SCALED)
            sup_fc_kernel<double, RHO_SCALED><<<blocks, 256, 0, ctx->stream>>>(gd, M, ctx->sup_flat, n, o);
        else
            sup_fc_kernel<double, ACOUSTIC><<<blocks, 256, 0, ctx->stream>>>(gd, M, ctx->sup_flat, n, o);
    }
    ctx->launches++;
    CK(cudaGetLastError());
    ctx->sup_fc_valid = true;
    return WO_OK;
}

// tile geometry for a two-step pass: 64 x 8 where it divides the plane, else
// 32 x 16 (measured equal at 256^3: 214 vs 212 Gcell/s; the tall tile's
// balanced warps and smaller ring are offset by narrower TMA rows);
// WB_T2_GEO=wide|tall forces one
int pick_geo(const wo_ctx* ctx) {
    static const int forced = [] {
        const char* e = getenv("WB_T2_GEO");
        if (!e) return (int)GEO_NONE;
        return strcmp(e, "wide") == 0 ? (int)GEO_WIDE : strcmp(e, "tall") == 0 ? (int)GEO_TALL
                                                                               : (int)GEO_NONE;
    }();
    const bool tall = ctx->kn2 % GeoTall::TBX == 0 && ctx->kn1 % GeoTall::TBY == 0;
    const bool wide = ctx->kn2 % GeoWide::TBX == 0 && ctx->kn1 % GeoWide::TBY == 0;
    if (forced == GEO_TALL && tall) return GEO_TALL;
    if (forced == GEO_WIDE && wide) return GEO_WIDE;
    return wide ? GEO_WIDE : tall ? GEO_TALL : GEO_NONE;
}

bool pair_ready(wo_ctx* ctx) {
    if (!ctx->use_two_step || !ctx->use_tma || !ctx->use_pair || ctx->part != 0 ||
        !ctx->material_set || pick_geo(ctx) == GEO_NONE)
        return false;
    // slabs: two ghost planes at every neighbour and at least two own planes
    // (the peer stores cover planes 0, 1 and n0-2, n0-1)
    if ((ctx->has_lo && ctx->gl < 2) || (ctx->has_hi && ctx->gh < 2) ||
        ((ctx->has_lo || ctx->has_hi) && ctx->kn0 < 2))
        return false;
    // fp64 two-step passes run 2 ring stages at 2 CTAs per SM (98 KB each):
    // 256^3 125-134 vs 106 Gcell-upd/s single-step, 512^3 127.7 vs 120.8,
    // 1024^3 125.7 vs 120.2 (profiles/r2/f64_two_step.txt); round 1's
    // 3-stage, 1-CTA variant was slower, so fp64 used to need option 2
    if (ctx->t2_oom) return false;
    if (ensure_four(ctx) || ensure_mat4(ctx)) {
        // the two extra levels and the material do not fit next to the rest:
        // give back what was taken and keep single steps (four field buffers)
        if (ctx->has_lo || ctx->has_hi) {   // slabs keep their 4 levels (peers)
            ctx->t2_oom = true;
            return false;
        }
        for (int b = 2; b < 4; ++b)
            if (ctx->u[b]) {
                cudaFree(ctx->u[b]);
                ctx->u[b] = nullptr;
                ctx->dev_bytes -= (int64_t)ctx->alloc_cells() * ctx->itemsize;
            }
        if (ctx->mat4) {
            cudaFree(ctx->mat4);
            ctx->mat4 = nullptr;
            ctx->dev_bytes -= 4 * (int64_t)ctx->alloc_cells() * ctx->itemsize;
        }
        ctx->tma_state = 0;
        ctx->t2_oom = true;
        return false;
    }
    if (ctx->t2_state == 0) {
        ctx->t2_state = -1;
        const int geo = pick_geo(ctx);
        const uint64_t np = (uint64_t)ctx->alloc_planes();   // plane coordinate = p + gl
        const uint32_t tbx = geo == GEO_TALL ? GeoTall::TBX : GeoWide::TBX;
        const uint32_t tby = geo == GEO_TALL ? GeoTall::TBY : GeoWide::TBY;
        const uint32_t hw = tbx + 2 * (ctx->itemsize == 4 ? th_ho<float>() : th_ho<double>());
        const uint32_t r2 = tby + 4, r1 = tby + 2;
        const size_t fb = (size_t)ctx->alloc_cells() * ctx->itemsize;
        bool ok = true;
        for (int b = 0; b < 4; ++b) {
            ok &= make_map(&ctx->t2maps.u_r2[b], ctx->u[b], ctx->itemsize, ctx->kn2, ctx->kn1, np,
                           hw, r2);
            ok &= make_map(&ctx->t2maps.u_r1[b], ctx->u[b], ctx->itemsize, ctx->kn2, ctx->kn1, np,
                           hw, r1);
        }
        ok &= make_map(&ctx->t2maps.c_r1, ctx->mat4, ctx->itemsize, ctx->kn2, ctx->kn1, np, hw, r1);
        ok &= make_map(&ctx->t2maps.fk_r1, ctx->mat4 + fb, ctx->itemsize, ctx->kn2, ctx->kn1, np,
                       hw, r1);
        ok &= make_map(&ctx->t2maps.fj_r2, ctx->mat4 + 2 * fb, ctx->itemsize, ctx->kn2, ctx->kn1,
                       np, hw, r2);
        ok &= make_map(&ctx->t2maps.fi_r1, ctx->mat4 + 3 * fb, ctx->itemsize, ctx->kn2, ctx->kn1,
                       np, hw, r1);
        ok &= make_map(&ctx->t2maps.a_ctr, ctx->acc, ctx->itemsize, ctx->kn2, ctx->kn1,
                       (uint64_t)ctx->kn0, tbx, tby);
        if (ok) {
            ctx->t2_state = 1;
            ++ctx->gen;
            ctx->t2_geo = geo;
        }
    }
    if (ctx->t2_state == 1 && ensure_sup_fc(ctx)) {   // out of memory: single steps
        if (ctx->has_lo || ctx->has_hi) ctx->t2_oom = true;   // slabs must launch alike (REQUIRE)
        return false;
    }
    return ctx->t2_state == 1;
}

// planes per CTA of a two-step pass.  Measured: a grid that fits in ONE wave
// of resident CTAs runs its CTAs in lockstep (all loading, then all
// computing) and is ~1.35x slower per plane than the same work spread over
// two or more waves, whose staggered CTAs overlap memory and compute (192^3:
// 106 vs 79 us per pass; 256^3 with 384 CTAs: 267 vs 137 us); partial last
// waves idle slots, and each chunk recomputes ~1 extra plane.  Model: at
// least ~2 waves of work when the grid allows it, then the fewest
// waves x (planes + 1).  WB_T2_NZ overrides (tuning runs).
constexpr double T2_LONG_CHUNK_PENALTY = 1.7e-4;   // per plane beyond 32

int choose_chunk2(const wo_ctx* ctx) {
    const int tbx = ctx->t2_geo == GEO_TALL ? GeoTall::TBX : GeoWide::TBX;
    const int tby = ctx->t2_geo == GEO_TALL ? GeoTall::TBY : GeoWide::TBY;
    const int tiles = (ctx->kn2 / tbx) * (ctx->kn1 / tby);
    static const int forced = [] {
        const char* e = getenv("WB_T2_NZ");
        return e ? atoi(e) : 0;
    }();
    int best_nz = 1;
    if (forced > 0) {
        best_nz = forced;
    } else {
        const int slots = ctx->num_sms * (ctx->itemsize == 4 ? T2_CTAS_F32 : T2_CTAS_F64);
        const int nz_max = std::min(ctx->kn0, 64);
        // dataflow-chained passes (t2_chain_enabled) overlap one pass's tail
        // with the next pass's start, so partial waves cost their CTAs only:
        // a continuous wave count, with >= 2.2 waves of CTAs (256^3: 8
        // layers, 254.9 Gcell/s, vs 250.4 for the whole-wave model's 10;
        // 7 layers / 2.0 waves 248.4; profiles/r2/nz_chain.txt)
        const bool chained = t2_chain_enabled() && !ctx->p2p && WB_T2_PDL;
        const double min_work = (chained ? 2.2 : 1.9) * slots;   // CTAs for ~2 waves
        const bool can_stagger = (double)tiles * nz_max >= min_work;
        double best = 1e30;
        for (int nz = 1; nz <= nz_max; ++nz) {
            if (can_stagger && (double)tiles * nz < min_work) continue;
            const int chunk = (ctx->kn0 + nz - 1) / nz;
            if (chained && chunk < 2 && nz > 1) continue;   // chaining needs >= 2 planes
            // (grids too small for two waves keep whole waves: fewer, longer
            // layers would only idle SMs)
            const double waves = chained && can_stagger
                                     ? (double)tiles * nz / slots
                                     : (double)((tiles * nz + slots - 1) / slots);
            // chunks past 32 planes also lose per plane (measured at 1024^3:
            // 128-plane chunks 222-260 Gcell/s, 64-plane 279-280; 512^3 keeps
            // 86): a mild length penalty on top of the wave count
            const double cost = waves * (chunk + 1) *
                                (1.0 + T2_LONG_CHUNK_PENALTY * std::max(0, chunk - 32));
            if (cost < best - 1e-9) { best = cost; best_nz = nz; }
        }
    }
    return std::max(1, (ctx->kn0 + best_nz - 1) / best_nz);
}

// z layers of a two-step launch: boundaries zb[0..nz] (returns nz).  Uniform
// chunks of choose_chunk2 unless WB_T2_LAYERS="len x count,..." (tuning
// runs; layers in launch order, lengths must sum to n0).
int n0_min_layer(const int* zb, int nz) {
    int m = 1 << 30;
    for (int z = 0; z < nz; ++z) m = std::min(m, zb[z + 1] - zb[z]);
    return m;
}

int choose_layers2(const wo_ctx* ctx, int* zb) {
    static const std::string spec = [] {
        const char* e = getenv("WB_T2_LAYERS");
        return std::string(e ? e : "");
    }();
    const int n0 = ctx->kn0;
    if (!spec.empty()) {
        int nz = 0, pos = 0;
        zb[0] = 0;
        size_t i = 0;
        bool ok = true;
        while (ok && i < spec.size()) {
            int len = 0, cnt = 0;
            if (sscanf(spec.c_str() + i, "%dx%d", &len, &cnt) != 2 || len < 1 || cnt < 1) ok = false;
            for (int c = 0; ok && c < cnt; ++c) {
                if (nz >= T2_MAXZ) { ok = false; break; }
                pos += len;
                zb[++nz] = pos;
            }
            const size_t comma = spec.find(',', i);
            i = comma == std::string::npos ? spec.size() : comma + 1;
        }
        if (ok && pos == n0) return nz;
    }
    const int chunk = choose_chunk2(ctx);
    int nz = 0;
    zb[0] = 0;
    for (int p = 0; p < n0 && nz < T2_MAXZ; p += chunk) zb[++nz] = std::min(p + chunk, n0);
    zb[nz] = n0;
    return nz;
}

// start of a run of two-step passes (a sweep): fresh block flags, so the
// values a captured sweep graph bakes in repeat on every replay
int t2_sweep_begin(wo_ctx* ctx) {
    ctx->t2_seq = 0;
    ctx->t2_chain_next = false;
    if (!ctx->tflags || ctx->p2p || !t2_chain_enabled()) return WO_OK;
    CK(cudaMemsetAsync(ctx->tflags, 0, ctx->tflags_bytes, ctx->stream));
    return WO_OK;
}

// ---- cluster-resident whole sweeps of small 2D grids (cluster_sweep.cuh) ----


// support slots a register-resident CTA may need (even, for the T array after them)
int64_t cluster_reg_sup_cap(const wo_ctx* ctx, int rows) {
    const int64_t cap = std::min<int64_t>(ctx->n_sup, (int64_t)rows * ctx->kn2);
    return cap + (cap & 1);
}

// Cluster engine of a sweep: 2 register-resident (cluster_reg.cuh: up to 16
// CTAs x 1024 threads x 2x2 cells = 65,536 cells), 1 shared-memory
// (cluster_sweep.cuh, WB_CLUSTER_ENGINE=smem), 0 none.
template <typename T>
int cluster_engine(wo_ctx* ctx) {
    const bool on = ctx->use_cluster != 0;
    const bool shape_ok = on && ctx->ndim == 2 && ctx->kn0 == 1 && !ctx->has_lo &&
                          !ctx->has_hi;
    if (ctx->cr_state == 0) {
        ctx->cr_state = -1;
        if (shape_ok && !cluster_smem_engine()) {
            int rows = (ctx->kn1 + CS_MAX_CLUSTER - 1) / CS_MAX_CLUSTER;
            rows += rows & 1;
            const int cl = (ctx->kn1 + rows - 1) / rows;
            const int pc = cluster_reg_pc();
            if (cr_txn(ctx->kn2, pc) * (rows / 2) <= CR_THREADS / pc &&
                cluster_reg_smem<T>(rows, ctx->kn2, 0, pc) + 1024 <= 227 * 1024) {
                ClusterSweepArgs<T> a{};
                a.reg = 1;
                a.pc = pc;
                a.rows = rows;
                a.n2 = ctx->kn2;
                if (launch_cluster_sweep<T>(RHO_SCALED, true, a, cl, ctx->stream, true) ==
                    cudaSuccess) {
                    ctx->cr_state = 1;
                    ctx->cr_size = cl;
                    ctx->cr_rows = rows;
                }
            }
            (void)cudaGetLastError();
        }
    }
    if (ctx->cr_state == 1 &&
        cluster_reg_smem<T>(ctx->cr_rows, ctx->kn2, cluster_reg_sup_cap(ctx, ctx->cr_rows),
                            cluster_reg_pc()) + 1024 <= 227 * 1024)
        return 2;
    if (ctx->cl_state == 0) {
        ctx->cl_state = -1;
        if (shape_ok && cluster_smem_engine() && ctx->kn1 >= 2 * CS_MAX_CLUSTER) {
            const int rows = (ctx->kn1 + CS_MAX_CLUSTER - 1) / CS_MAX_CLUSTER;
            const int cl = (ctx->kn1 + rows - 1) / rows;
            if (cluster_sweep_smem<T>(rows, ctx->kn2) + 1024 <= 227 * 1024 &&
                rows * ctx->kn2 <= CS_MAXC * CS_THREADS) {
                ClusterSweepArgs<T> a{};
                a.rows = rows;
                a.n2 = ctx->kn2;
                if (launch_cluster_sweep<T>(RHO_SCALED, true, a, cl, ctx->stream, true) ==
                    cudaSuccess) {
                    ctx->cl_state = 1;
                    ctx->cl_size = cl;
                    ctx->cl_rows = rows;
                }
            }
            (void)cudaGetLastError();
        }
    }
    return ctx->cl_state == 1 ? 1 : 0;
}
template <typename T>
bool cluster_ready(wo_ctx* ctx) {
    return cluster_engine<T>(ctx) != 0;
}

// steps n_first, n_first +- 1, ... (count of them) of an N-step sweep in one
// launch; the window indices rotate as count single steps would
template <typename T>
int run_cluster_sweep(wo_ctx* ctx, int backward, int64_t N, int64_t n_first, int64_t count,
                      int ns, const long long* sidx, const double* const* amp_rows, bool acc,
                      double sdt, int sup_mode) {
    ClusterSweepArgs<T> a{};
    const int engine = cluster_engine<T>(ctx);
    REQUIRE(engine != 0, "no cluster engine for this context");
    a.reg = engine == 2;
    a.pc = cluster_reg_pc();
    a.n1 = ctx->kn1;
    a.n2 = ctx->kn2;
    a.rows = a.reg ? ctx->cr_rows : ctx->cl_rows;
    a.sup_cap = a.reg ? (int)cluster_reg_sup_cap(ctx, a.rows) : 0;
    a.negz2 = 0x8000000080000000ull;
    a.backward = backward;
    a.n_first = (int)n_first;
    a.n_count = (int)count;
    a.N = N;
    a.gamma = reinterpret_cast<const T*>(ctx->base0(ctx->gamma));
    a.u_prev_in = reinterpret_cast<const T*>(ctx->uprev());
    a.u_cur_in = reinterpret_cast<const T*>(ctx->ucur());
    if (count % 2) std::swap(ctx->cur, ctx->prv);
    a.u_prev_out = reinterpret_cast<T*>(ctx->uprev());
    a.u_cur_out = reinterpret_cast<T*>(ctx->ucur());
    a.acc = reinterpret_cast<T*>(ctx->acc);
    a.accumulate = acc;
    a.mat = mat_scalars<T>(ctx);
    a.cv = (T)ctx->cv; a.cg = (T)ctx->cg; a.inv2dt = (T)ctx->inv2dt; a.inv2dx = (T)ctx->inv2dx;
    a.sdt = (T)sdt;
    a.n_src = 0;
    std::vector<double> table;
    for (int s = 0; s < ns; ++s) {
        const long long f = sidx[s];
        if (f < 0 || f >= ctx->cells()) continue;
        a.src_j[a.n_src] = (int)(f / ctx->kn2);
        a.src_k[a.n_src] = (int)(f % ctx->kn2);
        table.insert(table.end(), amp_rows[s], amp_rows[s] + N);
        a.n_src++;
    }
    if (a.n_src) {
        int rc = ensure(ctx, &ctx->amp_dev, &ctx->amp_cap, table.size() * sizeof(double));
        if (rc) return rc;
        CK(cudaMemcpyAsync(ctx->amp_dev, table.data(), table.size() * sizeof(double),
                           cudaMemcpyHostToDevice, ctx->stream));
        a.src_amp = ctx->amp_dev;
    }
    a.sup_mode = ctx->n_sup > 0 ? sup_mode : SUP_NONE;
    a.n_sup = ctx->n_sup;
    a.sup_mask = ctx->mask;
    a.sup_prefix = ctx->prefix;
    a.store = reinterpret_cast<T*>(ctx->store);
    a.maxslots = reinterpret_cast<typename FTraits<T>::Bits*>(ctx->maxslots);
    prof_begin(ctx, 0);
    const cudaError_t e = launch_cluster_sweep<T>(ctx->flavor, acc, a,
                                                  a.reg ? ctx->cr_size : ctx->cl_size,
                                                  ctx->stream, false);
    prof_end(ctx);
    ctx->launches++;
    ctx->step_launches++;
    ctx->t2_chain_next = false;
    CK(e);
    CK(cudaGetLastError());
    if (a.n_src) CK(cudaStreamSynchronize(ctx->stream));   // host table lifetime
    return WO_OK;
}

struct PairSpec {
    bool acc = false, check1 = false, check2 = false;
    double sdt = 0.0;
    int n_src = 0;
    const long long* src_flat = nullptr;
    const double* val1 = nullptr;
    const double* val2 = nullptr;
    int sup_mode = SUP_NONE;
    int64_t row1 = 0, row2 = 0, slot1 = 0, slot2 = 0;
};

template <typename T>
int launch_pair(wo_ctx* ctx, const PairSpec& sp) {
    int x[2], nx = 0;
    for (int b = 0; b < 4 && nx < 2; ++b)
        if (b != ctx->cur && b != ctx->prv) x[nx++] = b;
    Step2Args<T> a{};
    a.gamma = reinterpret_cast<const T*>(ctx->base0(ctx->gamma));
    a.u_prev = reinterpret_cast<const T*>(ctx->uprev());
    a.u_cur = reinterpret_cast<const T*>(ctx->ucur());
    a.fi = reinterpret_cast<const T*>(
        ctx->base0(ctx->mat4 + 3 * (size_t)ctx->alloc_cells() * ctx->itemsize));
    a.out1 = reinterpret_cast<T*>(ctx->base0(ctx->u[x[0]]));
    a.out2 = reinterpret_cast<T*>(ctx->base0(ctx->u[x[1]]));
    a.acc = reinterpret_cast<T*>(ctx->acc);
    a.n0 = ctx->kn0; a.n1 = ctx->kn1; a.n2 = ctx->kn2;
    const int nz = choose_layers2(ctx, a.zb);
    a.chunk = 0;
    for (int z = 0; z < nz; ++z) a.chunk = std::max(a.chunk, a.zb[z + 1] - a.zb[z]);
    a.resident = ctx->num_sms * (ctx->itemsize == 4 ? T2_CTAS_F32 : T2_CTAS_F64);
    a.negz = 0x8000000080000000ull;   // (-0.0f, -0.0f): packed fp32 products
    a.mat = mat_scalars<T>(ctx);
    a.cv = (T)ctx->cv; a.cg = (T)ctx->cg; a.inv2dt = (T)ctx->inv2dt; a.inv2dx = (T)ctx->inv2dx;
    a.sdt = (T)sp.sdt;
    a.lo_open = ctx->has_lo;
    a.hi_open = ctx->has_hi;
    a.zo = ctx->gl;
    if (ctx->p2p) {
        const size_t pb = (size_t)ctx->plane() * ctx->itemsize;
        const size_t up = (size_t)(ctx->kn0 - 2) * pb;   // own plane n0-2 -> ghost plane -2
        a.plo1 = reinterpret_cast<T*>(ctx->peer_lo[x[0]]);
        a.plo2 = reinterpret_cast<T*>(ctx->peer_lo[x[1]]);
        a.phi1 = ctx->peer_hi[x[0]] ? reinterpret_cast<T*>(ctx->peer_hi[x[0]] - up) : nullptr;
        a.phi2 = ctx->peer_hi[x[1]] ? reinterpret_cast<T*>(ctx->peer_hi[x[1]] - up) : nullptr;
    }
    a.n_src = 0;
    for (int s = 0; s < sp.n_src; ++s) {
        // local (i, j, k); a slab also takes sources on its ghost planes,
        // whose step n it recomputes
        const long long f = sp.src_flat[s];
        const long long pl = ctx->plane();
        if (f < -(long long)ctx->gl * pl || f >= ctx->cells() + (long long)ctx->gh * pl) continue;
        const long long pi = f >= 0 ? f / pl : -((-f + pl - 1) / pl);
        const long long r = f - pi * pl;
        a.src_i[a.n_src] = (int)pi;
        a.src_j[a.n_src] = (int)(r / ctx->kn2);
        a.src_k[a.n_src] = (int)(r % ctx->kn2);
        a.src_val1[a.n_src] = (T)sp.val1[s];
        a.src_val2[a.n_src] = (T)sp.val2[s];
        a.n_src++;
    }
    const int sup = ctx->n_sup > 0 ? sp.sup_mode : SUP_NONE;
    a.sup_lo = ctx->sup_lo; a.sup_hi = ctx->sup_hi;
    a.sup_mask = ctx->mask; a.sup_prefix = ctx->prefix;
    a.sup_fc = reinterpret_cast<const T*>(ctx->sup_fc);
    if (sup != SUP_NONE) {
        a.row1 = reinterpret_cast<T*>(ctx->store) + sp.row1 * ctx->n_sup;
        a.row2 = reinterpret_cast<T*>(ctx->store) + sp.row2 * ctx->n_sup;
    }
    a.check1 = sp.check1; a.check2 = sp.check2;
    // dataflow chaining: only right after a pass of this sweep, with z layers
    // of >= 2 planes (the 3x3x3 block neighbourhood then covers every plane a
    // block reads or overwrites), PDL launches and no stream operations
    // between.  (Single-layer 2D grids measured slower chained: C1 17.9 vs
    // 24.3 Gcell-upd/s — there the whole-grid dependency resolves faster than
    // the flag publish + poll; profiles/dev/cycle28.sh)
    int min_layer = n0_min_layer(a.zb, nz);
    const bool chain_ok = t2_chain_enabled() && !ctx->p2p && WB_T2_PDL && min_layer >= 2;
    if (chain_ok && !ctx->tflags) {
        const size_t need = (size_t)(ctx->kn2 / 32 + 1) * (ctx->kn1 / 8 + 1) * (T2_MAXZ + 1) * 4;
        if (dev_alloc(ctx, (void**)&ctx->tflags, need) == WO_OK) {
            ctx->tflags_bytes = need;
            CK(cudaMemsetAsync(ctx->tflags, 0, need, ctx->stream));
        }
        ctx->t2_chain_next = false;   // flags fresh from here on
    }
    if (chain_ok && ctx->tflags) {
        a.tflags = ctx->tflags;
        a.seq = ++ctx->t2_seq;
        a.chain = ctx->t2_chain_next ? 1 : 0;
        // WB_T2_ZREV=1: alternate the layer dispatch order from pass to pass
        static const bool zrev = [] {
            const char* e = getenv("WB_T2_ZREV");
            return e && atoi(e) != 0;
        }();
        a.zrev = zrev ? (int)(a.seq & 1u) : 0;
    }
    a.max1 = reinterpret_cast<typename FTraits<T>::Bits*>(ctx->maxslots) + sp.slot1;
    a.max2 = reinterpret_cast<typename FTraits<T>::Bits*>(ctx->maxslots) + sp.slot2;
    ctx->t2maps.prev = ctx->prv;
    ctx->t2maps.cur = ctx->cur;
    const int tbx = ctx->t2_geo == GEO_TALL ? GeoTall::TBX : GeoWide::TBX;
    const int tby = ctx->t2_geo == GEO_TALL ? GeoTall::TBY : GeoWide::TBY;
    dim3 grid(ctx->kn2 / tbx, ctx->kn1 / tby, nz);
#if WB_T2_TIMELINE
    // dev builds: the WB_T2_TL_CALL-th pair launch writes its CTA timeline
    // (header: grid x, y, z, chunk; then start, first data, end, smid per CTA)
    // to WB_T2_TL_FILE (profiles/dev/cta_timeline.py)
    static unsigned long long* d_tl = nullptr;
    static int tl_calls = 0;
    const size_t nblk = (size_t)grid.x * grid.y * grid.z;
    if (!d_tl) cudaMalloc(&d_tl, (size_t)32 << 20);
    a.timeline = nblk <= (1u << 20) ? d_tl : nullptr;
#endif
    if (ctx->p2p) {
        const int rc = p2p_wait(ctx);
        if (rc) return rc;
    }
    prof_begin(ctx, 1);
    t_no_pdl = ctx->p2p && !p2p_pdl();
    // feature level (T2Mode): peer stores or cell offsets beyond 32 bits ->
    // T2_FULL; completion flags -> T2_CHAIN; else the lean T2_BASE
    const bool big = (int64_t)(ctx->kn0 + 2) * ctx->plane() >= (int64_t)INT32_MAX;
    const int mode = (ctx->p2p || a.plo1 || a.phi1 || big) ? T2_FULL
                     : a.tflags                           ? T2_CHAIN
                                                          : T2_BASE;
    launch_step2_engine<T>(StepSel{ctx->flavor, true, sp.acc, false, sup}, ctx->t2_geo, mode, grid,
                           ctx->stream, a, ctx->t2maps);
    t_no_pdl = false;
    prof_end(ctx);
#if WB_T2_TIMELINE
    {
        const char* want = getenv("WB_T2_TL_CALL");
        const char* path = getenv("WB_T2_TL_FILE");
        if (++tl_calls == (want ? atoi(want) : -1) && path && a.timeline) {
            std::vector<unsigned long long> h(4 * nblk + 4);
            h[0] = grid.x; h[1] = grid.y; h[2] = grid.z; h[3] = (unsigned long long)a.chunk;
            cudaStreamSynchronize(ctx->stream);
            cudaMemcpy(h.data() + 4, d_tl, 4 * 8 * nblk, cudaMemcpyDeviceToHost);
            if (FILE* f = fopen(path, "wb")) {
                fwrite(h.data(), 8, h.size(), f);
                fclose(f);
            }
        }
    }
#endif
    ctx->launches++;
    ctx->step_launches++;
    ctx->pair_launches++;
    CK(cudaGetLastError());
    ctx->prv = x[0];
    ctx->cur = x[1];
    ctx->t2_chain_next = a.tflags != nullptr;
    return ctx->p2p ? p2p_signal(ctx) : WO_OK;
}

template <typename T>
int inject_host_list(wo_ctx* ctx, int n, const long long* idx, const double* vals) {
    // > MAX_SRC nodes: separate injection kernel after the step (no kernel
    // increment follows in these modes, so the order matches solver.py:173-177)
    int rc = ensure(ctx, &ctx->f_idx, &ctx->f_idx_cap, (size_t)n * 8);
    if (rc) return rc;
    rc = ensure(ctx, &ctx->f_vals, &ctx->f_vals_cap, (size_t)n * sizeof(T));
    if (rc) return rc;
    std::vector<T> tv(n);
    for (int s = 0; s < n; ++s) tv[s] = (T)vals[s];
    CK(cudaMemcpyAsync(ctx->f_idx, idx, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->f_vals, tv.data(), (size_t)n * sizeof(T), cudaMemcpyHostToDevice,
                       ctx->stream));
    // u_out was written into the prev buffer; after rotation it is ucur
    inject_kernel<T><<<(n + 127) / 128, 128, 0, ctx->stream>>>(
        reinterpret_cast<T*>(ctx->uprev()), reinterpret_cast<const T*>(ctx->base0(ctx->gamma)),
        mat_scalars<T>(ctx), ctx->f_idx, reinterpret_cast<const T*>(ctx->f_vals), n);
    ctx->launches++;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));  // host vector lifetime
    return WO_OK;
}

// forward steps n in [n_begin, n_end) of an N-step sweep; n_begin == 1
// initialises the check slots / store / history, finish evaluates the checks
template <typename T>
int sweep_forward_t(wo_ctx* ctx, int64_t N, int n_src, const int64_t* src_flat,
                    const double* src_amp, int flags, double dt, double scale,
                    double* peak_out, int64_t* fail_step, double* fail_max,
                    int64_t n_begin = 1, int64_t n_end = -1, bool finish = true) {
    if (n_end < 0) n_end = N;
    REQUIRE(1 <= n_begin && n_begin <= n_end && n_end <= N, "bad forward step range");
    const int accumulate = flags & WO_FWD_ACCUMULATE;
    const bool record = (flags & WO_FWD_HISTORY) != 0;
    const bool first = n_begin == 1;
    if (record && first) {
        REQUIRE(!ctx->has_lo && !ctx->has_hi, "history recording is single-domain only");
        int rc0 = ensure(ctx, &ctx->hist, &ctx->hist_bytes, (size_t)(N + 1) * ctx->field_bytes());
        if (rc0) return rc0;
        // history[0] = u_prev, history[1] = u_cur (gradients.py:233-235)
        CK(cudaMemcpyAsync(ctx->hist, ctx->uprev(), ctx->field_bytes(), cudaMemcpyDeviceToDevice,
                           ctx->stream));
        CK(cudaMemcpyAsync(ctx->hist + ctx->field_bytes(), ctx->ucur(), ctx->field_bytes(),
                           cudaMemcpyDeviceToDevice, ctx->stream));
    }
    std::vector<long long> sidx;
    std::vector<int> spos;
    dedupe_last(n_src, src_flat, sidx, spos);
    const int ns = (int)sidx.size();
    REQUIRE(ns <= MAX_SRC || !accumulate, "at most 8 source nodes per accumulating sweep");
    REQUIRE(!record || ctx->hist_bytes >= (size_t)(N + 1) * ctx->field_bytes(),
            "history not initialised");
    int rc = WO_OK;
    const bool gather = ctx->n_sup > 0;
    REQUIRE(ctx->part == 0 || (n_end - n_begin <= 1 && ns <= MAX_SRC && !record),
            "split (boundary / interior) steps go one in-kernel-source step per call");
    REQUIRE(!ctx->p2p || (ns <= MAX_SRC && !record),
            "peer-store sweeps take at most 8 in-kernel source nodes and no history");
    if (first && ctx->part != 2) {
        rc = ensure_slots(ctx, N);
        if (rc) return rc;
        CK(cudaMemsetAsync(ctx->maxslots, 0, (size_t)(N + 2) * 8, ctx->stream));
        if (gather) {
            rc = ensure(ctx, &ctx->store, &ctx->store_bytes, (size_t)N * ctx->n_sup * sizeof(T));
            if (rc) return rc;
            CK(cudaMemsetAsync(ctx->store, 0, (size_t)N * ctx->n_sup * sizeof(T), ctx->stream));
        }
        rc = p2p_epoch_begin(ctx);
        if (rc) return rc;
    }
    REQUIRE(ctx->maxslot_bytes >= (size_t)(N + 2) * 8 &&
                (!gather || ctx->store_bytes >= (size_t)N * ctx->n_sup * sizeof(T)),
            "sweep not initialised (first range must start at n = 1)");
    std::vector<double> vals(std::max(ns, 1));
    auto fcheck = [&](int64_t n) { return (n % STABILITY_CHECK_INTERVAL == 0) || (n == N - 1); };
    // small 2D grids: the whole range in one cluster-resident launch
    const bool cluster = !record && ns <= MAX_SRC && ctx->part == 0 && !ctx->p2p &&
                         n_end > n_begin && cluster_ready<T>(ctx);
    if (cluster) {
        std::vector<const double*> rows(ns);
        for (int s = 0; s < ns; ++s) rows[s] = src_amp + (int64_t)spos[s] * N;
        rc = run_cluster_sweep<T>(ctx, 0, N, n_begin, n_end - n_begin, ns, sidx.data(), rows.data(),
                                  accumulate != 0, -dt, gather ? SUP_GATHER : SUP_NONE);
        if (rc) return rc;
        n_end = n_begin;   // nothing left for the step loop
    }
    const bool pairs = ns <= MAX_SRC && !record && pair_ready(ctx);
    // a peer-store slab must launch exactly like its neighbours
    REQUIRE(!(ctx->p2p && ctx->t2_oom && ctx->use_two_step),
            "two-step buffers do not fit on this peer-store slab: disable two-step passes on "
            "every slab of the decomposition (wo_prepare_two_step)");
    std::vector<double> vals2(std::max(ns, 1));
    // graph of this sweep: the key covers everything the launches depend on
    // beyond the state generation
    const bool graphable = ctx->use_graphs && !ctx->prof && ctx->part == 0 && !record &&
                           !ctx->p2p && !cluster && ns <= MAX_SRC && n_end - n_begin >= 8;
    uint64_t gkey = 0;
    bool capturing = false;
    const int64_t l0 = ctx->launches, s0 = ctx->step_launches, p0 = ctx->pair_launches;
    if (graphable) {
        KeyHash kh;
        kh.val(0); kh.val(N); kh.val(n_begin); kh.val(n_end); kh.val(flags); kh.val(dt);
        kh.val(ctx->gen); kh.val(ctx->cur); kh.val(ctx->prv); kh.val(ns); kh.val(gather);
        kh.val((int)sizeof(T));
        hash_param_buffers(kh, ctx);
        for (int s = 0; s < ns; ++s) {
            kh.val(sidx[s]);
            kh.bytes(src_amp + (int64_t)spos[s] * N + n_begin, (size_t)(n_end - n_begin) * 8);
        }
        gkey = kh.h;
        if (graph_replay(ctx, 0, gkey)) n_end = n_begin;   // loop skipped
        else capturing = graph_capture_begin(ctx, 0, gkey);
    }
    if (pairs && n_end - n_begin >= 2) {
        rc = t2_sweep_begin(ctx);
        if (rc) return rc;
    }
    for (int64_t n = n_begin; n < n_end; ++n) {
        if (pairs && n + 1 < n_end) {   // steps n and n+1 in one pass
            PairSpec ps;
            ps.acc = accumulate != 0;
            ps.check1 = fcheck(n);
            ps.check2 = fcheck(n + 1);
            ps.sdt = -dt;
            for (int s = 0; s < ns; ++s) {
                vals[s] = src_amp[(int64_t)spos[s] * N + n];
                vals2[s] = src_amp[(int64_t)spos[s] * N + n + 1];
            }
            ps.n_src = ns;
            ps.src_flat = sidx.data();
            ps.val1 = vals.data();
            ps.val2 = vals2.data();
            ps.sup_mode = gather ? SUP_GATHER : SUP_NONE;
            ps.row1 = n; ps.row2 = n + 1; ps.slot1 = n; ps.slot2 = n + 1;
            rc = launch_pair<T>(ctx, ps);
            if (rc) return rc;
            ++n;
            continue;
        }
        StepSpec sp;
        sp.acc = accumulate != 0;
        sp.check = fcheck(n);
        sp.backward = 0;
        sp.sdt = -dt;
        for (int s = 0; s < ns; ++s) vals[s] = src_amp[(int64_t)spos[s] * N + n];
        const bool in_kernel = ns <= MAX_SRC;
        sp.n_src = in_kernel ? ns : 0;
        sp.src_flat = sidx.data();
        sp.src_val = vals.data();
        sp.sup_mode = gather ? SUP_GATHER : SUP_NONE;
        sp.row = n;
        sp.slot = n;
        if (record) {
            REQUIRE(in_kernel, "history recording supports at most 8 source nodes");
            sp.hist = ctx->hist + (size_t)(n + 1) * ctx->field_bytes();
        }
        if (!in_kernel && sp.check) {
            // stability max must see the injected values: check separately
            sp.check = false;
            rc = launch_step<T>(ctx, sp);
            if (rc) return rc;
            rc = inject_host_list<T>(ctx, ns, sidx.data(), vals.data());
            if (rc) return rc;
            max_abs_kernel<T><<<296, 256, 0, ctx->stream>>>(
                reinterpret_cast<const T*>(ctx->uprev()), ctx->cells(),
                reinterpret_cast<typename FTraits<T>::Bits*>(ctx->maxslots) + n);
            ctx->launches++;
        } else {
            rc = launch_step_part<T>(ctx, sp);
            if (rc) return rc;
            if (!in_kernel) {
                rc = inject_host_list<T>(ctx, ns, sidx.data(), vals.data());
                if (rc) return rc;
            }
        }
        // rotate (u^{n+1} was written over u^{n-1}); a split step rotates
        // after its interior part
        if (ctx->part != 1) std::swap(ctx->cur, ctx->prv);
    }
    if (capturing) {
        rc = graph_capture_end(ctx, 0, gkey, l0, s0, p0);
        if (rc) return rc;
    }
    // split steps and peer-store ranges stay asynchronous (the neighbours'
    // sweeps may not be enqueued yet); wo_check_maxima waits
    if (ctx->part != 0 || (ctx->p2p && !finish)) return WO_OK;
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->prof) harvest_events(ctx);
    if (!finish) return WO_OK;
    std::vector<char> hs((size_t)(N + 2) * 8);
    CK(cudaMemcpy(hs.data(), ctx->maxslots, hs.size(), cudaMemcpyDeviceToHost));
    double peak = 0.0;
    for (int64_t n = 1; n < N; ++n) {
        if (!((n % STABILITY_CHECK_INTERVAL == 0) || (n == N - 1))) continue;
        const double m = slot_value<T>(hs.data(), n);
        if (!std::isfinite(m) || (scale > 0.0 && m > STABILITY_GROWTH_FACTOR * scale)) {
            *fail_step = n + 1;
            *fail_max = m;
            ctx->err = "unstable field";
            return WO_ERR_UNSTABLE;
        }
        peak = std::max(peak, m);
    }
    if (peak_out) *peak_out = peak;
    return WO_OK;
}

// backward steps n = n_hi, n_hi-1, ..., n_lo+1 of an N-step sweep;
// n_hi == N-1 swaps the direction and initialises the check slots
template <typename T>
int sweep_backward_t(wo_ctx* ctx, int64_t N, int64_t src_flat, const double* src_amp,
                     int inject, int accumulate, double dt, int64_t* fail_step,
                     double* fail_max, int64_t n_hi = -1, int64_t n_lo = 0, bool finish = true) {
    if (n_hi < 0) n_hi = N - 1;
    REQUIRE(0 <= n_lo && n_lo <= n_hi && n_hi <= N - 1, "bad backward step range");
    REQUIRE(!inject || ctx->n_sup > 0, "backward support injection without a support");
    REQUIRE(!inject || ctx->store_bytes >= (size_t)N * ctx->n_sup * sizeof(T),
            "adjoint store not populated for this N");
    int rc = WO_OK;
    REQUIRE(ctx->part == 0 || n_hi - n_lo <= 1, "split steps go one step per call");
    if (n_hi == N - 1 && ctx->part != 2) {
        rc = ensure_slots(ctx, N);
        if (rc) return rc;
        CK(cudaMemsetAsync(ctx->maxslots, 0, (size_t)(N + 2) * 8, ctx->stream));
        std::swap(ctx->cur, ctx->prv);  // swap_direction: u_prev <- u^N, u_cur <- u^{N-1}
        rc = p2p_epoch_begin(ctx);
        if (rc) return rc;
    }
    REQUIRE(ctx->maxslot_bytes >= (size_t)(N + 2) * 8, "sweep not initialised");
    long long sf = (long long)src_flat;
    // no source: any negative index on a single domain; on a slab, negative
    // indices down to its lowest ghost plane are ghost-plane sources (the
    // two-step pass recomputes that plane) and WO_NO_SOURCE means none
    const bool has_src = (ctx->has_lo || ctx->has_hi)
                             ? src_flat != WO_NO_SOURCE && src_flat >= -(int64_t)ctx->gl * ctx->plane()
                             : src_flat >= 0;
    double val = 0.0;
    auto bcheck = [](int64_t n) { return (n % STABILITY_CHECK_INTERVAL == 0) || (n == 1); };
    const bool cluster = ctx->part == 0 && !ctx->p2p && n_hi > n_lo && cluster_ready<T>(ctx);
    if (cluster) {
        const double* row = src_amp;
        rc = run_cluster_sweep<T>(ctx, 1, N, n_hi, n_hi - n_lo, has_src ? 1 : 0, &sf, &row,
                                  accumulate != 0, dt, inject ? SUP_INJECT : SUP_NONE);
        if (rc) return rc;
        n_hi = n_lo;
    }
    const bool pairs = pair_ready(ctx);
    REQUIRE(!(ctx->p2p && ctx->t2_oom && ctx->use_two_step),
            "two-step buffers do not fit on this peer-store slab: disable two-step passes on "
            "every slab of the decomposition (wo_prepare_two_step)");
    double val2 = 0.0;
    const bool graphable = ctx->use_graphs && !ctx->prof && ctx->part == 0 && !ctx->p2p &&
                           !cluster && n_hi - n_lo >= 8;
    uint64_t gkey = 0;
    bool capturing = false;
    const int64_t l0 = ctx->launches, s0 = ctx->step_launches, p0 = ctx->pair_launches;
    if (graphable) {
        KeyHash kh;
        kh.val(1); kh.val(N); kh.val(n_hi); kh.val(n_lo); kh.val(inject); kh.val(accumulate);
        kh.val(dt); kh.val(ctx->gen); kh.val(ctx->cur); kh.val(ctx->prv); kh.val(src_flat);
        kh.val((int)sizeof(T));
        hash_param_buffers(kh, ctx);
        if (has_src) kh.bytes(src_amp + n_lo, (size_t)(n_hi - n_lo + 1) * 8);
        gkey = kh.h;
        if (graph_replay(ctx, 1, gkey)) n_hi = n_lo;   // loop skipped
        else capturing = graph_capture_begin(ctx, 1, gkey);
    }
    if (pairs && n_hi - n_lo >= 2) {
        rc = t2_sweep_begin(ctx);
        if (rc) return rc;
    }
    for (int64_t n = n_hi; n > n_lo; --n) {
        if (pairs && n - 1 > n_lo) {   // steps n and n-1 in one pass
            PairSpec ps;
            ps.acc = accumulate != 0;
            ps.check1 = bcheck(n);
            ps.check2 = bcheck(n - 1);
            ps.sdt = dt;
            if (has_src) {
                val = src_amp[n];
                val2 = src_amp[n - 1];
                ps.n_src = 1;
                ps.src_flat = &sf;
                ps.val1 = &val;
                ps.val2 = &val2;
            }
            ps.sup_mode = inject ? SUP_INJECT : SUP_NONE;
            ps.row1 = n; ps.row2 = n - 1; ps.slot1 = n; ps.slot2 = n - 1;
            rc = launch_pair<T>(ctx, ps);
            if (rc) return rc;
            --n;
            continue;
        }
        StepSpec sp;
        sp.acc = accumulate != 0;
        sp.check = bcheck(n);
        sp.backward = 1;
        sp.sdt = dt;
        if (has_src) {
            val = src_amp[n];
            sp.n_src = 1;
            sp.src_flat = &sf;
            sp.src_val = &val;
        }
        sp.sup_mode = inject ? SUP_INJECT : SUP_NONE;
        sp.row = n;
        sp.slot = n;
        rc = launch_step_part<T>(ctx, sp);
        if (rc) return rc;
        if (ctx->part != 1) std::swap(ctx->cur, ctx->prv);
    }
    if (capturing) {
        rc = graph_capture_end(ctx, 1, gkey, l0, s0, p0);
        if (rc) return rc;
    }
    if (ctx->part != 0 || (ctx->p2p && !finish)) return WO_OK;
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->prof) harvest_events(ctx);
    if (!finish) return WO_OK;
    std::vector<char> hs((size_t)(N + 2) * 8);
    CK(cudaMemcpy(hs.data(), ctx->maxslots, hs.size(), cudaMemcpyDeviceToHost));
    for (int64_t n = N - 1; n >= 1; --n) {
        if (!((n % STABILITY_CHECK_INTERVAL == 0) || (n == 1))) continue;
        const double m = slot_value<T>(hs.data(), n);
        if (!std::isfinite(m)) {
            *fail_step = n - 1;
            *fail_max = m;
            ctx->err = "unstable field";
            return WO_ERR_UNSTABLE;
        }
    }
    return WO_OK;
}

// gradient_reference adjoint sweep (gradients.py:371-386): a separate
// 3-level adjoint window from zero end conditions, no source, support
// injection of the UNSCALED adjoint store, mixed increment against the
// recorded forward history.
template <typename T>
int sweep_adjoint_reference_t(wo_ctx* ctx, int64_t N, double dt, int64_t* fail_step,
                              double* fail_max) {
    REQUIRE(ctx->hist_bytes >= (size_t)(N + 1) * ctx->field_bytes(), "no forward history recorded");
    REQUIRE(!ctx->p2p, "the reference engine runs on single-domain contexts");
    REQUIRE(ctx->n_sup > 0 && ctx->store_bytes >= (size_t)N * ctx->n_sup * sizeof(T),
            "adjoint store not populated");
    int rc = ensure(ctx, &ctx->u3, &ctx->u3_bytes, ctx->field_bytes());
    if (rc) return rc;
    rc = ensure_slots(ctx, N);
    if (rc) return rc;
    CK(cudaMemsetAsync(ctx->maxslots, 0, (size_t)(N + 2) * 8, ctx->stream));
    char* lv[3] = {ctx->uprev(), ctx->ucur(), ctx->u3};   // (prev, cur, next)
    for (char* p : lv) CK(cudaMemsetAsync(p, 0, ctx->field_bytes(), ctx->stream));
    // one fused launch per step: stencil + support forces + mixed increment
    RefAdjArgs<T> ra{};
    ra.nd = ctx->ndim;
    ra.n0 = ctx->kn0; ra.n1 = ctx->kn1; ra.n2 = ctx->kn2;
    ra.gamma = reinterpret_cast<const T*>(ctx->base0(ctx->gamma));
    ra.acc = reinterpret_cast<T*>(ctx->acc);
    ra.mat = mat_scalars<T>(ctx);
    ra.cv = (T)ctx->cv; ra.cg = (T)ctx->cg; ra.inv2dt = (T)ctx->inv2dt; ra.inv2dx = (T)ctx->inv2dx;
    ra.sdt = (T)dt;
    ra.sup_mask = ctx->mask;
    ra.sup_prefix = ctx->prefix;
    const size_t C = (size_t)ctx->cells();
    const unsigned blocks = (unsigned)std::min<size_t>((C + 255) / 256, (size_t)ctx->num_sms * 8);
    const T* h = reinterpret_cast<const T*>(ctx->hist);
    for (int64_t n = N - 1; n >= 1; --n) {
        ra.u_prev = reinterpret_cast<const T*>(lv[0]);
        ra.u_cur = reinterpret_cast<const T*>(lv[1]);
        ra.u_out = reinterpret_cast<T*>(lv[2]);
        ra.h_old = h + (n - 1) * C;
        ra.h_mid = h + n * C;
        ra.h_new = h + (n + 1) * C;
        ra.adj_row = reinterpret_cast<const T*>(ctx->store) + n * ctx->n_sup;
        ra.check = (n % STABILITY_CHECK_INTERVAL == 0) || (n == 1);
        ra.max_slot = reinterpret_cast<typename FTraits<T>::Bits*>(ctx->maxslots) + n;
        if (ctx->flavor == RHO_SCALED)
            ref_adjoint_step_kernel<T, RHO_SCALED><<<blocks, 256, 0, ctx->stream>>>(ra);
        else
            ref_adjoint_step_kernel<T, ACOUSTIC><<<blocks, 256, 0, ctx->stream>>>(ra);
        ctx->launches++;
        ctx->step_launches++;
        CK(cudaGetLastError());
        char* t = lv[0];   // rotate: (prev, cur, next) <- (cur, next, prev)
        lv[0] = lv[1];
        lv[1] = lv[2];
        lv[2] = t;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->prof) harvest_events(ctx);
    std::vector<char> hs((size_t)(N + 2) * 8);
    CK(cudaMemcpy(hs.data(), ctx->maxslots, hs.size(), cudaMemcpyDeviceToHost));
    for (int64_t n = N - 1; n >= 1; --n) {
        if (!((n % STABILITY_CHECK_INTERVAL == 0) || (n == 1))) continue;
        const double m = slot_value<T>(hs.data(), n);
        if (!std::isfinite(m)) {
            *fail_step = n - 1;
            *fail_max = m;
            ctx->err = "unstable field";
            return WO_ERR_UNSTABLE;
        }
    }
    return WO_OK;
}

template <typename T>
int step_t(wo_ctx* ctx, int64_t n_force, const int64_t* idx, const double* vals,
           const double* dense, int want_max, double* max_out) {
    REQUIRE(!ctx->p2p, "single steps on a peer-store slab: run sweeps (or clear the peers)");
    int rc = ensure_slots(ctx, 1);
    if (rc) return rc;
    CK(cudaMemsetAsync(ctx->maxslots, 0, 8, ctx->stream));
    std::vector<long long> sidx;
    std::vector<int> spos;
    dedupe_last((int)n_force, idx, sidx, spos);
    std::vector<double> sv(sidx.size());
    for (size_t s = 0; s < sidx.size(); ++s) sv[s] = vals[spos[s]];
    const int ns = (int)sidx.size();
    const bool in_kernel = ns <= MAX_SRC && !dense;
    StepSpec sp;
    sp.check = want_max && in_kernel;
    sp.n_src = in_kernel ? ns : 0;
    sp.src_flat = sidx.data();
    sp.src_val = sv.data();
    sp.slot = 0;
    rc = launch_step<T>(ctx, sp);
    if (rc) return rc;
    if (dense) {
        rc = ensure(ctx, &ctx->f_dense, &ctx->f_dense_cap, (size_t)ctx->cells() * 8);
        if (rc) return rc;
        double* d = ctx->f_dense;
        CK(cudaMemcpyAsync(d, dense, (size_t)ctx->cells() * 8, cudaMemcpyHostToDevice, ctx->stream));
        dense_force_kernel<T><<<592, 256, 0, ctx->stream>>>(
            reinterpret_cast<T*>(ctx->uprev()), reinterpret_cast<const T*>(ctx->base0(ctx->gamma)),
            mat_scalars<T>(ctx), d, ctx->cells());
        ctx->launches++;
        CK(cudaGetLastError());
    }
    if (!in_kernel && ns > 0) {
        rc = inject_host_list<T>(ctx, ns, sidx.data(), sv.data());
        if (rc) return rc;
    }
    if (want_max && !in_kernel) {
        max_abs_kernel<T><<<296, 256, 0, ctx->stream>>>(
            reinterpret_cast<const T*>(ctx->uprev()), ctx->cells(),
            reinterpret_cast<typename FTraits<T>::Bits*>(ctx->maxslots));
        ctx->launches++;
        CK(cudaGetLastError());
    }
    std::swap(ctx->cur, ctx->prv);
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->prof) harvest_events(ctx);
    if (want_max && max_out) {
        char hs[8];
        CK(cudaMemcpy(hs, ctx->maxslots, 8, cudaMemcpyDeviceToHost));
        *max_out = slot_value<T>(hs, 0);
    }
    return WO_OK;
}

template <typename T>
int misfit_t(wo_ctx* ctx, int64_t N, int kind, const double* measured, double c1, double c2,
             double c3, double c4, double adj_coef, int write_adj, double k, double* cost_out) {
    REQUIRE(ctx->n_sup > 0, "shot misfit needs a support");
    REQUIRE(ctx->store_bytes >= (size_t)N * ctx->n_sup * sizeof(T), "no recorded support values");
    int rc;
    if (kind == SHOT_FWI && measured) {
        rc = ensure(ctx, &ctx->measured, &ctx->measured_bytes, (size_t)N * ctx->n_sup * 8);
        if (rc) return rc;
        CK(cudaMemcpyAsync(ctx->measured, measured, (size_t)N * ctx->n_sup * 8,
                           cudaMemcpyHostToDevice, ctx->stream));
    }
    // measured == NULL: reuse the traces uploaded by the previous call
    REQUIRE(kind != SHOT_FWI || ctx->measured_bytes >= (size_t)N * ctx->n_sup * 8,
            "FWI misfit without measured traces");
    rc = ensure(ctx, &ctx->partial, &ctx->partial_bytes, (size_t)N * 8 + 8);
    if (rc) return rc;
    if (!ctx->cost) {
        rc = dev_alloc(ctx, (void**)&ctx->cost, 8);
        if (rc) return rc;
    }
    misfit_kernel<T><<<(unsigned)N, 256, 0, ctx->stream>>>(
        reinterpret_cast<T*>(ctx->store), ctx->measured, (long long)N, (int)ctx->n_sup, kind, c1,
        c2, c3, c4, adj_coef, write_adj, (T)k, ctx->partial);
    cost_sum_kernel<<<1, 256, 0, ctx->stream>>>(ctx->partial, (long long)N, ctx->cost);
    ctx->launches += 2;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(cost_out, ctx->cost, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return WO_OK;
}

// Device field -> caller's (pageable) host array through a persistent pinned
// double buffer: the D2H of chunk i+1 overlaps the host copy of chunk i
// (a plain pageable cudaMemcpy of a 67 MB field ran at ~4.6 GB/s).
constexpr size_t HSTAGE_HALF = 8u << 20;

int download_field(wo_ctx* ctx, void* out, const char* dev, size_t bytes) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, out) == cudaSuccess && pa.type == cudaMemoryTypeHost) {
        // page-locked destination: one DMA, no staging
        CK(cudaMemcpyAsync(out, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        return WO_OK;
    }
    (void)cudaGetLastError();
    if (!ctx->hstage) {
        CK(cudaHostAlloc((void**)&ctx->hstage, 2 * HSTAGE_HALF, cudaHostAllocDefault));
        for (auto& e : ctx->hev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    char* dst = static_cast<char*>(out);
    size_t prev_off = 0, prev_n = 0;
    int half = 0;
    for (size_t off = 0; off < bytes || prev_n; off += HSTAGE_HALF, half ^= 1) {
        const size_t n = off < bytes ? std::min(HSTAGE_HALF, bytes - off) : 0;
        if (n) {
            CK(cudaMemcpyAsync(ctx->hstage + half * HSTAGE_HALF, dev + off, n,
                               cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaEventRecord(ctx->hev[half], ctx->stream));
        }
        if (prev_n) {
            CK(cudaEventSynchronize(ctx->hev[half ^ 1]));
            // fresh destination pages fault on first touch: copy with a few
            // threads so the faults (not the bandwidth) overlap
            const char* src = ctx->hstage + (half ^ 1) * HSTAGE_HALF;
            constexpr int NT = 4;
            const size_t part = (prev_n / NT + 63) & ~size_t(63);
            std::thread th[NT - 1];
            for (int t = 1; t < NT; ++t) {
                const size_t b = std::min(prev_n, t * part), e = std::min(prev_n, (t + 1) * part);
                th[t - 1] = std::thread([=] { if (e > b) std::memcpy(dst + prev_off + b, src + b, e - b); });
            }
            std::memcpy(dst + prev_off, src, std::min(prev_n, part));
            for (auto& t : th) t.join();
        }
        prev_off = off;
        prev_n = n;
    }
    return WO_OK;
}

template <typename T>
int gradient_t(wo_ctx* ctx, double two_k, void* out) {
    scale_div_kernel<T><<<592, 256, 0, ctx->stream>>>(reinterpret_cast<T*>(ctx->acc), ctx->cells(),
                                                      (T)two_k);
    ctx->launches++;
    CK(cudaGetLastError());
    if (out) return download_field(ctx, out, ctx->acc, ctx->field_bytes());
    CK(cudaStreamSynchronize(ctx->stream));
    return WO_OK;
}

// gamma.astype(T) (solver.py:94,100) on the device: fp64 host data goes up
// through a fixed double-buffered staging area and is cast by a kernel, so
// the host never loops over the field and big grids need no fp64 twin.
template <typename T>
__global__ void cast_kernel(const double* src, T* dst, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        dst[i] = (T)src[i];
}

template <typename T>
int upload_cast_t(wo_ctx* ctx, const double* host, char* dev, int64_t n) {
    const int64_t chunk = 4 << 20;  // doubles per staging half (32 MiB)
    // persistent staging buffer: a per-call cudaMalloc/cudaFree pair stalls
    // the host for up to ~0.5 s on a busy device
    int rc = ensure(ctx, &ctx->stage, &ctx->stage_bytes, (size_t)std::min(n, 2 * chunk) * 8);
    if (rc) return rc;
    double* stage = reinterpret_cast<double*>(ctx->stage);
    int half = 0;  // stream order keeps a half busy until its cast kernel ran
    for (int64_t off = 0; off < n; off += chunk, half ^= 1) {
        const int64_t m = std::min(chunk, n - off);
        double* s = stage + (size_t)half * chunk;
        CK(cudaMemcpyAsync(s, host + off, (size_t)m * 8, cudaMemcpyHostToDevice, ctx->stream));
        cast_kernel<T><<<296, 256, 0, ctx->stream>>>(s, reinterpret_cast<T*>(dev) + off, m);
        ctx->launches++;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return WO_OK;
}

int create_common(wo_ctx* ctx) {
    // plane offsets are 64-bit in the single-step kernels and in the
    // two-step kernel's T2_FULL level (chosen for allocations of >= 2^31
    // cells); in-plane offsets and plane indices stay 32-bit (n1*n2 < 2^31)
    REQUIRE(ctx->plane() < (1ll << 31), "plane too large (n1*n2 >= 2^31 cells)");
    CK(cudaSetDevice(ctx->device));
    CK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    const size_t ab = (size_t)ctx->alloc_cells() * ctx->itemsize;
    int rc;
    if ((rc = dev_alloc(ctx, (void**)&ctx->gamma, ab))) return rc;
    if ((rc = dev_alloc(ctx, (void**)&ctx->u[0], ab))) return rc;
    if ((rc = dev_alloc(ctx, (void**)&ctx->u[1], ab))) return rc;
    if ((rc = dev_alloc(ctx, (void**)&ctx->acc, ctx->field_bytes()))) return rc;
    CK(cudaMemsetAsync(ctx->u[0], 0, ab, ctx->stream));
    CK(cudaMemsetAsync(ctx->u[1], 0, ab, ctx->stream));
    CK(cudaMemsetAsync(ctx->acc, 0, ctx->field_bytes(), ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return WO_OK;
}

}  // namespace

#define DISPATCH(ctx, FN, ...) \
    ((ctx)->itemsize == 4 ? FN<float>(__VA_ARGS__) : FN<double>(__VA_ARGS__))

// Decide the division path of the step kernel for the current material
// (fastdiv.cuh): branch-free sequences only if every derived coefficient is
// bit-identical to the IEEE intrinsic, checked over the whole allocation
// (ghost planes included).
template <typename T>
static int verify_fast_div_t(wo_ctx* ctx) {
    const bool before = ctx->fast_div;   // selects the kernel variant (sweep graphs)
    ctx->fast_div = false;
    if (!ctx->allow_fast_div) {
        if (before) ++ctx->gen;
        return WO_OK;
    }
    int rc = ensure(ctx, &ctx->flag, &ctx->flag_bytes, sizeof(int));
    if (rc) return rc;
    int* d_ok = reinterpret_cast<int*>(ctx->flag);
    const int one = 1;
    CK(cudaMemcpyAsync(d_ok, &one, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    const int n0 = ctx->alloc_planes();
    const T* g = reinterpret_cast<const T*>(ctx->gamma);
    if (ctx->flavor == RHO_SCALED)
        verify_material_kernel<T, RHO_SCALED><<<592, 256, 0, ctx->stream>>>(
            g, n0, ctx->kn1, ctx->kn2, mat_scalars<T>(ctx), d_ok);
    else
        verify_material_kernel<T, ACOUSTIC><<<592, 256, 0, ctx->stream>>>(
            g, n0, ctx->kn1, ctx->kn2, mat_scalars<T>(ctx), d_ok);
    ctx->launches++;
    int ok = 0;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->fast_div = ok != 0;
    if (ctx->fast_div != before) ++ctx->gen;
    return WO_OK;
}

static int verify_fast_div(wo_ctx* ctx) { return DISPATCH(ctx, verify_fast_div_t, ctx); }

extern "C" {

int wo_version(void) { return 100; }

int wo_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

const char* wo_last_error(const wo_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

int wo_create(wo_ctx** out, int ndim, const int64_t* shape, double dx, int itemsize, int device) {
    *out = nullptr;
    if (ndim < 1 || ndim > 3 || (itemsize != 4 && itemsize != 8) || !(dx > 0)) {
        g_create_error = "invalid grid / dtype";
        return WO_ERR_CONFIG;
    }
    for (int a = 0; a < ndim; ++a)
        if (shape[a] < 3 || shape[a] > (1ll << 30)) {
            g_create_error = "every axis needs at least 3 nodes";
            return WO_ERR_CONFIG;
        }
    wo_ctx* ctx = new wo_ctx();
    ctx->device = device;
    ctx->ndim = ndim;
    ctx->itemsize = itemsize;
    ctx->dx = dx;
    for (int a = 0; a < ndim; ++a) ctx->shape[a] = shape[a];
    if (ndim == 3) { ctx->kn0 = (int)shape[0]; ctx->kn1 = (int)shape[1]; ctx->kn2 = (int)shape[2]; }
    else if (ndim == 2) { ctx->kn0 = 1; ctx->kn1 = (int)shape[0]; ctx->kn2 = (int)shape[1]; }
    else { ctx->kn0 = 1; ctx->kn1 = 1; ctx->kn2 = (int)shape[0]; }
    ctx->n0g = ctx->kn0;
    int rc = create_common(ctx);
    if (rc) {
        g_create_error = ctx->err;
        wo_destroy(ctx);
        return rc;
    }
    *out = ctx;
    return WO_OK;
}

int wo_create_slab(wo_ctx** out, const int64_t* gshape, int64_t i_begin, int64_t i_end, double dx,
                   int itemsize, int device) {
    *out = nullptr;
    if (!(0 <= i_begin && i_begin < i_end && i_end <= gshape[0]) || gshape[0] < 3 ||
        gshape[1] < 3 || gshape[2] < 3 || (itemsize != 4 && itemsize != 8)) {
        g_create_error = "invalid slab";
        return WO_ERR_CONFIG;
    }
    wo_ctx* ctx = new wo_ctx();
    ctx->device = device;
    ctx->ndim = 3;
    ctx->itemsize = itemsize;
    ctx->dx = dx;
    ctx->shape[0] = i_end - i_begin;
    ctx->shape[1] = gshape[1];
    ctx->shape[2] = gshape[2];
    ctx->kn0 = (int)(i_end - i_begin);
    ctx->kn1 = (int)gshape[1];
    ctx->kn2 = (int)gshape[2];
    ctx->i_off = (int)i_begin;
    ctx->n0g = (int)gshape[0];
    ctx->has_lo = i_begin > 0;
    ctx->has_hi = i_end < gshape[0];
    // two ghost planes per neighbour (the two-step pass recomputes one plane
    // beyond the slab and reads one more); one where the global end is closer
    ctx->gl = (int)std::min<int64_t>(2, i_begin);
    ctx->gh = (int)std::min<int64_t>(2, gshape[0] - i_end);
    // two-step passes on slabs only when the caller enables them for every
    // slab of the decomposition (all slabs must take the same launches)
    ctx->use_two_step = 0;
    int rc = create_common(ctx);
    if (rc) {
        g_create_error = ctx->err;
        wo_destroy(ctx);
        return rc;
    }
    *out = ctx;
    return WO_OK;
}

void wo_destroy(wo_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    void* bufs[] = {ctx->gamma, ctx->u[0], ctx->u[1], ctx->u[2], ctx->u[3], ctx->mat4, ctx->stage,
                    ctx->snap, ctx->scratch, ctx->opt, ctx->opt_frozen, ctx->opt_partial,
                    ctx->dsn, ctx->dmask, ctx->dfp_off, ctx->dfp_w,
                    ctx->flag, ctx->acc, reinterpret_cast<char*>(ctx->in_flags),
                    ctx->mask, ctx->prefix, reinterpret_cast<char*>(ctx->sup_flat), ctx->sup_fc,
                    ctx->store, ctx->measured, ctx->partial, ctx->cost, ctx->maxslots,
                    ctx->f_idx, ctx->f_vals, ctx->f_dense, ctx->hist, ctx->u3,
                    reinterpret_cast<char*>(ctx->amp_dev), reinterpret_cast<char*>(ctx->tflags)};
    for (auto& m : ctx->ipc_maps) cudaIpcCloseMemHandle(m.second);
    for (void* b : bufs)
        if (b) cudaFree(b);
    for (auto e : ctx->marks)
        if (e) cudaEventDestroy(e);
    for (auto e : ctx->hev)
        if (e) cudaEventDestroy(e);
    for (auto& g : ctx->graph)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    if (ctx->hstage) cudaFreeHost(ctx->hstage);
    for (auto e : ctx->ev_free) cudaEventDestroy(e);
    for (auto e : ctx->ev_used) cudaEventDestroy(e);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int wo_set_material(wo_ctx* ctx, int flavor, const double* gamma, double rho0, double rho1,
                    double kappa1, double rho2, double kappa2, double dt, double ratio2) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(flavor == WO_RHO_SCALED || flavor == WO_ACOUSTIC, "unknown material flavor");
    // the scalars enter kernel parameters (sweep graphs); gamma is data
    const bool same = ctx->material_set && ctx->flavor == flavor && ctx->rho0 == rho0 &&
                      ctx->rho1 == rho1 && ctx->kappa1 == kappa1 && ctx->rho2 == rho2 &&
                      ctx->kappa2 == kappa2 && ctx->dt_mat == dt && ctx->ratio2 == ratio2;
    if (!same) ++ctx->gen;
    ctx->flavor = flavor;
    ctx->rho0 = rho0; ctx->rho1 = rho1; ctx->kappa1 = kappa1;
    ctx->rho2 = rho2; ctx->kappa2 = kappa2; ctx->dt_mat = dt; ctx->ratio2 = ratio2;
    // gamma.astype(T) (solver.py:94/100): fp64 staged up and cast on the device
    const int64_t n = ctx->alloc_cells();
    if (ctx->itemsize == 4) {
        rc = upload_cast_t<float>(ctx, gamma, ctx->gamma, n);
        if (rc) return rc;
    } else {
        CK(cudaMemcpyAsync(ctx->gamma, gamma, n * 8, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    ctx->material_set = true;
    ctx->mat4_valid = false;
    ctx->sup_fc_valid = false;
    return verify_fast_div(ctx);
}

int wo_opt_init(wo_ctx* ctx, const double* params, const unsigned char* frozen, int zero_frozen_grad,
                double lo, double hi, double frozen_value, double alpha, double beta1,
                double beta2, double eps) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(!ctx->has_lo && !ctx->has_hi, "the device optimiser runs on single-domain contexts");
    REQUIRE(lo < hi, "need lo < hi");
    const int64_t n = ctx->cells();
    if (!ctx->opt) {
        if ((rc = dev_alloc(ctx, (void**)&ctx->opt, (size_t)n * 24))) return rc;
        if ((rc = dev_alloc(ctx, (void**)&ctx->opt_frozen, (size_t)n))) return rc;
        if ((rc = dev_alloc(ctx, (void**)&ctx->opt_partial, 592 * 8))) return rc;
    }
    CK(cudaMemcpyAsync(ctx->opt, params, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->opt + n, 0, (size_t)n * 16, ctx->stream));   // m = v = 0
    if (frozen)
        CK(cudaMemcpyAsync(ctx->opt_frozen, frozen, (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
    else
        CK(cudaMemsetAsync(ctx->opt_frozen, 0, (size_t)n, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->opt_zero_frozen = zero_frozen_grad;
    ctx->design_active = 0;
    ctx->adam = AdamScalars{beta1, beta2, 1.0 - beta1, 1.0 - beta2, 1.0, 1.0, alpha, eps, lo, hi,
                            frozen_value};
    return WO_OK;
}

int wo_opt_step(wo_ctx* ctx, int t, double* grad_norm) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->opt && ctx->material_set, "wo_opt_init / material missing");
    REQUIRE(t >= 1, "Adam step count starts at 1");
    AdamScalars s = ctx->adam;
    s.bc1 = 1.0 - std::pow(s.beta1, (double)t);   // Python float ** int, then 1 - x
    s.bc2 = 1.0 - std::pow(s.beta2, (double)t);
    const int64_t n = ctx->cells();
    char* g = ctx->base0(ctx->gamma);
    double* m = ctx->opt + n;
    double* v = ctx->opt + 2 * n;
    if (ctx->design_active)   // TATO: chain-rule gradient, the material comes from g_bar
        adam_clip_kernel<double, double><<<592, 256, 0, ctx->stream>>>(
            ctx->dsn + 2 * n, ctx->opt, m, v, ctx->opt_frozen, ctx->opt_zero_frozen, s, n,
            (double*)nullptr, ctx->opt_partial);
    else if (ctx->itemsize == 4)
        adam_clip_kernel<float, float><<<592, 256, 0, ctx->stream>>>(
            reinterpret_cast<const float*>(ctx->acc), ctx->opt, m, v, ctx->opt_frozen,
            ctx->opt_zero_frozen, s, n, reinterpret_cast<float*>(g), ctx->opt_partial);
    else
        adam_clip_kernel<double, double><<<592, 256, 0, ctx->stream>>>(
            reinterpret_cast<const double*>(ctx->acc), ctx->opt, m, v, ctx->opt_frozen,
            ctx->opt_zero_frozen, s, n, reinterpret_cast<double*>(g), ctx->opt_partial);
    ctx->launches++;
    CK(cudaGetLastError());
    double part[592];
    CK(cudaMemcpyAsync(part, ctx->opt_partial, sizeof(part), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    double sq = 0.0;
    for (double x : part) sq += x;
    if (grad_norm) *grad_norm = std::sqrt(sq);
    if (ctx->design_active) return WO_OK;   // the material changes in wo_design_material
    ctx->mat4_valid = false;                // gamma changed on the device
    ctx->sup_fc_valid = false;
    return verify_fast_div(ctx);
}

int wo_design_setup(wo_ctx* ctx, const unsigned char* mask, int n_fp, const int* offsets,
                    const double* weights) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(!ctx->has_lo && !ctx->has_hi, "the design loop runs on single-domain contexts");
    REQUIRE(n_fp >= 1, "empty filter footprint");
    const int64_t n = ctx->cells();
    if (!ctx->dsn && (rc = dev_alloc(ctx, (void**)&ctx->dsn, (size_t)n * 48))) return rc;
    if (mask) {
        if (!ctx->dmask && (rc = dev_alloc(ctx, (void**)&ctx->dmask, (size_t)n))) return rc;
        CK(cudaMemcpyAsync(ctx->dmask, mask, (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
    } else if (ctx->dmask) {
        cudaFree(ctx->dmask);
        ctx->dev_bytes -= n;
        ctx->dmask = nullptr;
    }
    std::vector<int> o3((size_t)n_fp * 3, 0);   // footprint offsets in kernel space
    for (int f = 0; f < n_fp; ++f)
        for (int a = 0; a < ctx->ndim; ++a)
            o3[(size_t)f * 3 + (3 - ctx->ndim) + a] = offsets[(size_t)f * ctx->ndim + a];
    if (ctx->dfp_off) { cudaFree(ctx->dfp_off); ctx->dfp_off = nullptr; }
    if (ctx->dfp_w) { cudaFree(ctx->dfp_w); ctx->dfp_w = nullptr; }
    ctx->dev_bytes -= (int64_t)ctx->dfp_n * (12 + 8);
    if ((rc = dev_alloc(ctx, (void**)&ctx->dfp_off, o3.size() * sizeof(int)))) return rc;
    if ((rc = dev_alloc(ctx, (void**)&ctx->dfp_w, (size_t)n_fp * 8))) return rc;
    CK(cudaMemcpyAsync(ctx->dfp_off, o3.data(), o3.size() * sizeof(int), cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemcpyAsync(ctx->dfp_w, weights, (size_t)n_fp * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->dfp_n = n_fp;
    ctx->design_active = 1;
    return WO_OK;
}

int wo_design_material(wo_ctx* ctx, double beta, double eta, double t_be, double denom) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->opt && ctx->dsn && ctx->material_set, "wo_opt_init / wo_design_setup missing");
    const int64_t n = ctx->cells();
    double *gt = ctx->dsn, *gb = ctx->dsn + n, *t1 = ctx->dsn + 3 * n, *t2 = ctx->dsn + 4 * n;
    const Footprint fp{ctx->dfp_n, ctx->dfp_off, ctx->dfp_w};
    // g_tilde = density_filter(gamma_raw), g_bar = heaviside_project(g_tilde)
    masked_correlate_kernel<<<592, 256, 0, ctx->stream>>>(ctx->kn0, ctx->kn1, ctx->kn2, ctx->opt,
                                                          ctx->dmask, 1, fp, t1, t2);
    filter_finish_kernel<<<592, 256, 0, ctx->stream>>>(n, ctx->opt, ctx->dmask, t1, t2, gt);
    heaviside_kernel<<<592, 256, 0, ctx->stream>>>(n, gt, beta, eta, t_be, denom, ctx->dmask, gb);
    // the material is g_bar.astype(T) (TatoProblem.material, solver.py:100)
    char* g = ctx->base0(ctx->gamma);
    if (ctx->itemsize == 4)
        cast_kernel<float><<<296, 256, 0, ctx->stream>>>(gb, reinterpret_cast<float*>(g), n);
    else
        cast_kernel<double><<<296, 256, 0, ctx->stream>>>(gb, reinterpret_cast<double*>(g), n);
    ctx->launches += 4;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->mat4_valid = false;
    ctx->sup_fc_valid = false;
    return verify_fast_div(ctx);
}

int wo_design_gradient(wo_ctx* ctx, double beta, double eta, double denom) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->dsn, "wo_design_setup missing");
    const int64_t n = ctx->cells();
    double *gt = ctx->dsn, *gr = ctx->dsn + 2 * n;
    double *t1 = ctx->dsn + 3 * n, *t2 = ctx->dsn + 4 * n, *t3 = ctx->dsn + 5 * n;
    const Footprint fp{ctx->dfp_n, ctx->dfp_off, ctx->dfp_w};
    // chain_rule(double(dC/dg_bar), g_tilde, ...) (tato.py:124-140)
    if (ctx->itemsize == 4)
        widen_kernel<float><<<592, 256, 0, ctx->stream>>>(reinterpret_cast<const float*>(ctx->acc),
                                                         gr, n);
    else
        widen_kernel<double><<<592, 256, 0, ctx->stream>>>(
            reinterpret_cast<const double*>(ctx->acc), gr, n);
    chain_inner_kernel<<<592, 256, 0, ctx->stream>>>(n, gr, gt, beta, eta, denom, ctx->dmask, t1);
    masked_correlate_kernel<<<592, 256, 0, ctx->stream>>>(ctx->kn0, ctx->kn1, ctx->kn2, t1,
                                                          ctx->dmask, 1, fp, nullptr, t2);
    chain_ratio_kernel<<<592, 256, 0, ctx->stream>>>(n, t1, t2, ctx->dmask, t3);
    masked_correlate_kernel<<<592, 256, 0, ctx->stream>>>(ctx->kn0, ctx->kn1, ctx->kn2, t3,
                                                          nullptr, 0, fp, gr, nullptr);
    mask_zero_kernel<<<592, 256, 0, ctx->stream>>>(n, ctx->dmask, gr);
    ctx->launches += 6;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    return WO_OK;
}

int wo_design_get(wo_ctx* ctx, int which, double* out) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->dsn && which >= 0 && which <= 2, "wo_design_setup missing / bad field");
    return download_field(ctx, out, reinterpret_cast<const char*>(ctx->dsn + which * ctx->cells()),
                          (size_t)ctx->cells() * 8);
}

int wo_opt_get(wo_ctx* ctx, double* params) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->opt, "wo_opt_init missing");
    return download_field(ctx, params, reinterpret_cast<const char*>(ctx->opt),
                          (size_t)ctx->cells() * 8);
}

int wo_set_option(wo_ctx* ctx, int option, int value) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    ++ctx->gen;
    REQUIRE(option == WO_OPT_FAST_DIV || option == WO_OPT_PAIR_KERNEL ||
                option == WO_OPT_TMA_KERNEL || option == WO_OPT_TWO_STEP ||
                option == WO_OPT_PLANE_PART || option == WO_OPT_GRAPHS ||
                option == WO_OPT_CLUSTER,
            "unknown option");
    if (option == WO_OPT_CLUSTER) {
        ctx->use_cluster = value == 2 ? 2 : value != 0;
        ctx->cl_state = 0;   // probe again on the next sweep
        ctx->cr_state = 0;
        return WO_OK;
    }
    if (option == WO_OPT_GRAPHS) {
        ctx->use_graphs = value != 0;
        return WO_OK;
    }
    if (option == WO_OPT_PLANE_PART) {
        REQUIRE(value >= 0 && value <= 2, "plane part is 0, 1 or 2");
        ctx->part = value;
        return WO_OK;
    }
    if (option == WO_OPT_TWO_STEP) {
        ctx->use_two_step = value;   // 0 off, 1 (2: same) fp32 and fp64 grids
        return WO_OK;
    }
    if (option == WO_OPT_PAIR_KERNEL) {
        ctx->use_pair = value != 0;
        return WO_OK;
    }
    if (option == WO_OPT_TMA_KERNEL) {
        ctx->use_tma = value != 0;   // 0 off, else the TMA kernels (default)
        return WO_OK;
    }
    ctx->allow_fast_div = value != 0;
    if (ctx->material_set) return verify_fast_div(ctx);
    ctx->fast_div = false;
    return WO_OK;
}

int wo_fast_div_active(const wo_ctx* ctx) { return ctx && ctx->fast_div ? 1 : 0;
    return WO_OK;
}

int wo_set_kernel_coefficients(wo_ctx* ctx, double cv, double cg, double inv2dt, double inv2dx) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    ctx->cv = cv; ctx->cg = cg; ctx->inv2dt = inv2dt; ctx->inv2dx = inv2dx;
    ++ctx->gen;
    return WO_OK;
}

int wo_set_support(wo_ctx* ctx, int64_t n_sup, const int64_t* flat) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    const int64_t C = ctx->cells();
    for (int64_t s = 0; s < n_sup; ++s) {
        REQUIRE(flat[s] >= 0 && flat[s] < C, "support index outside the grid");
        REQUIRE(s == 0 || flat[s] > flat[s - 1], "support indices must be strictly increasing");
    }
    const int64_t words = (C + 31) / 32;
    if (!ctx->mask) {
        if ((rc = dev_alloc(ctx, (void**)&ctx->mask, words * 4))) return rc;
        if ((rc = dev_alloc(ctx, (void**)&ctx->prefix, words * 4))) return rc;
    }
    std::vector<unsigned int> m(words, 0u);
    std::vector<int> p(words, 0);
    for (int64_t s = 0; s < n_sup; ++s) m[flat[s] >> 5] |= 1u << (flat[s] & 31);
    ctx->sup_lo = n_sup ? (int)(flat[0] / ctx->plane()) : 0;
    ctx->sup_hi = n_sup ? (int)(flat[n_sup - 1] / ctx->plane()) : -1;
    int run = 0;
    for (int64_t w = 0; w < words; ++w) {
        p[w] = run;
        run += __builtin_popcount(m[w]);
    }
    CK(cudaMemcpy(ctx->mask, m.data(), words * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->prefix, p.data(), words * 4, cudaMemcpyHostToDevice));
    if (n_sup) {
        if ((rc = ensure(ctx, &ctx->sup_flat, &ctx->sup_flat_bytes, (size_t)n_sup * 8))) return rc;
        static_assert(sizeof(long long) == sizeof(int64_t), "support index width");
        CK(cudaMemcpy(ctx->sup_flat, flat, (size_t)n_sup * 8, cudaMemcpyHostToDevice));
    }
    ctx->sup_fc_valid = false;
    ctx->n_sup = n_sup;
    ++ctx->gen;
    return WO_OK;
}

int wo_reset_window(wo_ctx* ctx) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    const size_t ab = (size_t)ctx->alloc_cells() * ctx->itemsize;
    // both levels are zeroed: restart the rotation at buffers (0, 1), so a
    // repeated evaluation repeats its launch sequence exactly (sweep graphs)
    ctx->cur = 0;
    ctx->prv = 1;
    CK(cudaMemsetAsync(ctx->u[ctx->cur], 0, ab, ctx->stream));
    CK(cudaMemsetAsync(ctx->u[ctx->prv], 0, ab, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return WO_OK;
}

int wo_set_window(wo_ctx* ctx, const void* u_prev, const void* u_cur) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    CK(cudaMemcpy(ctx->uprev(), u_prev, ctx->field_bytes(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->ucur(), u_cur, ctx->field_bytes(), cudaMemcpyHostToDevice));
    return WO_OK;
}

int wo_get_window(wo_ctx* ctx, void* u_prev, void* u_cur) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    if (u_prev) CK(cudaMemcpy(u_prev, ctx->uprev(), ctx->field_bytes(), cudaMemcpyDeviceToHost));
    if (u_cur) CK(cudaMemcpy(u_cur, ctx->ucur(), ctx->field_bytes(), cudaMemcpyDeviceToHost));
    return WO_OK;
}

int wo_snapshot(wo_ctx* ctx, int op, int64_t n_steps) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(op == WO_SNAP_SAVE || op == WO_SNAP_RESTORE || op == WO_SNAP_FREE, "unknown snapshot op");
    if (op == WO_SNAP_FREE) {
        if (ctx->snap) {
            CK(cudaStreamSynchronize(ctx->stream));
            cudaFree(ctx->snap);
            ctx->dev_bytes -= (int64_t)ctx->snap_bytes;
        }
        ctx->snap = nullptr;
        ctx->snap_bytes = 0;
        ctx->snap_store = -1;
        return WO_OK;
    }
    const size_t ab = (size_t)ctx->alloc_cells() * ctx->itemsize, fb = ctx->field_bytes();
    const size_t sb = (size_t)std::max<int64_t>(n_steps, 0) * ctx->n_sup * ctx->itemsize;
    if (op == WO_SNAP_SAVE) {
        REQUIRE(sb <= ctx->store_bytes, "support store smaller than n_steps rows");
        rc = ensure(ctx, &ctx->snap, &ctx->snap_bytes, 2 * ab + fb + sb);
        if (rc) return rc;
        CK(cudaMemcpyAsync(ctx->snap, ctx->u[ctx->prv], ab, cudaMemcpyDeviceToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->snap + ab, ctx->u[ctx->cur], ab, cudaMemcpyDeviceToDevice,
                           ctx->stream));
        CK(cudaMemcpyAsync(ctx->snap + 2 * ab, ctx->acc, fb, cudaMemcpyDeviceToDevice, ctx->stream));
        if (sb)
            CK(cudaMemcpyAsync(ctx->snap + 2 * ab + fb, ctx->store, sb, cudaMemcpyDeviceToDevice,
                               ctx->stream));
        ctx->snap_store = (int64_t)sb;
    } else {
        REQUIRE(ctx->snap && ctx->snap_store == (int64_t)sb, "no snapshot for this step count");
        CK(cudaMemcpyAsync(ctx->u[ctx->prv], ctx->snap, ab, cudaMemcpyDeviceToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->u[ctx->cur], ctx->snap + ab, ab, cudaMemcpyDeviceToDevice,
                           ctx->stream));
        CK(cudaMemcpyAsync(ctx->acc, ctx->snap + 2 * ab, fb, cudaMemcpyDeviceToDevice, ctx->stream));
        if (sb)
            CK(cudaMemcpyAsync(ctx->store, ctx->snap + 2 * ab + fb, sb, cudaMemcpyDeviceToDevice,
                               ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return WO_OK;
}

int wo_swap_direction(wo_ctx* ctx) {
    if (!ctx) return WO_ERR_CONFIG;
    std::swap(ctx->cur, ctx->prv);
    return WO_OK;
}

int wo_zero_accumulator(wo_ctx* ctx) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    CK(cudaMemsetAsync(ctx->acc, 0, ctx->field_bytes(), ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return WO_OK;
}

int wo_get_accumulator(wo_ctx* ctx, void* out) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    return download_field(ctx, out, ctx->acc, ctx->field_bytes());
}

int wo_set_accumulator(wo_ctx* ctx, const void* in) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    CK(cudaMemcpy(ctx->acc, in, ctx->field_bytes(), cudaMemcpyHostToDevice));
    return WO_OK;
}

int wo_sweep_forward(wo_ctx* ctx, int64_t n_steps, int n_src, const int64_t* src_flat,
                     const double* src_amp, int flags, double dt, double scale,
                     double* peak_out, int64_t* fail_step, double* fail_max) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->material_set, "material not set");
    REQUIRE(n_steps >= 2, "need at least 2 time steps");
    return DISPATCH(ctx, sweep_forward_t, ctx, n_steps, n_src, src_flat, src_amp, flags, dt,
                    scale, peak_out, fail_step, fail_max);
}

int wo_sweep_forward_range(wo_ctx* ctx, int64_t n_steps, int64_t n_begin, int64_t n_end,
                           int n_src, const int64_t* src_flat, const double* src_amp, int flags,
                           double dt) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->material_set, "material not set");
    REQUIRE(n_steps >= 2, "need at least 2 time steps");
    int64_t fs = 0;
    double fm = 0.0;
    return DISPATCH(ctx, sweep_forward_t, ctx, n_steps, n_src, src_flat, src_amp, flags, dt, 0.0,
                    nullptr, &fs, &fm, n_begin, n_end, false);
}

int wo_sweep_backward_range(wo_ctx* ctx, int64_t n_steps, int64_t n_hi, int64_t n_lo,
                            int64_t src_flat, const double* src_amp, int inject_support,
                            int accumulate, double dt) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->material_set, "material not set");
    int64_t fs = 0;
    double fm = 0.0;
    return DISPATCH(ctx, sweep_backward_t, ctx, n_steps, src_flat, src_amp, inject_support,
                    accumulate, dt, &fs, &fm, n_hi, n_lo, false);
}

int wo_check_maxima(wo_ctx* ctx, int64_t n_steps, double* out) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->maxslot_bytes >= (size_t)(n_steps + 2) * 8, "no sweep recorded");
    CK(cudaStreamSynchronize(ctx->stream));
    std::vector<char> hs((size_t)(n_steps + 2) * 8);
    CK(cudaMemcpy(hs.data(), ctx->maxslots, hs.size(), cudaMemcpyDeviceToHost));
    for (int64_t n = 0; n < n_steps + 2; ++n)
        out[n] = ctx->itemsize == 4 ? slot_value<float>(hs.data(), n)
                                    : slot_value<double>(hs.data(), n);
    return WO_OK;
}

int wo_halo_planes(wo_ctx* ctx, void** first, void** last, void** ghost_lo, void** ghost_hi,
                   int64_t* plane_bytes) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    const size_t pb = (size_t)ctx->plane() * ctx->itemsize;
    char* c = ctx->ucur();
    *first = c;
    *last = c + (size_t)(ctx->kn0 - 1) * pb;
    *ghost_lo = ctx->has_lo ? c - pb : nullptr;
    *ghost_hi = ctx->has_hi ? c + (size_t)ctx->kn0 * pb : nullptr;
    *plane_bytes = (int64_t)pb;
    return WO_OK;
}

static int ensure_flags(wo_ctx* ctx) {
    if (ctx->in_flags) return WO_OK;
    int rc = dev_alloc(ctx, (void**)&ctx->in_flags, 4 * sizeof(unsigned int));
    if (rc) return rc;
    // on the context's stream, complete before any neighbour can see the address
    CK(cudaMemsetAsync(ctx->in_flags, 0, 4 * sizeof(unsigned int), ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return WO_OK;
}

int wo_slab_ghosts(wo_ctx* ctx, void** ghost_lo, void** ghost_hi, void** flags) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->has_lo || ctx->has_hi, "not a slab context");
    // all four level buffers exist from here on: their ghost planes are what
    // the neighbours store into, whichever buffers a launch writes
    if ((rc = ensure_four(ctx))) return rc;
    if ((rc = ensure_flags(ctx))) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    const size_t pb = (size_t)ctx->plane() * ctx->itemsize;
    for (int b = 0; b < 4; ++b) {
        char* u = ctx->base0(ctx->u[b]);
        ghost_lo[b] = ctx->has_lo ? u - (size_t)ctx->gl * pb : nullptr;   // plane -gl
        ghost_hi[b] = ctx->has_hi ? u + (size_t)ctx->kn0 * pb : nullptr;   // plane n0
    }
    flags[0] = ctx->in_flags;       // bumped by the lower neighbour (+2: odd epochs)
    flags[1] = ctx->in_flags + 1;   // bumped by the upper neighbour
    return WO_OK;
}

// Release every stream that waits on this slab's flags or its neighbours'
// (set them to the maximum): after an error left a sweep half enqueued, the
// other slabs' streams would otherwise wait forever.  Their results are void.
int wo_slab_abort(wo_ctx* ctx) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (!ctx->in_flags) return WO_OK;
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaMemsetAsync(ctx->in_flags, 0xff, 4 * sizeof(unsigned int), s);
    for (unsigned int* f : {ctx->peer_lo_flag, ctx->peer_hi_flag})
        if (f) {   // the two parity words of the neighbour's flag
            cudaMemsetAsync(f, 0xff, sizeof(unsigned int), s);
            cudaMemsetAsync(f + 2, 0xff, sizeof(unsigned int), s);
        }
    const cudaError_t e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    CK(e);
    return WO_OK;
}

// Diagnostics of the peer-store protocol without touching the context's
// stream: out = {flag words [4], signals sent this epoch, epoch, stream idle}
int wo_prepare_two_step(wo_ctx* ctx, int* ready) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ready, "wo_prepare_two_step: null output");
    CK(cudaSetDevice(ctx->device));
    // allocates the extra levels and the material, builds the maps and the
    // support forces now (pair_ready), so a decomposition can agree on the
    // launch kind before any peer-store sweep
    *ready = pair_ready(ctx) ? 1 : 0;
    CK(cudaStreamSynchronize(ctx->stream));
    return WO_OK;
}

int wo_slab_state(wo_ctx* ctx, int64_t* out) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    unsigned int w[4] = {0, 0, 0, 0};
    if (ctx->in_flags) {
        cudaStream_t s = nullptr;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        cudaMemcpyAsync(w, ctx->in_flags, sizeof(w), cudaMemcpyDeviceToHost, s);
        const cudaError_t e = cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
        CK(e);
    }
    for (int i = 0; i < 4; ++i) out[i] = w[i];
    out[4] = ctx->p2p_seq;
    out[5] = ctx->p2p_epoch;
    out[6] = cudaStreamQuery(ctx->stream) == cudaSuccess ? 1 : 0;
    (void)cudaGetLastError();
    return WO_OK;
}

int wo_slab_peers(wo_ctx* ctx, void* const* lo_ghost, void* const* hi_ghost, void* lo_flag,
                  void* hi_flag) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->stream));
    bool any = false;
    for (int b = 0; b < 4; ++b) {
        ctx->peer_lo[b] = ctx->has_lo && lo_ghost ? static_cast<char*>(lo_ghost[b]) : nullptr;
        ctx->peer_hi[b] = ctx->has_hi && hi_ghost ? static_cast<char*>(hi_ghost[b]) : nullptr;
        any |= ctx->peer_lo[b] || ctx->peer_hi[b];
    }
    ctx->peer_lo_flag = ctx->has_lo ? static_cast<unsigned int*>(lo_flag) : nullptr;
    ctx->peer_hi_flag = ctx->has_hi ? static_cast<unsigned int*>(hi_flag) : nullptr;
    bool full = true;
    for (int b = 0; b < 4; ++b)
        full &= (!ctx->has_lo || ctx->peer_lo[b]) && (!ctx->has_hi || ctx->peer_hi[b]);
    REQUIRE(!any || (full && (!ctx->has_lo || ctx->peer_lo_flag) &&
                     (!ctx->has_hi || ctx->peer_hi_flag)),
            "peer ghost stores need all four level buffers and the flag of every neighbour");
    REQUIRE(!any || ((!ctx->has_lo || ctx->gl == 2) && (!ctx->has_hi || ctx->gh == 2) &&
                     ctx->kn0 >= 2),
            "peer ghost stores need two ghost planes per neighbour and slabs of >= 2 planes");
    // stores into another GPU's memory need peer access from this device
    const void* ptrs[4] = {ctx->peer_lo[0], ctx->peer_hi[0], ctx->peer_lo_flag, ctx->peer_hi_flag};
    for (const void* q : ptrs) {
        if (!q) continue;
        cudaPointerAttributes pa{};
        CK(cudaPointerGetAttributes(&pa, q));
        if (pa.type == cudaMemoryTypeDevice && pa.device != ctx->device) {
            const cudaError_t e = cudaDeviceEnablePeerAccess(pa.device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
            else CK(e);
        }
    }
    if (any) {
        // no lazy kernel load (a context-wide synchronisation) may happen
        // while a stream waits on a neighbour (launchers.cuh)
        if (ctx->itemsize == 4) {
            preload_step_kernels<float>();
            preload_step2_kernels<float>();
        } else {
            preload_step_kernels<double>();
            preload_step2_kernels<double>();
        }
        CK(cudaGetLastError());
    }
    if (any) {   // fresh flags on every slab before any sweep (wire up all slabs first)
        if ((rc = ensure_four(ctx))) return rc;
        if ((rc = ensure_flags(ctx))) return rc;
        CK(cudaMemsetAsync(ctx->in_flags, 0, 4 * sizeof(unsigned int), ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    ctx->p2p_seq = 0;
    ctx->p2p_epoch = 0;
    ctx->p2p = any;
    ++ctx->gen;
    return WO_OK;
}

typedef CUresult (*PfnAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

int wo_ipc_export(wo_ctx* ctx, const void* dev_ptr, void* handle, int64_t* offset) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(dev_ptr && handle && offset, "wo_ipc_export: null argument");
    CK(cudaSetDevice(ctx->device));
    static PfnAddressRange range = [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        return cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) ==
                               cudaSuccess && q == cudaDriverEntryPointSuccess
                   ? reinterpret_cast<PfnAddressRange>(p)
                   : nullptr;
    }();
    if (!range) return cu_fail(ctx, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS)
        return cu_fail(ctx, "cuMemGetAddressRange failed (not a device allocation?)");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    std::memcpy(handle, &h, sizeof(h));
    *offset = (int64_t)((CUdeviceptr)dev_ptr - base);
    return WO_OK;
}

int wo_ipc_open(wo_ctx* ctx, const void* handle, int64_t offset, void** ptr) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(handle && ptr && offset >= 0, "wo_ipc_open: bad argument");
    CK(cudaSetDevice(ctx->device));
    const std::string key(static_cast<const char*>(handle), sizeof(cudaIpcMemHandle_t));
    char* base = nullptr;
    for (auto& m : ctx->ipc_maps)   // one mapping per exported allocation
        if (m.first == key) base = m.second;
    if (!base) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        void* p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        base = static_cast<char*>(p);
        ctx->ipc_maps.emplace_back(key, base);
    }
    *ptr = base + offset;
    return WO_OK;
}

int wo_halo_planes_out(wo_ctx* ctx, void** first, void** last, void** ghost_lo, void** ghost_hi,
                       int64_t* plane_bytes) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    const size_t pb = (size_t)ctx->plane() * ctx->itemsize;
    char* c = ctx->uprev();   // before the interior part rotates: the new level
    *first = c;
    *last = c + (size_t)(ctx->kn0 - 1) * pb;
    *ghost_lo = ctx->has_lo ? c - pb : nullptr;
    *ghost_hi = ctx->has_hi ? c + (size_t)ctx->kn0 * pb : nullptr;
    *plane_bytes = (int64_t)pb;
    return WO_OK;
}

void* wo_stream(wo_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

static int exchange_local(wo_ctx* lower, wo_ctx* upper, bool out_level) {
    if (!lower || !upper) return WO_ERR_CONFIG;
    wo_ctx* ctx = lower;
    REQUIRE(lower->has_hi && upper->has_lo && lower->plane() == upper->plane() &&
                lower->itemsize == upper->itemsize,
            "contexts are not adjacent slabs");
    const size_t pb = (size_t)lower->plane() * lower->itemsize;
    CK(cudaStreamSynchronize(lower->stream));
    CK(cudaSetDevice(upper->device));
    CK(cudaStreamSynchronize(upper->stream));
    char* lo = out_level ? lower->uprev() : lower->ucur();
    char* up = out_level ? upper->uprev() : upper->ucur();
    char* lo_last = lo + (size_t)(lower->kn0 - 1) * pb;
    char* lo_ghost = lo + (size_t)lower->kn0 * pb;
    char* up_first = up;
    char* up_ghost = up - pb;
    if (lower->device == upper->device) {
        CK(cudaMemcpy(up_ghost, lo_last, pb, cudaMemcpyDeviceToDevice));
        CK(cudaMemcpy(lo_ghost, up_first, pb, cudaMemcpyDeviceToDevice));
    } else {
        CK(cudaMemcpyPeer(up_ghost, upper->device, lo_last, lower->device, pb));
        CK(cudaMemcpyPeer(lo_ghost, lower->device, up_first, upper->device, pb));
    }
    CK(cudaSetDevice(lower->device));
    return WO_OK;
}

int wo_exchange_local(wo_ctx* lower, wo_ctx* upper) { return exchange_local(lower, upper, false); }

int wo_exchange_local_out(wo_ctx* lower, wo_ctx* upper) { return exchange_local(lower, upper, true); }

int wo_sweep_adjoint_reference(wo_ctx* ctx, int64_t n_steps, double dt, int64_t* fail_step,
                               double* fail_max) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->material_set, "material not set");
    return DISPATCH(ctx, sweep_adjoint_reference_t, ctx, n_steps, dt, fail_step, fail_max);
}

int wo_get_history(wo_ctx* ctx, int64_t n_first, int64_t n_count, void* out) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    const size_t fb = ctx->field_bytes();
    REQUIRE(n_first >= 0 && n_count >= 0 &&
                (size_t)(n_first + n_count) * fb <= ctx->hist_bytes,
            "history levels out of range (record them with WO_FWD_HISTORY)");
    return download_field(ctx, out, ctx->hist + (size_t)n_first * fb, (size_t)n_count * fb);
}

int wo_free_history(wo_ctx* ctx) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->hist) {
        cudaFree(ctx->hist);
        ctx->dev_bytes -= (int64_t)ctx->hist_bytes;
        ctx->hist = nullptr;
        ctx->hist_bytes = 0;
    }
    if (ctx->u3) {
        cudaFree(ctx->u3);
        ctx->dev_bytes -= (int64_t)ctx->u3_bytes;
        ctx->u3 = nullptr;
        ctx->u3_bytes = 0;
    }
    return WO_OK;
}

int wo_shot_misfit(wo_ctx* ctx, int64_t n_steps, int kind, const double* measured, double c1,
                   double c2, double c3, double c4, double adj_coef, int write_adj, double k,
                   double* cost_out) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(kind == WO_SHOT_FWI || kind == WO_SHOT_TATO, "unknown shot kind");
    return DISPATCH(ctx, misfit_t, ctx, n_steps, kind, measured, c1, c2, c3, c4, adj_coef,
                    write_adj, k, cost_out);
}

int wo_get_store(wo_ctx* ctx, int64_t n_steps, void* out) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    const size_t b = (size_t)n_steps * ctx->n_sup * ctx->itemsize;
    REQUIRE(ctx->store_bytes >= b, "store smaller than requested");
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(out, ctx->store, b, cudaMemcpyDeviceToHost));
    return WO_OK;
}

int wo_sweep_backward(wo_ctx* ctx, int64_t n_steps, int64_t src_flat, const double* src_amp,
                      int inject_support, int accumulate, double dt, int64_t* fail_step,
                      double* fail_max) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->material_set, "material not set");
    return DISPATCH(ctx, sweep_backward_t, ctx, n_steps, src_flat, src_amp, inject_support,
                    accumulate, dt, fail_step, fail_max);
}

int wo_get_field(wo_ctx* ctx, int which, int first_axis_fastest, void* out) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(which >= WO_FIELD_GAMMA && which <= WO_FIELD_ACC, "unknown field");
    REQUIRE(out, "null output");
    const char* src = which == WO_FIELD_GAMMA ? ctx->base0(ctx->gamma)
                      : which == WO_FIELD_UPREV ? ctx->uprev()
                      : which == WO_FIELD_UCUR ? ctx->ucur()
                                               : ctx->acc;
    const size_t fb = ctx->field_bytes();
    if (!first_axis_fastest) return download_field(ctx, out, src, fb);
    rc = ensure(ctx, &ctx->scratch, &ctx->scratch_bytes, fb);
    if (rc) return rc;
    const int A = ctx->kn0, B = ctx->kn1, C = ctx->kn2;
    dim3 grid((C + 31) / 32, (A + 31) / 32, B), block(32, 8);
    if (ctx->itemsize == 4)
        reverse_axes_kernel<float><<<grid, block, 0, ctx->stream>>>(
            reinterpret_cast<const float*>(src), reinterpret_cast<float*>(ctx->scratch), A, B, C);
    else
        reverse_axes_kernel<double><<<grid, block, 0, ctx->stream>>>(
            reinterpret_cast<const double*>(src), reinterpret_cast<double*>(ctx->scratch), A, B, C);
    ctx->launches++;
    CK(cudaGetLastError());
    return download_field(ctx, out, ctx->scratch, fb);
}

int wo_get_gradient(wo_ctx* ctx, double two_k, void* out) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    return DISPATCH(ctx, gradient_t, ctx, two_k, out);
}

int wo_step(wo_ctx* ctx, int64_t n_force, const int64_t* idx, const double* vals,
            const double* dense_force, int want_max, double* max_out) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(ctx->material_set, "material not set");
    return DISPATCH(ctx, step_t, ctx, n_force, idx, vals, dense_force, want_max, max_out);
}

int wo_set_profiling(wo_ctx* ctx, int on) {
    if (!ctx) return WO_ERR_CONFIG;
    ctx->prof = on > 0;
    ctx->prof_every = on > 0 ? on : 0;
    ctx->prof_tick = 0;
    return WO_OK;
}

int wo_stats(wo_ctx* ctx, int64_t* launches, int64_t* step_launches, double* step_kernel_ms) {
    if (!ctx) return WO_ERR_CONFIG;
    if (launches) *launches = ctx->launches;
    if (step_launches) *step_launches = ctx->step_launches;
    if (step_kernel_ms) *step_kernel_ms = ctx->step_ms;
    return WO_OK;
}

int wo_reset_stats(wo_ctx* ctx) {
    if (!ctx) return WO_ERR_CONFIG;
    ctx->launches = ctx->step_launches = ctx->pair_launches = 0;
    ctx->step_ms = 0.0;
    ctx->prof_ms[0] = ctx->prof_ms[1] = 0.0;
    ctx->prof_n[0] = ctx->prof_n[1] = 0;
    return WO_OK;
}

int64_t wo_device_bytes(const wo_ctx* ctx) { return ctx ? ctx->dev_bytes : 0; }

int wo_field_buffers(const wo_ctx* ctx) {
    if (!ctx) return 0;
    int n = 0;
    for (const char* p : {ctx->gamma, ctx->u[0], ctx->u[1], ctx->u[2], ctx->u[3], ctx->acc, ctx->u3})
        n += p ? 1 : 0;
    return n + (ctx->mat4 ? 4 : 0);
}

int64_t wo_pair_launches(const wo_ctx* ctx) { return ctx ? ctx->pair_launches : 0; }

int wo_profile_stats(const wo_ctx* ctx, double* single_ms, int64_t* single_n, double* pair_ms,
                     int64_t* pair_n) {
    if (!ctx) return WO_ERR_CONFIG;
    if (single_ms) *single_ms = ctx->prof_ms[0];
    if (single_n) *single_n = ctx->prof_n[0];
    if (pair_ms) *pair_ms = ctx->prof_ms[1];
    if (pair_n) *pair_n = ctx->prof_n[1];
    return WO_OK;
}

int wo_timer_mark(wo_ctx* ctx, int idx) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(idx >= 0 && idx < 8, "timer slot out of range");
    if (!ctx->marks[idx]) CK(cudaEventCreate(&ctx->marks[idx]));
    CK(cudaEventRecord(ctx->marks[idx], ctx->stream));
    return WO_OK;
}

int wo_timer_elapsed(wo_ctx* ctx, int a, int b, double* ms) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    REQUIRE(a >= 0 && a < 8 && b >= 0 && b < 8 && ctx->marks[a] && ctx->marks[b],
            "timer slots not recorded");
    CK(cudaEventSynchronize(ctx->marks[b]));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, ctx->marks[a], ctx->marks[b]));
    *ms = f;
    return WO_OK;
}

void* wo_accumulator_ptr(wo_ctx* ctx) { return ctx ? (void*)ctx->acc : nullptr; }

int wo_synchronize(wo_ctx* ctx) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    return WO_OK;
}

// ---------------------------------------------------------------- drop-ins
namespace {
struct Scratch {
    std::vector<void*> p;
    ~Scratch() {
        for (void* q : p) cudaFree(q);
    }
    void* put(const void* h, size_t b) {
        void* d = nullptr;
        if (cudaMalloc(&d, b ? b : 16) != cudaSuccess) return nullptr;
        p.push_back(d);
        if (h) cudaMemcpy(d, h, b, cudaMemcpyHostToDevice);
        return d;
    }
};

void map3(int ndim, const int64_t* shape, int& n0, int& n1, int& n2) {
    if (ndim == 3) { n0 = (int)shape[0]; n1 = (int)shape[1]; n2 = (int)shape[2]; }
    else if (ndim == 2) { n0 = 1; n1 = (int)shape[0]; n2 = (int)shape[1]; }
    else { n0 = 1; n1 = 1; n2 = (int)shape[0]; }
}
}  // namespace

int wo_apply_step(int ndim, const int64_t* shape, int itemsize, const void* u_prev,
                  const void* u_cur, const void* wf0, const void* wf1, const void* wf2,
                  const void* coef, void* out, int device) {
    if (ndim < 1 || ndim > 3 || (itemsize != 4 && itemsize != 8)) return WO_ERR_CONFIG;
    if (cudaSetDevice(device) != cudaSuccess) return WO_ERR_CUDA;
    int n0, n1, n2;
    map3(ndim, shape, n0, n1, n2);
    const long long C = (long long)n0 * n1 * n2;
    const size_t fb = (size_t)C * itemsize;
    // face arrays in kernel space: axis a of the reference -> kernel axis
    const void* wf[3] = {wf0, wf1, wf2};
    const void* kw[3] = {nullptr, nullptr, nullptr};
    const int first = 3 - ndim;
    for (int a = 0; a < ndim; ++a) kw[first + a] = wf[a];
    size_t wb_[3];
    wb_[0] = (size_t)(n0 - 1) * n1 * n2 * itemsize;
    wb_[1] = (size_t)n0 * (n1 - 1) * n2 * itemsize;
    wb_[2] = (size_t)n0 * n1 * (n2 - 1) * itemsize;
    Scratch s;
    void* d_up = s.put(u_prev, fb);
    void* d_u = s.put(u_cur, fb);
    void* d_c = s.put(coef, fb);
    void* d_o = s.put(nullptr, fb);
    void* d_w[3] = {nullptr, nullptr, nullptr};
    for (int a = 0; a < 3; ++a)
        if (kw[a]) d_w[a] = s.put(kw[a], wb_[a]);
    if (!d_up || !d_u || !d_c || !d_o) return WO_ERR_CUDA;
    if (itemsize == 4)
        dropin_step_kernel<float><<<592, 256>>>(n0, n1, n2, (const float*)d_up, (const float*)d_u,
                                                (const float*)d_w[0], (const float*)d_w[1],
                                                (const float*)d_w[2], (const float*)d_c, (float*)d_o);
    else
        dropin_step_kernel<double><<<592, 256>>>(n0, n1, n2, (const double*)d_up,
                                                 (const double*)d_u, (const double*)d_w[0],
                                                 (const double*)d_w[1], (const double*)d_w[2],
                                                 (const double*)d_c, (double*)d_o);
    if (cudaGetLastError() != cudaSuccess) return WO_ERR_CUDA;
    if (cudaMemcpy(out, d_o, fb, cudaMemcpyDeviceToHost) != cudaSuccess) return WO_ERR_CUDA;
    return WO_OK;
}

int wo_apply_kernel_increment(int ndim, const int64_t* shape, int itemsize, void* acc,
                              const void* a_old, const void* a_mid, const void* a_new,
                              const void* b_old, const void* b_mid, const void* b_new, double cv,
                              double cg, double inv2dt, double inv2dx, double sdt, int device) {
    if (ndim < 1 || ndim > 3 || (itemsize != 4 && itemsize != 8)) return WO_ERR_CONFIG;
    if (cudaSetDevice(device) != cudaSuccess) return WO_ERR_CUDA;
    int n0, n1, n2;
    map3(ndim, shape, n0, n1, n2);
    const size_t fb = (size_t)n0 * n1 * n2 * itemsize;
    Scratch s;
    void* d[7] = {s.put(acc, fb), s.put(a_old, fb), s.put(a_mid, fb), s.put(a_new, fb),
                  s.put(b_old, fb), s.put(b_mid, fb), s.put(b_new, fb)};
    for (void* q : d)
        if (!q) return WO_ERR_CUDA;
    if (itemsize == 4)
        dropin_ki_kernel<float><<<592, 256>>>(
            ndim, n0, n1, n2, (float*)d[0], (const float*)d[1], (const float*)d[2],
            (const float*)d[3], (const float*)d[4], (const float*)d[5], (const float*)d[6],
            (float)cv, (float)cg, (float)inv2dt, (float)inv2dx, (float)sdt);
    else
        dropin_ki_kernel<double><<<592, 256>>>(
            ndim, n0, n1, n2, (double*)d[0], (const double*)d[1], (const double*)d[2],
            (const double*)d[3], (const double*)d[4], (const double*)d[5], (const double*)d[6], cv,
            cg, inv2dt, inv2dx, sdt);
    if (cudaGetLastError() != cudaSuccess) return WO_ERR_CUDA;
    if (cudaMemcpy(acc, d[0], fb, cudaMemcpyDeviceToHost) != cudaSuccess) return WO_ERR_CUDA;
    return WO_OK;
}

// ------------------------------------------------------------ design chain
namespace {
struct DevFootprint {
    Scratch s;
    Footprint fp{};
    bool ok = false;
    DevFootprint(int ndim, int n, const int* off, const double* w) {
        std::vector<int> o3((size_t)n * 3, 0);
        for (int f = 0; f < n; ++f)
            for (int a = 0; a < ndim; ++a) o3[(size_t)f * 3 + (3 - ndim) + a] = off[(size_t)f * ndim + a];
        fp.n = n;
        fp.off = (const int*)s.put(o3.data(), o3.size() * sizeof(int));
        fp.w = (const double*)s.put(w, (size_t)n * sizeof(double));
        ok = fp.off && fp.w;
    }
};
}  // namespace

int wo_design_filter(int ndim, const int64_t* shape, const double* gamma,
                     const unsigned char* mask, int n_fp, const int* offsets,
                     const double* weights, double* out, int device) {
    if (ndim < 1 || ndim > 3 || n_fp < 1) return WO_ERR_CONFIG;
    if (cudaSetDevice(device) != cudaSuccess) return WO_ERR_CUDA;
    int n0, n1, n2;
    map3(ndim, shape, n0, n1, n2);
    const long long N = (long long)n0 * n1 * n2;
    DevFootprint F(ndim, n_fp, offsets, weights);
    Scratch s;
    double* d_g = (double*)s.put(gamma, N * 8);
    unsigned char* d_m = mask ? (unsigned char*)s.put(mask, N) : nullptr;
    double* d_num = (double*)s.put(nullptr, N * 8);
    double* d_den = (double*)s.put(nullptr, N * 8);
    double* d_o = (double*)s.put(nullptr, N * 8);
    if (!F.ok || !d_g || !d_num || !d_den || !d_o || (mask && !d_m)) return WO_ERR_CUDA;
    masked_correlate_kernel<<<592, 256>>>(n0, n1, n2, d_g, d_m, 1, F.fp, d_num, d_den);
    filter_finish_kernel<<<592, 256>>>(N, d_g, d_m, d_num, d_den, d_o);
    if (cudaGetLastError() != cudaSuccess) return WO_ERR_CUDA;
    if (cudaMemcpy(out, d_o, N * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return WO_ERR_CUDA;
    return WO_OK;
}

int wo_design_project(int64_t n, const double* g_tilde, double beta, double eta, double t_be,
                      double denom, const unsigned char* mask, double* out, int device) {
    if (cudaSetDevice(device) != cudaSuccess) return WO_ERR_CUDA;
    Scratch s;
    double* d_g = (double*)s.put(g_tilde, n * 8);
    unsigned char* d_m = mask ? (unsigned char*)s.put(mask, n) : nullptr;
    double* d_o = (double*)s.put(nullptr, n * 8);
    if (!d_g || !d_o || (mask && !d_m)) return WO_ERR_CUDA;
    heaviside_kernel<<<592, 256>>>(n, d_g, beta, eta, t_be, denom, d_m, d_o);
    if (cudaGetLastError() != cudaSuccess) return WO_ERR_CUDA;
    if (cudaMemcpy(out, d_o, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return WO_ERR_CUDA;
    return WO_OK;
}

int wo_design_chain(int ndim, const int64_t* shape, const double* dcdbar, const double* g_tilde,
                    double beta, double eta, double denom, const unsigned char* mask, int n_fp,
                    const int* offsets, const double* weights, double* out, int device) {
    if (ndim < 1 || ndim > 3 || n_fp < 1) return WO_ERR_CONFIG;
    if (cudaSetDevice(device) != cudaSuccess) return WO_ERR_CUDA;
    int n0, n1, n2;
    map3(ndim, shape, n0, n1, n2);
    const long long N = (long long)n0 * n1 * n2;
    DevFootprint F(ndim, n_fp, offsets, weights);
    Scratch s;
    double* d_g = (double*)s.put(dcdbar, N * 8);
    double* d_t = (double*)s.put(g_tilde, N * 8);
    unsigned char* d_m = mask ? (unsigned char*)s.put(mask, N) : nullptr;
    double* d_inner = (double*)s.put(nullptr, N * 8);
    double* d_den = (double*)s.put(nullptr, N * 8);
    double* d_ratio = (double*)s.put(nullptr, N * 8);
    double* d_o = (double*)s.put(nullptr, N * 8);
    if (!F.ok || !d_g || !d_t || !d_inner || !d_den || !d_ratio || !d_o || (mask && !d_m))
        return WO_ERR_CUDA;
    chain_inner_kernel<<<592, 256>>>(N, d_g, d_t, beta, eta, denom, d_m, d_inner);
    masked_correlate_kernel<<<592, 256>>>(n0, n1, n2, d_inner, d_m, 1, F.fp, nullptr, d_den);
    chain_ratio_kernel<<<592, 256>>>(N, d_inner, d_den, d_m, d_ratio);
    masked_correlate_kernel<<<592, 256>>>(n0, n1, n2, d_ratio, nullptr, 0, F.fp, d_o, nullptr);
    mask_zero_kernel<<<592, 256>>>(N, d_m, d_o);
    if (cudaGetLastError() != cudaSuccess) return WO_ERR_CUDA;
    if (cudaMemcpy(out, d_o, N * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return WO_ERR_CUDA;
    return WO_OK;
}

}  // extern "C"
