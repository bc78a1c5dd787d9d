/*
 * waveb200 — C ABI of the B200-native superposed-adjoint hot path.
 *
 * The reference (waveopt, /root/reference/pkg/src/waveopt) has no native
 * boundary: its hot loops are Numba functions called per time step from
 * Python (kernels.py:136-152) inside the sweep loops of gradients.py and
 * solver.py.  A per-step FFI call would serialise 2N host round trips, so
 * this ABI exports SWEEP-level entry points that replace whole reference
 * loops; per-step entries remain for propagate_step / run_backward.
 *
 * Conventions
 *  - Plain C types only: host pointers + sizes.  Arrays are C-order
 *    (axis 0 outermost, last axis contiguous), exactly numpy's default.
 *  - Field dtype is chosen per context: itemsize 4 ("single") or 8
 *    ("double"); void* field arrays use that dtype.  Costs, amplitudes,
 *    measured traces and scalars are always double (fwi.py:57-63).
 *  - A context owns its device buffers (gamma, two field levels,
 *    accumulator — the four field buffers of gradients.py:302-303 — plus
 *    compact support storage).  Calls are blocking and not thread-safe;
 *    one context per GPU.
 *  - Status codes mirror the CLI exit codes of cli.py:333-342.
 */
#ifndef WAVEB200_H
#define WAVEB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WO_OK 0
#define WO_ERR_CONFIG 1   /* ConfigError            (grids.py:20)  */
#define WO_ERR_UNSTABLE 2 /* SolverInstabilityError (solver.py:34) */
#define WO_ERR_BUDGET 3   /* ResourceBudgetError    (solver.py:44) */
#define WO_ERR_CUDA 4     /* device / driver failure                */

#define WO_RHO_SCALED 0   /* grids.py:99  */
#define WO_ACOUSTIC 1     /* grids.py:100 */

#define WO_SHOT_FWI 1     /* fwi.py:48-63  FwiShot  */
#define WO_SHOT_TATO 2    /* tato.py:143-163 TatoShot */

typedef struct wo_ctx wo_ctx;

/* Library version (major*10000 + minor*100 + patch). */
int wo_version(void);
/* Number of visible CUDA devices (0 when none). */
int wo_device_count(void);
/* Message of the last failed call on ctx (ctx == NULL: last wo_create). */
const char* wo_last_error(const wo_ctx* ctx);

/* Create a context for one grid (grids.py:31-72: 1 <= ndim <= 3) at one
 * dtype on one device.  Replaces the allocations of gradients.py:302-303 and
 * solver.py:138-143 (SolverWindow.zeros). */
int wo_create(wo_ctx** out, int ndim, const int64_t* shape, double dx, int itemsize,
              int device);
/* Slab of a 3D grid for slab decomposition along axis 0: the context holds
 * global planes [i_begin, i_end) plus one ghost plane on each side that has
 * a neighbour. */
int wo_create_slab(wo_ctx** out, const int64_t* global_shape, int64_t i_begin,
                   int64_t i_end, double dx, int itemsize, int device);
void wo_destroy(wo_ctx* ctx);

/* Material: replaces prepare_material (solver.py:89-125).  gamma is fp64,
 * C-order over the context's planes including ghosts (slab: planes
 * [max(i_begin-1,0), min(i_end+1,n0)) ).  Coefficients are recomputed from
 * gamma on the fly with the reference's exact operations.  ratio2 is the
 * squared Courant-type ratio evaluated by the caller exactly as the
 * reference does with Python's ** operator: (c0*dt/dx)**2 for rho_scaled
 * (solver.py:96), (dt/dx)**2 for acoustic (solver.py:108). */
int wo_set_material(wo_ctx* ctx, int flavor, const double* gamma, double rho0, double rho1,
                    double kappa1, double rho2, double kappa2, double dt, double ratio2);
/* Options.  WO_OPT_FAST_DIV (default 1): let wo_set_material enable the
 * branch-free division path when it verifies bit-identical to the IEEE
 * intrinsics for every coefficient of the material (0 = always intrinsics).
 * wo_fast_div_active reports the path in use. */
#define WO_OPT_FAST_DIV 1
/* WO_OPT_PAIR_KERNEL (default 1): two-cells-per-thread vectorised step kernel
 * on grids with an even last axis (0 = scalar kernel everywhere). */
#define WO_OPT_PAIR_KERNEL 2
/* WO_OPT_TMA_KERNEL (default 1): TMA/mbarrier-pipelined step kernel when the
 * grid tiles exactly into 64 x 8 cells (0 = never). */
#define WO_OPT_TMA_KERNEL 3
/* WO_OPT_TWO_STEP (default 1; slab contexts 0): advance two time steps per
 * pass over HBM (temporal blocking, identical arithmetic) on fp32 and fp64
 * contexts whose plane tiles into 64 x 8 or 32 x 16 cells (2: the same,
 * kept for compatibility); 0 = never.  Sweeps fall back to single steps at odd range ends, while
 * recording history, and everywhere else.  Slabs take two-step passes only
 * with peer ghost stores and two ghost planes per neighbour; the caller
 * enables them on every slab of a decomposition or on none (all slabs must
 * launch alike) and only when no support node lies on a plane next to a
 * slab boundary (the recomputed planes do not inject the neighbour's
 * adjoint store).  Single-domain contexts with 0 hold the reference's four
 * solution-sized buffers: gamma, two window levels (u^{n+1} in place over
 * u^{n-1}) and the accumulator. */
#define WO_OPT_TWO_STEP 4
/* WO_OPT_PLANE_PART (slab contexts, default 0): 1 = the next single step
 * computes only the boundary planes 0 and n0-1 (no rotation), 2 = only the
 * interior planes, then rotates.  Split calls do not synchronise the
 * stream, so the halo exchange of the new boundary planes (wo_halo_planes_out,
 * on any stream ordered after the boundary part) overlaps the interior. */
#define WO_OPT_PLANE_PART 5
/* WO_OPT_GRAPHS (default 1): a sweep whose launch sequence repeats (same
 * range, sources, amplitudes, window state and context settings) is
 * captured into a CUDA graph on its second occurrence and replayed from then
 * on (launch-bound small grids gain most); 0 = always launch directly. */
#define WO_OPT_GRAPHS 6
/* WO_OPT_CLUSTER (default 2): small 2D grids (up to 65,536 cells: one
 * 16-CTA thread-block cluster, 2 x 4 cells per thread) run every sweep as ONE
 * cluster-resident launch (fields in registers, neighbour rows exchanged
 * through shared memory / st.async into the cluster peers, identical
 * arithmetic); 1 = on, 0 = step launches, 2 = the default (on). */
#define WO_OPT_CLUSTER 7
int wo_set_option(wo_ctx* ctx, int option, int value);
/* Device-resident optimisation loop (fwi.py:178-238 with
 * optim.py adam_step / clip_bounds): fp64 parameters (gamma), the Adam
 * moments and a frozen mask live on the GPU.  wo_opt_step(t) reads the
 * finished gradient from the accumulator (zeroed on frozen cells when
 * zero_frozen_grad), applies Adam step t and the [lo, hi] clip with numpy's
 * fp64 operation order, pins frozen cells to frozen_value, writes
 * gamma.astype(T) as the context's new material and returns the gradient's
 * L2 norm (fixed-order fp64 sum; a log value).  wo_opt_get downloads the
 * parameters. */
int wo_opt_init(wo_ctx* ctx, const double* params, const unsigned char* frozen, int zero_frozen_grad,
                double lo, double hi, double frozen_value, double alpha, double beta1,
                double beta2, double eps);
int wo_opt_step(wo_ctx* ctx, int t, double* grad_norm);
int wo_opt_get(wo_ctx* ctx, double* params);
/* Device-resident TATO design loop (tato.py:238-304): the optimiser's
 * parameters are gamma_raw; wo_design_setup stores the design mask (NULL =
 * everywhere) and the filter footprint (as wo_design_filter) and switches
 * wo_opt_step to the chain-rule gradient.  wo_design_material: g_tilde =
 * density_filter(gamma_raw), g_bar = heaviside_project(g_tilde) -> material
 * g_bar.astype(T).  wo_design_gradient: chain_rule(acc, g_tilde) -> the
 * gradient of the next wo_opt_step.  wo_design_get: 0 g_tilde, 1 g_bar,
 * 2 gradient (fp64 fields). */
int wo_design_setup(wo_ctx* ctx, const unsigned char* mask, int n_fp, const int* offsets,
                    const double* weights);
int wo_design_material(wo_ctx* ctx, double beta, double eta, double t_be, double denom);
int wo_design_gradient(wo_ctx* ctx, double beta, double eta, double denom);
int wo_design_get(wo_ctx* ctx, int which, double* out);
int wo_fast_div_active(const wo_ctx* ctx);
/* Kernel-increment scalars (gradients.py:117-129, kernels.py:149-152): the
 * fp64 values cv, cg, 1/(2dt), 1/(2dx); cast to the field dtype here. */
int wo_set_kernel_coefficients(wo_ctx* ctx, double cv, double cg, double inv2dt,
                               double inv2dx);
/* Support nodes (sensor or objective-region flat indices, strictly
 * increasing, local to the context).  Device support order = this order. */
int wo_set_support(wo_ctx* ctx, int64_t n_sup, const int64_t* flat_sorted);

/* Window management (solver.py:128-151). */
int wo_reset_window(wo_ctx* ctx);                                  /* u^0 = u^1 = 0 */
int wo_set_window(wo_ctx* ctx, const void* u_prev, const void* u_cur);
int wo_get_window(wo_ctx* ctx, void* u_prev, void* u_cur);
int wo_swap_direction(wo_ctx* ctx);
/* Device snapshot of the state a forward sweep leaves behind — the two window
 * levels, the accumulator and the first n_steps rows of the support store —
 * so k-dependent backward sweeps can be repeated from it (batched
 * calibrate_k / ksweep of a single-shot problem, gradients.py:480-548: the
 * forward sweep and the traces do not depend on k).  op: WO_SNAP_SAVE,
 * WO_SNAP_RESTORE (n_steps must match the save), WO_SNAP_FREE. */
#define WO_SNAP_FREE 0
#define WO_SNAP_SAVE 1
#define WO_SNAP_RESTORE 2
int wo_snapshot(wo_ctx* ctx, int op, int64_t n_steps);                                /* solver.py:149 */
int wo_zero_accumulator(wo_ctx* ctx);
int wo_get_accumulator(wo_ctx* ctx, void* out);
int wo_set_accumulator(wo_ctx* ctx, const void* in);

#define WO_FWD_ACCUMULATE 1 /* subtract the self-kernel (superposed engine) */
#define WO_FWD_HISTORY 2    /* keep all N+1 levels on the device (reference engine) */

/* Forward sweep n = 1..N-1 (gradients.py:214-250 _forward_pass;
 * solver.py:282-340 run_forward): steps the window, injects the sources
 * (src_flat[n_src], amplitudes src_amp[n_src][N] in fp64), records u^n on
 * the support into the compact store when a support is set, subtracts the
 * self-kernel when flags & WO_FWD_ACCUMULATE (sdt = -dt), records the full
 * history when flags & WO_FWD_HISTORY, and checks stability every 50 steps
 * and at the last one against 1e6*scale (scale <= 0: finiteness only).  On
 * WO_ERR_UNSTABLE, *fail_step / *fail_max hold the first failing check.
 * *peak_out = max over the checks. */
int wo_sweep_forward(wo_ctx* ctx, int64_t n_steps, int n_src, const int64_t* src_flat,
                     const double* src_amp, int flags, double dt, double scale,
                     double* peak_out, int64_t* fail_step, double* fail_max);
/* Step ranges of the two sweeps, for drivers that exchange slab halos
 * between steps (multi-GPU slab decomposition).  Forward: steps n in
 * [n_begin, n_end); the range starting at n = 1 initialises the sweep.
 * Backward: steps n = n_hi .. n_lo+1 descending; the range starting at
 * n_hi = N-1 swaps the direction.  No stability evaluation: read the
 * per-step max|u| with wo_check_maxima (out[n], n in [0, N+2), step n's
 * check value) and combine across slabs.  Each call returns synchronised,
 * except on a slab with peer ghost stores (wo_slab_peers), where the ranges
 * only enqueue (a whole sweep is one range; the neighbours' sweeps may still
 * have to be enqueued) and wo_check_maxima waits for the stream.
 * Slab contexts take source indices local to their own planes, negative ones
 * down to their lowest ghost plane included (a two-step pass recomputes one
 * plane beyond each slab boundary, sources there included); the backward
 * sweeps of a slab take WO_NO_SOURCE for "no source". */
#define WO_NO_SOURCE INT64_MIN
int wo_sweep_forward_range(wo_ctx* ctx, int64_t n_steps, int64_t n_begin, int64_t n_end,
                           int n_src, const int64_t* src_flat, const double* src_amp, int flags,
                           double dt);
int wo_sweep_backward_range(wo_ctx* ctx, int64_t n_steps, int64_t n_hi, int64_t n_lo,
                            int64_t src_flat, const double* src_amp, int inject_support,
                            int accumulate, double dt);
int wo_check_maxima(wo_ctx* ctx, int64_t n_steps, double* out);
/* Device addresses of the current level's first/last local planes and its
 * ghost planes (NULL when absent), plane size in bytes: the buffers a
 * halo exchange (NCCL send/recv) reads and fills. */
int wo_halo_planes(wo_ctx* ctx, void** first, void** last, void** ghost_lo, void** ghost_hi,
                   int64_t* plane_bytes);
/* Same-process halo exchange between adjacent slabs (same device or peer
 * devices): lower's last plane -> upper's low ghost, upper's first plane ->
 * lower's high ghost, on the current level. */
int wo_exchange_local(wo_ctx* lower, wo_ctx* upper);
/* The planes of the level a split step is writing (before its rotation):
 * what wo_halo_planes returns for the current level after it. */
int wo_halo_planes_out(wo_ctx* ctx, void** first, void** last, void** ghost_lo, void** ghost_hi,
                       int64_t* plane_bytes);
/* The context's CUDA stream (cudaStream_t), for ordering a caller's
 * communication with the library's kernels. */
void* wo_stream(wo_ctx* ctx);
/* wo_exchange_local for the level a split step is writing. */
int wo_exchange_local_out(wo_ctx* lower, wo_ctx* upper);
/* Peer ghost stores (replaces the exchange; the reference has no multi-GPU
 * path — solver.py:128-151 steps one array).  A slab holds two ghost planes
 * per neighbour.  wo_slab_ghosts returns, per level buffer (4), the address of
 * its lowest ghost plane (plane -2) and of its first high ghost plane (plane
 * n0), NULL when absent, and the addresses of its two incoming flags (bumped
 * by the lower / upper neighbour; each flag word has a twin 2 words further
 * for odd sweeps).  wo_slab_peers hands a slab its neighbours' addresses:
 * lo_ghost[4] = the lower neighbour's HIGH ghost planes, hi_ghost[4] = the
 * upper neighbour's LOW ghost planes, lo_flag = the lower neighbour's flag
 * [1], hi_flag = the upper neighbour's flag [0] (all NULL: off).  Then every
 * launch of a sweep (single step or two-step pass) waits on its stream until
 * both neighbours completed their previous launch, stores its own planes 0, 1
 * and n0-2, n0-1 of the level(s) it writes into both its own buffer and the
 * neighbour's ghost planes (NVLink stores when the neighbour is on another
 * GPU; IPC-mapped addresses across processes), and bumps the neighbours'
 * flags: no copy or collective per step.  Each sweep is an epoch with its own
 * flag slot, begun after the window reset; the caller synchronises every slab
 * between sweeps (wo_check_maxima + its cost / stability reduction).  Set up
 * every slab before stepping any; split steps are refused meanwhile. */
int wo_slab_ghosts(wo_ctx* ctx, void** ghost_lo, void** ghost_hi, void** flags);
/* Error recovery: set this slab's and its neighbours' flags to the maximum
 * so no stream keeps waiting on a sweep that was only partly enqueued. */
int wo_slab_abort(wo_ctx* ctx);
/* Prepare two-step passes now (replaces nothing in the reference: the
 * launch-kind agreement of a slab decomposition).  Allocates the two extra
 * level buffers and the precomputed material, builds the tensor maps and the
 * support forces; *ready = 1 when this context will take two-step passes,
 * 0 when it will not (option off, grid shape, or the buffers do not fit).
 * Peer-store slabs must all launch alike: a decomposition whose slabs do not
 * all report 1 sets WO_OPT_TWO_STEP 0 on every slab. */
int wo_prepare_two_step(wo_ctx* ctx, int* ready);

/* Diagnostics (no wait on the context's stream): out[0..3] the flag words,
 * out[4] signals sent in the current epoch, out[5] epochs begun, out[6] 1 if
 * the stream is idle. */
int wo_slab_state(wo_ctx* ctx, int64_t* out);
int wo_slab_peers(wo_ctx* ctx, void* const* lo_ghost, void* const* hi_ghost, void* lo_flag,
                  void* hi_flag);
/* CUDA IPC for peer ghost stores across processes (one slab per rank, the
 * torchrun layout; the reference has no multi-GPU path).  wo_ipc_export
 * writes the 64-byte cudaIpcMemHandle of the allocation holding dev_ptr (a
 * ghost plane or flag from wo_slab_ghosts) and dev_ptr's byte offset in it;
 * the neighbour's process passes both to wo_ipc_open, which maps the
 * allocation once per context (peer access enabled lazily) and returns the
 * address to hand to wo_slab_peers.  Mappings close in wo_destroy. */
int wo_ipc_export(wo_ctx* ctx, const void* dev_ptr, void* handle, int64_t* offset);
int wo_ipc_open(wo_ctx* ctx, const void* handle, int64_t offset, void** ptr);

/* Standard-adjoint sweep of gradient_reference (gradients.py:371-386) using
 * the recorded history and the unscaled compact adjoint store; accumulates
 * the mixed kernel.  wo_free_history releases the history buffer. */
int wo_sweep_adjoint_reference(wo_ctx* ctx, int64_t n_steps, double dt, int64_t* fail_step,
                               double* fail_max);
int wo_free_history(wo_ctx* ctx);
/* Levels u^{n_first} .. u^{n_first+n_count-1} of the history recorded by a
 * WO_FWD_HISTORY forward sweep, C order, to host memory (run_forward's
 * full_history / on_step: solver.py:306-336 in one fused sweep). */
int wo_get_history(wo_ctx* ctx, int64_t n_first, int64_t n_count, void* out);

/* Per-step shot cost and compact adjoint store from the recorded support
 * values (fwi.py:57-63, tato.py:154-163, gradients.py:231-239, 263):
 * cost_n = (((c1*dot)*c2)*c3)/c4; FWI uses measured[n_sup][N] (device
 * support order; NULL reuses the traces of the previous call), TATO adj =
 * adj_coef*u.  When write_adj, the store becomes T(adj)*T(k).  *cost_out =
 * sum over n in order. */
int wo_shot_misfit(wo_ctx* ctx, int64_t n_steps, int kind, const double* measured,
                   double c1, double c2, double c3, double c4, double adj_coef, int write_adj,
                   double k, double* cost_out);
/* Copy the compact store [N][n_sup] (traces, or adjoint after misfit). */
int wo_get_store(wo_ctx* ctx, int64_t n_steps, void* out);

/* Backward superposed sweep n = N-1..1 (gradients.py:253-281) on the
 * swapped window: step + source + support injection of the k-scaled store
 * + self-kernel (sdt = +dt); stability checked every 50 steps and at n=1. */
int wo_sweep_backward(wo_ctx* ctx, int64_t n_steps, int64_t src_flat, const double* src_amp,
                      int inject_support, int accumulate, double dt, int64_t* fail_step,
                      double* fail_max);

/* acc /= T(2k) in place, then copy out (gradients.py:315); out == NULL
 * leaves the gradient resident on the device. */
int wo_get_gradient(wo_ctx* ctx, double two_k, void* out);
/* One device field to the host (io.py:29-52 dump layout when
 * first_axis_fastest != 0: the axes reversed on the device, so the bytes are
 * exactly np.ravel(field, order="F") of the reference's dump_field). */
#define WO_FIELD_GAMMA 0
#define WO_FIELD_UPREV 1
#define WO_FIELD_UCUR 2
#define WO_FIELD_ACC 3
int wo_get_field(wo_ctx* ctx, int which, int first_axis_fastest, void* out);

/* One explicit step with an optional sparse (idx, vals) or dense (fp64
 * field) force and a finiteness max (solver.py:173-177, 189-202; the
 * backward replay of solver.py:343-372).  Rotates the window. */
int wo_step(wo_ctx* ctx, int64_t n_force, const int64_t* idx, const double* vals,
            const double* dense_force, int want_max, double* max_out);

/* Literal per-step drop-ins for kernels.apply_step / apply_kernel_increment
 * (kernels.py:136-152) on host arrays with precomputed face weights. */
int wo_apply_step(int ndim, const int64_t* shape, int itemsize, const void* u_prev,
                  const void* u_cur, const void* wf0, const void* wf1, const void* wf2,
                  const void* coef, void* out, int device);
int wo_apply_kernel_increment(int ndim, const int64_t* shape, int itemsize, void* acc,
                              const void* a_old, const void* a_mid, const void* a_new,
                              const void* b_old, const void* b_mid, const void* b_new,
                              double cv, double cg, double inv2dt, double inv2dx, double sdt,
                              int device);

/* Topology-optimisation design chain in fp64 (tato.py:61-140), host arrays
 * in/out.  The filter footprint (offsets [n_fp][ndim], weights [n_fp]) is
 * the non-zero part of the linear-decay kernel in C order; mask may be NULL
 * (everything in the design region).
 *   wo_design_filter  density_filter     (tato.py:78-94, bit-exact sums)
 *   wo_design_project heaviside_project + design masking (tato.py:97-108, 226);
 *                     t_be = tanh(beta*eta), denom = t_be + tanh(beta*(1-eta))
 *   wo_design_chain   chain_rule         (tato.py:124-140) */
int wo_design_filter(int ndim, const int64_t* shape, const double* gamma,
                     const unsigned char* mask, int n_fp, const int* offsets,
                     const double* weights, double* out, int device);
int wo_design_project(int64_t n, const double* g_tilde, double beta, double eta, double t_be,
                      double denom, const unsigned char* mask, double* out, int device);
int wo_design_chain(int ndim, const int64_t* shape, const double* dcdbar, const double* g_tilde,
                    double beta, double eta, double denom, const unsigned char* mask, int n_fp,
                    const int* offsets, const double* weights, double* out, int device);

/* Profiling: on = k > 0 brackets every k-th fused step launch with CUDA
 * events on the context stream (1 = all; sampling keeps the event overhead
 * out of a timed region); wo_stats returns launches and the summed bracketed
 * kernel ms; wo_profile_stats splits the bracketed time and count into
 * single-step launches and two-step passes. */
int wo_set_profiling(wo_ctx* ctx, int on);
int wo_profile_stats(const wo_ctx* ctx, double* single_ms, int64_t* single_n, double* pair_ms,
                     int64_t* pair_n);
int wo_stats(wo_ctx* ctx, int64_t* launches, int64_t* step_launches, double* step_kernel_ms);
int wo_reset_stats(wo_ctx* ctx);
/* Device bytes held by the context (fields + support storage). */
int64_t wo_device_bytes(const wo_ctx* ctx);
/* Solution-sized device buffers the context holds right now: gamma, the
 * window levels (2; 4 once two-step passes ran), the accumulator, the third
 * adjoint level of the reference engine, and the 4 precomputed material
 * fields of the two-step kernel (coef and 3 face arrays).  The history of
 * the reference engine is not included (see wo_device_bytes). */
int wo_field_buffers(const wo_ctx* ctx);
/* Step launches since the last wo_reset_stats that were two-step passes
 * (WO_OPT_TWO_STEP); the rest of wo_stats' step_launches are single steps. */
int64_t wo_pair_launches(const wo_ctx* ctx);
/* CUDA-event marks on the context stream (8 slots) for device timing. */
int wo_timer_mark(wo_ctx* ctx, int idx);
int wo_timer_elapsed(wo_ctx* ctx, int a, int b, double* ms);
int wo_synchronize(wo_ctx* ctx);
/* Device address of the accumulator (C-order field at the context dtype),
 * for collectives that sum per-shot accumulators across GPUs in place. */
void* wo_accumulator_ptr(wo_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* WAVEB200_H */
