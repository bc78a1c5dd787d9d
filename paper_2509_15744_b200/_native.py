"""ctypes binding of the in-tree native library (include/waveb200.h).

There is no CPU fallback: if ``_lib/libwaveb200.so`` is missing or no CUDA
device is visible, every device entry point raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# WAVEB200_LIB selects an alternative in-tree build (kernel-variant A/B runs)
LIB_PATH = os.environ.get("WAVEB200_LIB") or os.path.join(_HERE, "_lib", "libwaveb200.so")

WO_OK, WO_ERR_CONFIG, WO_ERR_UNSTABLE, WO_ERR_BUDGET, WO_ERR_CUDA = 0, 1, 2, 3, 4
WO_RHO_SCALED, WO_ACOUSTIC = 0, 1
WO_SHOT_FWI, WO_SHOT_TATO = 1, 2
WO_FWD_ACCUMULATE, WO_FWD_HISTORY = 1, 2
WO_NO_SOURCE = -(2 ** 63)   # slab backward sweeps: no source

# every symbol declared in include/waveb200.h
EXPORTS = (
    "wo_version", "wo_device_count", "wo_last_error", "wo_create", "wo_create_slab",
    "wo_destroy", "wo_set_material", "wo_set_kernel_coefficients", "wo_set_support",
    "wo_reset_window", "wo_set_window", "wo_get_window", "wo_swap_direction",
    "wo_zero_accumulator", "wo_get_accumulator", "wo_set_accumulator", "wo_sweep_forward",
    "wo_shot_misfit", "wo_get_store", "wo_sweep_backward", "wo_get_gradient", "wo_step",
    "wo_apply_step", "wo_apply_kernel_increment", "wo_set_profiling", "wo_stats",
    "wo_reset_stats", "wo_device_bytes", "wo_field_buffers", "wo_slab_abort", "wo_slab_state", "wo_prepare_two_step", "wo_sweep_adjoint_reference", "wo_free_history", "wo_get_history",
    "wo_design_filter", "wo_design_project", "wo_design_chain", "wo_timer_mark",
    "wo_timer_elapsed", "wo_synchronize", "wo_accumulator_ptr", "wo_set_option",
    "wo_fast_div_active", "wo_sweep_forward_range", "wo_sweep_backward_range",
    "wo_check_maxima", "wo_halo_planes", "wo_exchange_local", "wo_pair_launches", "wo_snapshot",
    "wo_get_field", "wo_opt_init", "wo_opt_step", "wo_opt_get", "wo_design_setup",
    "wo_design_material", "wo_design_gradient", "wo_design_get", "wo_profile_stats",
    "wo_halo_planes_out", "wo_stream", "wo_exchange_local_out", "wo_slab_ghosts", "wo_slab_peers",
    "wo_ipc_export", "wo_ipc_open",
)


class NativeUnavailable(RuntimeError):
    """The CUDA library cannot run here (not built, or no GPU)."""


_lib = None

c_int, c_i64, c_dbl, c_vp = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
P_i64, P_dbl = ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double)

_SIGS = {
    "wo_version": (c_int, []),
    "wo_device_count": (c_int, []),
    "wo_last_error": (ctypes.c_char_p, [c_vp]),
    "wo_create": (c_int, [ctypes.POINTER(c_vp), c_int, P_i64, c_dbl, c_int, c_int]),
    "wo_create_slab": (c_int, [ctypes.POINTER(c_vp), P_i64, c_i64, c_i64, c_dbl, c_int, c_int]),
    "wo_destroy": (None, [c_vp]),
    "wo_set_material": (c_int, [c_vp, c_int, c_vp] + [c_dbl] * 7),
    "wo_set_kernel_coefficients": (c_int, [c_vp] + [c_dbl] * 4),
    "wo_set_support": (c_int, [c_vp, c_i64, c_vp]),
    "wo_reset_window": (c_int, [c_vp]),
    "wo_set_window": (c_int, [c_vp, c_vp, c_vp]),
    "wo_get_window": (c_int, [c_vp, c_vp, c_vp]),
    "wo_swap_direction": (c_int, [c_vp]),
    "wo_zero_accumulator": (c_int, [c_vp]),
    "wo_get_accumulator": (c_int, [c_vp, c_vp]),
    "wo_set_accumulator": (c_int, [c_vp, c_vp]),
    "wo_sweep_forward": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_int, c_dbl, c_dbl,
                                 P_dbl, P_i64, P_dbl]),
    "wo_shot_misfit": (c_int, [c_vp, c_i64, c_int, c_vp] + [c_dbl] * 5
                       + [c_int, c_dbl, P_dbl]),
    "wo_get_store": (c_int, [c_vp, c_i64, c_vp]),
    "wo_sweep_backward": (c_int, [c_vp, c_i64, c_i64, c_vp, c_int, c_int, c_dbl, P_i64, P_dbl]),
    "wo_get_gradient": (c_int, [c_vp, c_dbl, c_vp]),
    "wo_step": (c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_int, P_dbl]),
    "wo_apply_step": (c_int, [c_int, P_i64, c_int] + [c_vp] * 7 + [c_int]),
    "wo_apply_kernel_increment": (c_int, [c_int, P_i64, c_int] + [c_vp] * 7 + [c_dbl] * 5
                                  + [c_int]),
    "wo_set_profiling": (c_int, [c_vp, c_int]),
    "wo_stats": (c_int, [c_vp, P_i64, P_i64, P_dbl]),
    "wo_reset_stats": (c_int, [c_vp]),
    "wo_device_bytes": (c_i64, [c_vp]),
    "wo_field_buffers": (c_int, [c_vp]),
    "wo_slab_abort": (c_int, [c_vp]),
    "wo_slab_state": (c_int, [c_vp, c_vp]),
    "wo_prepare_two_step": (c_int, [c_vp, ctypes.POINTER(c_int)]),
    "wo_sweep_adjoint_reference": (c_int, [c_vp, c_i64, c_dbl, P_i64, P_dbl]),
    "wo_free_history": (c_int, [c_vp]),
    "wo_get_history": (c_int, [c_vp, c_i64, c_i64, c_vp]),
    "wo_design_filter": (c_int, [c_int, P_i64, c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_int]),
    "wo_design_project": (c_int, [c_i64, c_vp, c_dbl, c_dbl, c_dbl, c_dbl, c_vp, c_vp, c_int]),
    "wo_design_chain": (c_int, [c_int, P_i64, c_vp, c_vp, c_dbl, c_dbl, c_dbl, c_vp, c_int,
                                c_vp, c_vp, c_vp, c_int]),
    "wo_timer_mark": (c_int, [c_vp, c_int]),
    "wo_timer_elapsed": (c_int, [c_vp, c_int, c_int, P_dbl]),
    "wo_synchronize": (c_int, [c_vp]),
    "wo_accumulator_ptr": (c_vp, [c_vp]),
    "wo_set_option": (c_int, [c_vp, c_int, c_int]),
    "wo_fast_div_active": (c_int, [c_vp]),
    "wo_sweep_forward_range": (c_int, [c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_vp, c_int,
                                       c_dbl]),
    "wo_sweep_backward_range": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_int, c_int,
                                        c_dbl]),
    "wo_check_maxima": (c_int, [c_vp, c_i64, c_vp]),
    "wo_halo_planes": (c_int, [c_vp] + [ctypes.POINTER(c_vp)] * 4 + [P_i64]),
    "wo_exchange_local": (c_int, [c_vp, c_vp]),
    "wo_pair_launches": (c_i64, [c_vp]),
    "wo_snapshot": (c_int, [c_vp, c_int, c_i64]),
    "wo_get_field": (c_int, [c_vp, c_int, c_int, c_vp]),
    "wo_opt_init": (c_int, [c_vp, c_vp, c_vp, c_int, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl,
                            c_dbl]),
    "wo_opt_step": (c_int, [c_vp, c_int, ctypes.POINTER(c_dbl)]),
    "wo_opt_get": (c_int, [c_vp, c_vp]),
    "wo_design_setup": (c_int, [c_vp, c_vp, c_int, c_vp, c_vp]),
    "wo_design_material": (c_int, [c_vp, c_dbl, c_dbl, c_dbl, c_dbl]),
    "wo_design_gradient": (c_int, [c_vp, c_dbl, c_dbl, c_dbl]),
    "wo_design_get": (c_int, [c_vp, c_int, c_vp]),
    "wo_profile_stats": (c_int, [c_vp, ctypes.POINTER(c_dbl), ctypes.POINTER(c_i64),
                                 ctypes.POINTER(c_dbl), ctypes.POINTER(c_i64)]),
    "wo_halo_planes_out": (c_int, [c_vp] + [ctypes.POINTER(c_vp)] * 4 + [P_i64]),
    "wo_stream": (c_vp, [c_vp]),
    "wo_exchange_local_out": (c_int, [c_vp, c_vp]),
    "wo_slab_ghosts": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "wo_slab_peers": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "wo_ipc_export": (c_int, [c_vp, c_vp, c_vp, P_i64]),
    "wo_ipc_open": (c_int, [c_vp, c_vp, c_i64, ctypes.POINTER(c_vp)]),
}
WO_OPT_FAST_DIV = 1
WO_OPT_PAIR_KERNEL = 2
WO_OPT_TMA_KERNEL = 3
WO_OPT_TWO_STEP = 4
WO_OPT_CLUSTER = 7
WO_OPT_PLANE_PART = 5
WO_OPT_GRAPHS = 6
WO_SNAP_FREE, WO_SNAP_SAVE, WO_SNAP_RESTORE = 0, 1, 2
WO_FIELD_GAMMA, WO_FIELD_UPREV, WO_FIELD_UCUR, WO_FIELD_ACC = 0, 1, 2, 3


def load(require_device=False):
    """Load the library (raises NativeUnavailable when it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is not built; run `python -m paper_2509_15744_b200.build_native` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    if require_device and _lib.wo_device_count() < 1:
        raise NativeUnavailable("no CUDA device visible; the waveb200 path runs on the GPU only")
    return _lib


def ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def shape3(shape):
    return (ctypes.c_int64 * 3)(*(list(shape) + [1] * (3 - len(shape))))
