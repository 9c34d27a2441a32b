"""ctypes loader for libmgcuda.so (the C-ABI in include/mgcuda.h).

The shared library is built in-tree (`make -C paper_2309_15676_b200/csrc`,
or __graft_entry__.build()).  There is no fallback: if it is missing or no
sm_100 device is visible, load()/Context() raise.
"""
import ctypes as C
import os

from . import _abi

HERE = os.path.dirname(os.path.abspath(__file__))
# MG_LIB overrides the library path (A/B timing of two builds only)
LIB_PATH = os.environ.get("MG_LIB") or os.path.join(HERE, "libmgcuda.so")

_vp = C.c_void_p
_lib = None


class MgError(RuntimeError):
    """Raised for a non-zero mg_status; .status holds the code."""

    def __init__(self, status, msg):
        super().__init__(f"[mg_status {status}] {msg}")
        self.status = status


class InvalidArgument(MgError, ValueError):      # std::invalid_argument
    pass


class LogicError(MgError):                       # std::logic_error
    pass


class DomainError(MgError, ArithmeticError):     # std::domain_error
    pass


_EXC = {_abi.MG_EINVAL: InvalidArgument, _abi.MG_ELOGIC: LogicError,
        _abi.MG_EDOMAIN: DomainError}


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libmgcuda.so not built ({LIB_PATH}); run "
                           "`make -C paper_2309_15676_b200/csrc` — there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    sig = {
        "mg_last_error": (C.c_char_p, []),
        "mg_abi_version": (C.c_int, []),
        "mg_set_option": (C.c_int, [C.c_char_p, C.c_int64]),
        "mg_config_defaults": (None, [P(_abi.ExperimentConfigC)]),
        "mg_config_validate": (C.c_int, [P(_abi.ExperimentConfigC)]),
        "mg_ctx_create": (C.c_int, [C.c_int, _vp, P(_vp)]),
        "mg_ctx_destroy": (C.c_int, [_vp]),
        "mg_ctx_synchronize": (C.c_int, [_vp]),
        "mg_ctx_stream": (_vp, [_vp]),
        "mg_ctx_launch_count": (C.c_int64, [_vp]),
        "mg_malloc": (C.c_int, [_vp, C.c_size_t, P(_vp)]),
        "mg_free": (C.c_int, [_vp, _vp]),
        "mg_copy_to_device": (C.c_int, [_vp, _vp, _vp, C.c_size_t]),
        "mg_copy_to_host": (C.c_int, [_vp, _vp, _vp, C.c_size_t]),
        "mg_copy_device": (C.c_int, [_vp, _vp, _vp, C.c_size_t]),
        "mg_fill": (C.c_int, [_vp, C.c_int32, C.c_int64, _vp, C.c_double]),
        "mg_mix64": (C.c_uint64, [C.c_uint64]),
        "mg_stream_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
        "mg_mt64_create": (C.c_int, [_vp, C.c_int32, _vp, P(_vp)]),
        "mg_mt64_destroy": (C.c_int, [_vp]),
        "mg_mt64_draw": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, _vp]),
        "mg_mt64_jump": (C.c_int, [_vp, _vp, C.c_uint64]),
        "mg_mt64_split": (C.c_int, [_vp, C.c_uint64, C.c_int32, C.c_uint64, P(_vp)]),
        "mg_mt64_jump_polynomial": (C.c_int, [C.c_uint64, _vp, P(C.c_int32)]),
        "mg_moment2_step": (C.c_int, [_vp, C.c_int32, C.c_int64, P(_abi.Moment2Scalars), _vp,
                                      _vp]),
        "mg_meta_step": (C.c_int, [_vp, C.c_int32, C.c_int64, P(_abi.MetaParams), C.c_int32] +
                         [_vp] * 8),
        "mg_adam_step": (C.c_int, [_vp, C.c_int32, C.c_int64, P(_abi.AdamScalars)] + [_vp] * 4),
        "mg_meta_update": (C.c_int, [_vp, C.c_int32, C.c_int64, P(_abi.MetaUpdateArgs)] +
                           [_vp] * 9 + [_vp, P(_abi.MetaExtras)]),
        "mg_meta_update_fixed": (C.c_int, [_vp, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                           P(_abi.MetaUpdateArgs)] + [_vp] * 8 +
                                 [_vp, P(_abi.MetaExtras)]),
        "mg_meta_update_fixed_touch": (C.c_int, [_vp, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                                 P(_abi.MetaUpdateArgs)] + [_vp] * 9 +
                                       [_vp, P(_abi.MetaExtras)]),
        "mg_shared_meta_update": (C.c_int, [_vp, C.c_int32, C.c_int64, C.c_int64, C.c_int32,
                                            P(_abi.MetaUpdateArgs), _vp, _vp, _vp] +
                                  [_vp] * 7 + [_vp]),
        "mg_adam_update": (C.c_int, [_vp, C.c_int32, C.c_int64, P(_abi.AdamScalars), C.c_int32,
                                     C.c_double] + [_vp] * 7),
        "mg_scalars_read": (C.c_int, [_vp, _vp, P(_abi.UpdateScalars)]),
        "mg_scalars_write": (C.c_int, [_vp, _vp, P(_abi.UpdateScalars)]),
        "mg_minirender_generate": (C.c_int, [_vp, C.c_int32, C.c_uint64, C.c_double, _vp, _vp]),
        "mg_minirender_sample_pair": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32] +
                                      [_vp] * 8),
        "mg_exprate_sample_pair": (C.c_int, [_vp, C.c_int32, C.c_double, C.c_int32] + [_vp] * 6),
        "mg_multnoise_sample_pair": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_double,
                                               C.c_int32] + [_vp] * 7),
        "mg_minirender_meta_iteration": (C.c_int, [_vp, C.c_int32, C.c_int64, P(_abi.RenderArgs)] +
                                         [_vp] * 10 + [_vp, _vp, _vp]),
        "mg_quad_render": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _vp,
                                     C.c_int32, C.c_uint64, C.c_uint32, _vp, _vp]),
        "mg_quad_sample_pair": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _vp,
                                          _vp, _vp, _vp, C.c_uint64, C.c_uint32, C.c_uint32,
                                          C.c_int32, C.c_int32, _vp, _vp, _vp, _vp]),
        "mg_helix_render": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _vp, _vp,
                                      _vp, _vp, _vp, C.c_int32, C.c_uint64, _vp]),
        "mg_helix_sample_pair": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _vp,
                                           _vp, _vp, _vp, _vp, _vp, _vp, C.c_uint64, C.c_uint32,
                                           C.c_int32, C.c_int32, _vp, _vp, _vp, _vp]),
        "mg_run_replicates": (C.c_int, [_vp, P(_abi.ExperimentConfigC), C.c_int32, C.c_int32,
                                        _vp, P(_abi.RunSeriesC), _vp]),
        "mg_run_replicates_full": (C.c_int, [_vp, P(_abi.ExperimentConfigC), C.c_int32,
                                             C.c_int32, _vp, P(_abi.RunSeriesC), _vp, _vp]),
        "mg_mt64_set_state": (C.c_int, [_vp, _vp, C.c_int32, _vp, C.c_int32]),
        "mg_mt64_get_state": (C.c_int, [_vp, _vp, C.c_int32, _vp, _vp]),
        "mg_meshscene_create": (C.c_int, [_vp, C.c_int32, _vp, _vp, C.c_int32, C.c_int32,
                                          C.c_int32, _vp]),
        "mg_meshscene_destroy": (C.c_int, [_vp]),
        "mg_meshscene_info": (C.c_int, [_vp, _vp, _vp, _vp]),
        "mg_meshscene_set_prev_reuse": (C.c_int, [_vp, C.c_int32]),
        "mg_meshscene_set_touch_map": (C.c_int, [_vp, _vp]),
        "mg_meshscene_queue_counts": (C.c_int, [_vp, _vp, C.c_int32, _vp]),
        "mg_ctx_set_iteration_offset": (C.c_int, [_vp, _vp]),
        "mg_iteration_offset_add": (C.c_int, [_vp, _vp, C.c_uint32]),
        "mg_meshscene_intersect": (C.c_int, [_vp, _vp, C.c_int32, _vp, _vp, _vp]),
        "mg_meshscene_render": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_int32, _vp,
                                          C.c_int32, C.c_uint64, _vp, _vp]),
        "mg_meshscene_sample_pair": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_int32, _vp,
                                               _vp, _vp, _vp, C.c_uint64, C.c_uint32, C.c_int32,
                                               C.c_int32, C.c_int32, _vp, _vp, _vp, _vp]),
        "mg_meshscene_sample_pair_sharded": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_int32,
                                                       _vp, _vp, _vp, _vp, C.c_uint64,
                                                       C.c_uint32, C.c_int32, C.c_int32,
                                                       C.c_int32, C.c_int32, _vp, C.c_int64,
                                                       _vp]),
        "mg_fixed_finalize": (C.c_int, [_vp, C.c_int32, C.c_int64, _vp, _vp, _vp]),
        "mg_debug_selftest": (C.c_int, [_vp]),
        "mg_mt_stream_probe": (C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_int64, _vp, _vp]),
        "mg_host_malloc": (C.c_int, [C.c_size_t, _vp]),
        "mg_host_free": (C.c_int, [_vp]),
        "mg_copy_async": (C.c_int, [_vp, _vp, _vp, C.c_size_t]),
        "mg_compute_alpha": (C.c_int, [_vp, C.c_int32, C.c_int64, _vp, _vp, _vp, _vp, C.c_double,
                                       _vp]),
        "mg_scalar_op": (C.c_int, [_vp, C.c_int32, C.c_int64, _vp, C.c_double, C.c_int32, _vp]),
        "mg_aggregate_series": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, _vp, _vp, _vp,
                                          _vp]),
        "mg_run_experiment_stats": (C.c_int, [_vp, P(_abi.ExperimentConfigC), C.c_int32,
                                              C.c_int32, _vp, _vp, _vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    if L.mg_abi_version() != 1:
        raise RuntimeError("libmgcuda ABI version mismatch")
    _lib = L
    return L


def check(status):
    """Map an mg_status to the reference's exception types (include/mgcuda.h)."""
    if status == _abi.MG_OK:
        return
    msg = load().mg_last_error().decode(errors="replace")
    raise _EXC.get(status, MgError)(status, msg)
