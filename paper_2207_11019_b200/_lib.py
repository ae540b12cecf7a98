"""ctypes binding of the C ABI in include/pipeplan_b200.h.

The shared library is built in-tree (``make -C paper_2207_11019_b200``, or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PPB_LIB_PATH") or os.path.join(_HERE, "libpipeplan_b200.so")  # override: A/B experiments

PPB_OK = 0
PPB_ERR_INVALID_ARGUMENT = 1
PPB_ERR_RUNTIME = 2
PPB_ERR_OUT_OF_RANGE = 3
PPB_ERR_CUDA = 4
PPB_ERR_NO_DEVICE = 5
PPB_ERR_BUFFER = 6

_lib = None

_i32p = C.POINTER(C.c_int)
_f64p = C.POINTER(C.c_double)
_f32p = C.POINTER(C.c_float)


class TrainConfigC(C.Structure):
    _fields_ = [
        ("alpha0", C.c_double),
        ("decay", C.c_double),
        ("loss", C.c_int),
        ("iterations", C.c_int),
        ("seed", C.c_uint64),
    ]


class OptionsC(C.Structure):
    _fields_ = [
        ("receive_timeout_s", C.c_double),
        ("precision", C.c_int),
        ("multiclass_accuracy", C.c_int),
        ("use_graph", C.c_int),
        ("pipeline_gate", C.c_int),
        ("memory_mode", C.c_int),
        ("merge_backend", C.c_int),
        ("reserved", C.c_int * 6),
    ]


class LayerC(C.Structure):
    _fields_ = [("kind", C.c_int), ("in_units", C.c_int), ("out_units", C.c_int), ("act", C.c_int),
                ("height", C.c_int), ("width", C.c_int), ("ksize", C.c_int), ("pad", C.c_int), ("pool", C.c_int),
                ("res_from", C.c_int), ("pool_kind", C.c_int), ("stride", C.c_int)]


# name -> (restype, argtypes)
_SIGS = {
    "ppb_last_error": (C.c_char_p, []),
    "ppb_version": (C.c_char_p, []),
    "ppb_device_count": (C.c_int, [_i32p]),
    "ppb_split_layer": (C.c_int, [C.c_int, C.c_int, _i32p, C.c_int, C.c_int, _i32p, _i32p, _i32p]),
    "ppb_split_microbatches": (C.c_int, [C.c_int, C.c_int, _i32p]),
    "ppb_build_plan": (C.c_int, [_i32p, _i32p, _f64p, C.c_int, C.c_int, C.c_int, C.c_int, _i32p, C.c_int, _i32p]),
    "ppb_build_staged_plan": (C.c_int, [_i32p, _i32p, _f64p, C.c_int, _i32p, _i32p, C.c_int, C.c_int, _i32p, C.c_int, _i32p]),
    "ppb_build_plan_with_cuts": (C.c_int, [_i32p, _i32p, C.c_int, C.c_int, _i32p, C.c_int, C.c_int, _i32p, C.c_int, _i32p]),
    "ppb_merge_submodules": (C.c_int, [_i32p, C.c_int, _i32p, C.c_int]),
    "ppb_merge_all": (C.c_int, [_i32p, C.c_int]),
    "ppb_validate_plan": (C.c_int, [_i32p, C.c_int, _i32p, _i32p, C.c_int, C.c_int]),
    "ppb_serialize_plan": (C.c_int, [_i32p, C.c_int, C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "ppb_parse_plan": (C.c_int, [C.c_char_p, _i32p, C.c_int, _i32p, C.c_char_p, C.c_size_t]),
    "ppb_default_options": (None, [C.POINTER(OptionsC)]),
    "ppb_default_config": (None, [C.POINTER(TrainConfigC)]),
    "ppb_context_create": (C.c_int, [_i32p, C.c_int, C.POINTER(C.c_void_p)]),
    "ppb_context_destroy": (None, [C.c_void_p]),
    "ppb_train_partitioned": (C.c_int, [C.c_void_p, _i32p, _i32p, C.c_int, _f64p, _f64p, _f64p, _i32p,
                                        C.c_int, _i32p, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(TrainConfigC), C.POINTER(OptionsC),
                                        _f64p, _f64p, _f64p, _f64p]),
    "ppb_session_create": (C.c_int, [C.c_void_p, _i32p, _i32p, C.c_int, _f64p, _f64p, C.c_int, _i32p,
                                     C.c_int, C.c_int, C.c_int, C.POINTER(TrainConfigC),
                                     C.POINTER(OptionsC), C.POINTER(C.c_void_p)]),
    "ppb_session_destroy": (None, [C.c_void_p]),
    "ppb_session_create_layers": (C.c_int, [C.c_void_p, C.POINTER(LayerC), C.c_int, _f64p, _f64p, C.c_int, _i32p,
                                            C.c_int, C.c_int, C.c_int, C.POINTER(TrainConfigC),
                                            C.POINTER(OptionsC), C.POINTER(C.c_void_p)]),
    "ppb_train_partitioned_layers": (C.c_int, [C.c_void_p, C.POINTER(LayerC), C.c_int, _f64p, _f64p, _f64p, _i32p,
                                               C.c_int, _i32p, C.c_int, C.c_int, C.c_int,
                                               C.POINTER(TrainConfigC), C.POINTER(OptionsC),
                                               _f64p, _f64p, _f64p, _f64p]),
    "ppb_session_load_batch": (C.c_int, [C.c_void_p, _f64p, _i32p]),
    "ppb_session_load_batch_f32": (C.c_int, [C.c_void_p, _f32p, _i32p]),
    "ppb_session_step": (C.c_int, [C.c_void_p, C.c_int]),
    "ppb_session_step_host": (C.c_int, [C.c_void_p, _f32p, _i32p, _f64p]),
    "ppb_session_step_host_f64": (C.c_int, [C.c_void_p, _f64p, _i32p, _f64p]),
    "ppb_session_step_host_pipelined": (C.c_int, [C.c_void_p, _f32p, _f64p, _i32p, _f64p]),
    "ppb_session_sync": (C.c_int, [C.c_void_p]),
    "ppb_session_history": (C.c_int, [C.c_void_p, _f64p, _f64p, C.c_int, _i32p]),
    "ppb_session_get_net": (C.c_int, [C.c_void_p, _f64p, _f64p]),
    "ppb_session_memory": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "ppb_session_read_tensor": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, _f64p, C.c_size_t,
                                          C.POINTER(C.c_size_t)]),
    "ppb_session_kernels_per_step": (C.c_int, [C.c_void_p, _i32p]),
    "ppb_session_time_steps": (C.c_int, [C.c_void_p, C.c_int, _f32p]),
    "ppb_session_profile": (C.c_int, [C.c_void_p, C.c_int, _f64p, _i32p, _f64p, C.c_int]),
    "ppb_session_profile_ops": (C.c_int, [C.c_void_p, _i32p, _i32p, _i32p, _f64p, _f64p, C.c_int, _i32p]),
    "ppb_session_profile_starts": (C.c_int, [C.c_void_p, _f64p, _i32p, C.c_int, _i32p]),
    "ppb_session_profile_concurrent": (C.c_int, [C.c_void_p, C.c_int]),
    "ppb_session_op_meta": (C.c_int, [C.c_void_p, _i32p, _i32p, _i32p, C.c_int, _i32p]),
    "ppb_debug_gemm": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_longlong, C.c_int,
                                 C.c_void_p, C.c_int, C.c_int, C.c_longlong, C.c_int,
                                 C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_longlong,
                                 C.c_void_p, C.c_int, C.c_void_p, C.c_longlong, C.c_void_p,
                                 C.c_float, C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "ppb_debug_conv": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_longlong, C.c_int,
                                 C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_longlong, C.c_void_p, C.c_longlong,
                                 C.c_int, C.c_void_p]),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Load (once) and return the ctypes handle; raises if the build is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `make -C {_HERE}` or __graft_entry__.build()"
        )
    handle = C.CDLL(LIB_PATH)
    missing = []
    for name, (res, args) in _SIGS.items():
        try:
            fn = getattr(handle, name)
        except AttributeError:
            missing.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    handle.missing_symbols = tuple(missing)
    _lib = handle
    return _lib


class PipeplanError(RuntimeError):
    pass


def check(code: int) -> None:
    """Raise the reference's exception type for a PPB_* status."""
    if code == PPB_OK:
        return
    msg = lib().ppb_last_error().decode("utf-8", "replace")
    if code == PPB_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if code == PPB_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    raise PipeplanError(msg)
