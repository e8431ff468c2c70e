"""ctypes binding of include/asnn_dev.h (libasnn_b200.so, built in-tree).

The product path has no fallback: if the shared object is missing or has no
GPU behind it, calls raise (BackendUnavailable / OSError) instead of
computing anything on the host.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "libasnn_b200.so"

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)

ASNN_OK = 0
ASNN_E_UNAVAILABLE = 1
ASNN_E_ARITY = 2
ASNN_E_UNASSIGNED_OUTPUT = 3
ASNN_E_LAYER_RANGE = 4
ASNN_E_INVALID = 5
ASNN_E_CUDA = 6
ASNN_E_OOM = 7
ASNN_E_INFEASIBLE = 8
ASNN_E_PARSE = 9
ASNN_E_VALIDATION = 10
ASNN_E_IO = 11
UNASSIGNED = 0xFFFFFFFF


class NetworkDesc(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_uint32), ("nodes", u32p),
        ("n_inputs", C.c_uint32), ("inputs", u32p),
        ("n_outputs", C.c_uint32), ("outputs", u32p),
        ("n_connections", C.c_uint64),
        ("source", u32p), ("target", u32p), ("weight", f32p),
    ]


class LayoutDesc(C.Structure):
    _fields_ = [
        ("total_layers", C.c_uint32), ("layer_offsets", u32p),
        ("node_count", C.c_uint32), ("node_ids", u32p),
        ("row_ptr", u64p), ("in_nodes", u32p), ("in_weights", f32p),
        ("n_inputs", C.c_uint32), ("input_order", u32p),
        ("id_bound", C.c_uint32),
        ("n_outputs", C.c_uint32), ("outputs", u32p),
    ]


class EvalDims(C.Structure):
    _fields_ = [
        ("total_layers", C.c_uint32), ("node_count", C.c_uint32),
        ("sensor_count", C.c_uint32), ("id_bound", C.c_uint32),
        ("edge_count", C.c_uint64),
    ]


class EvalStage(C.Structure):
    _fields_ = [
        ("layer_offsets", u32p), ("node_ids", u32p), ("row_ptr", u32p),
        ("in_nodes", u32p), ("in_weights", f32p), ("sensor_inputs", f32p),
    ]


class LayoutInfo(C.Structure):
    _fields_ = [
        ("n_networks", C.c_uint32), ("total_layers", C.c_uint32),
        ("node_count", C.c_uint32), ("edge_count", C.c_uint64),
        ("dropped_connections", C.c_uint64), ("id_bound", C.c_uint32),
        ("n_inputs", C.c_uint32), ("n_outputs", C.c_uint32),
        ("max_layer_width", C.c_uint32), ("max_in_degree", C.c_uint32),
    ]


class Timings(C.Structure):
    _fields_ = [(n, C.c_float) for n in
                ("upload_ms", "required_ms", "segment_ms", "flatten_ms", "activate_ms")]


# name -> (restype, argtypes); every symbol include/asnn_dev.h declares.
PROTOTYPES = {
    "asnn_dev_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "asnn_dev_open": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "asnn_dev_close": (None, [C.c_void_p]),
    "asnn_dev_last_error": (C.c_char_p, [C.c_void_p]),
    "asnn_dev_version": (C.c_char_p, []),
    "asnn_dev_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "asnn_dev_get_stream": (C.c_void_p, [C.c_void_p]),
    "asnn_dev_synchronize": (C.c_int, [C.c_void_p]),
    "asnn_dev_set_heavy_threshold": (C.c_int, [C.c_void_p, C.c_uint32]),
    "asnn_dev_set_sweep_mode": (C.c_int, [C.c_void_p, C.c_uint32]),
    "asnn_dev_last_timings": (C.c_int, [C.c_void_p, C.POINTER(Timings)]),
    "asnn_dev_compute_required": (C.c_int, [C.c_void_p, C.POINTER(NetworkDesc), u8p]),
    "asnn_dev_segment": (C.c_int, [C.c_void_p, C.POINTER(NetworkDesc), u8p, u32p, u32p]),
    "asnn_dev_build_layout": (C.c_int, [C.c_void_p, C.POINTER(NetworkDesc), C.POINTER(C.c_void_p)]),
    "asnn_dev_build_population": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(NetworkDesc),
                                            C.POINTER(C.c_void_p)]),
    "asnn_dev_upload_layout": (C.c_int, [C.c_void_p, C.POINTER(LayoutDesc), C.POINTER(C.c_void_p)]),
    "asnn_dev_free_layout": (None, [C.c_void_p]),
    "asnn_dev_layout_info": (C.c_int, [C.c_void_p, C.POINTER(LayoutInfo)]),
    "asnn_dev_layer_slice": (C.c_int, [C.c_void_p, C.c_uint32, u32p, u32p]),
    "asnn_dev_network_info": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(LayoutInfo)]),
    "asnn_dev_layout_download": (C.c_int, [C.c_void_p, C.c_uint32, u32p, u32p, u64p, u32p, f32p, u32p]),
    "asnn_dev_activate": (C.c_int, [C.c_void_p, f32p, C.c_uint32, C.c_uint64, f32p, f32p]),
    "asnn_eval_buf_create": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "asnn_eval_buf_free": (None, [C.c_void_p]),
    "asnn_eval_buf_stage": (C.c_int, [C.c_void_p, C.POINTER(EvalDims), C.POINTER(EvalStage)]),
    "asnn_eval_buf_run": (C.c_int, [C.c_void_p, f32p]),
    "asnn_eval_buf_mode": (C.c_int, [C.c_void_p, u32p]),
    "asnn_dev_eval_layout": (C.c_int, [C.c_void_p, C.POINTER(LayoutDesc), f32p, C.c_uint64, f32p]),
    "asnn_dev_activate_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p]),
    "asnn_dev_server_start": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p)]),
    "asnn_dev_server_activate": (C.c_int, [C.c_void_p, f32p, C.c_uint32, C.c_uint64, f32p]),
    "asnn_dev_server_stop": (None, [C.c_void_p]),
    "asnn_dev_server_timings": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "asnn_dev_activate_plan": (C.c_int, [C.c_void_p, C.c_uint32, u32p, u64p, u64p]),
    "asnn_dev_profile_sweep": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, f32p, u32p]),
    "asnn_dev_sweep_kind": (C.c_int, [C.c_void_p, C.c_uint32, u32p]),
    "asnn_dev_debug_write_counts": (C.c_int, [C.c_void_p, C.c_uint32, u32p]),
    "asnn_dev_sigmoid_selfcheck": (C.c_int, [C.c_void_p, u64p, u64p]),
    "asnn_dev_sigmoid32": (C.c_int, [C.c_void_p, f32p, f32p, C.c_uint64]),
    "asnn_dev_latency_probe": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "asnn_gen_reference": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                                     C.c_float, C.c_float, C.c_uint64, C.POINTER(C.c_void_p)]),
    "asnn_gen_max_connections": (C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
    "asnn_gen_mlp": (C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64, C.POINTER(C.c_void_p)]),
    "asnn_gen_powerlaw": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                    C.c_double, C.c_uint64, C.POINTER(C.c_void_p)]),
    "asnn_dev_parse_network": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.POINTER(C.c_void_p), u32p]),
    "asnn_dev_load_layout": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.POINTER(C.c_void_p), u32p]),
    "asnn_dev_validate": (C.c_int, [C.c_void_p, C.POINTER(NetworkDesc), C.c_char_p, C.c_uint64, u32p]),
    "asnn_dev_normalize": (C.c_int, [C.c_void_p, C.POINTER(NetworkDesc), C.POINTER(C.c_void_p)]),
    "asnn_dev_read_network": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p), u32p]),
    "asnn_dev_parse_weights": (C.c_int, [C.c_void_p, C.c_char_p, u64p, C.c_uint64, f32p, u8p]),
    "asnn_group_open": (C.c_int, [C.POINTER(C.c_int), C.c_uint32, C.POINTER(C.c_void_p)]),
    "asnn_group_close": (None, [C.c_void_p]),
    "asnn_group_last_error": (C.c_char_p, [C.c_void_p]),
    "asnn_group_info": (C.c_int, [C.c_void_p, u32p, u32p]),
    "asnn_group_gather_note": (C.c_char_p, [C.c_void_p]),
    "asnn_group_device": (C.c_void_p, [C.c_void_p, C.c_uint32]),
    "asnn_group_build_layout": (C.c_int, [C.c_void_p, C.POINTER(NetworkDesc), C.POINTER(C.c_void_p)]),
    "asnn_group_upload_layout": (C.c_int, [C.c_void_p, C.POINTER(LayoutDesc), C.POINTER(C.c_void_p)]),
    "asnn_group_build_population": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(NetworkDesc),
                                              C.POINTER(C.c_void_p)]),
    "asnn_group_layout_member": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p)]),
    "asnn_group_shard": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, u32p, u64p, u64p, u64p, u64p]),
    "asnn_group_activate": (C.c_int, [C.c_void_p, f32p, C.c_uint32, C.c_uint64, f32p, f32p]),
    "asnn_group_stage_inputs": (C.c_int, [C.c_void_p, f32p, C.c_uint32, C.c_uint64]),
    "asnn_group_sweep": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_float)]),
    "asnn_group_read_outputs": (C.c_int, [C.c_void_p, f32p]),
    "asnn_group_free_layout": (None, [C.c_void_p]),
    "asnn_comm_unique_id": (C.c_int, [u8p]),
    "asnn_dev_comm_init": (C.c_int, [C.c_void_p, u8p, C.c_int, C.c_int]),
    "asnn_dev_allgather": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, u64p]),
    "asnn_dev_gen_mlp": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_double, C.c_uint64,
                                   C.POINTER(C.c_void_p)]),
    "asnn_dev_gen_mlp_layout": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_double, C.c_uint64,
                                          C.POINTER(C.c_void_p)]),
    "asnn_dev_gen_powerlaw": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.c_uint64, C.c_double, C.c_uint64, C.POINTER(C.c_void_p)]),
    "asnn_dev_gen_powerlaw_layout": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                               C.c_uint64, C.c_double, C.c_uint64, C.POINTER(C.c_void_p)]),
    "asnn_corpus_desc": (C.c_int, [C.c_void_p, C.POINTER(NetworkDesc)]),
    "asnn_corpus_free": (None, [C.c_void_p]),
}

_lib = None


def load() -> C.CDLL:
    """Load libasnn_b200.so once; raises OSError if it was not built."""
    global _lib
    if _lib is None:
        path = os.environ.get("ASNN_B200_LIB", str(LIB_PATH))
        if not os.path.exists(path):
            raise OSError(f"{path} is missing: run __graft_entry__.build() "
                          "(make -C paper_2005_04347_b200/csrc)")
        lib = C.CDLL(path)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        # asnn_dev_activate taking raw addresses (pinned / mapped buffers held
        # by the caller as integers): no per-call ctypes casts
        lib.activate_addr = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64,
                                        C.c_void_p, C.c_void_p)(("asnn_dev_activate", lib))
        lib.server_activate_addr = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64,
                                               C.c_void_p)(("asnn_dev_server_activate", lib))
        _lib = lib
    return _lib


def ptr(a, ctype):
    """ctypes pointer to a contiguous numpy array (None for None)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))
