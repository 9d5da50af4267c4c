"""ctypes binding of libtg.so (include/tg_abi.h).

This is the reference-side binding a maintainer would add to call the C-ABI
from Python.  There is deliberately no fallback: if the
library is missing or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtg.so")

TG_F64, TG_F32 = 0, 1
TG_NODE_OP, TG_LEAF_PARAM, TG_LEAF_INPUT, TG_LEAF_CONST = 0, 1, 2, 3
TG_GATHER_FLAG = 0x80000000
TG_OP_STOPGRAD_MAX = 64

STATUS = {
    0: "TG_OK", 1: "TG_INVALID_ARGUMENT", 2: "TG_CAPACITY", 3: "TG_INVALID_HANDLE",
    4: "TG_INVALID_CHECKPOINT", 5: "TG_DOMAIN", 6: "TG_FORMAT", 7: "TG_IO", 8: "TG_CUDA",
    9: "TG_UNSUPPORTED", 10: "TG_NCCL",
}


class tg_gather(C.Structure):
    _fields_ = [("first_node", C.c_uint32), ("stride", C.c_uint32), ("n_rows", C.c_uint32),
                ("index_col", C.c_uint32), ("offset", C.c_uint32)]


class tg_tape_desc(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_uint32), ("dtype", C.c_int),
        ("op", C.POINTER(C.c_uint8)), ("child_offset", C.POINTER(C.c_uint64)),
        ("child", C.POINTER(C.c_uint32)), ("constant", C.POINTER(C.c_double)),
        ("leaf_class", C.POINTER(C.c_uint8)), ("leaf_index", C.POINTER(C.c_uint32)),
        ("leaf_value", C.POINTER(C.c_double)),
        ("n_gathers", C.c_uint32), ("gathers", C.POINTER(tg_gather)),
        ("root", C.c_uint32), ("n_params", C.c_uint32), ("n_inputs", C.c_uint32),
        ("n_index_inputs", C.c_uint32),
    ]


class tg_checkpoint(C.Structure):
    _fields_ = [("mark", C.c_uint32), ("params", C.c_uint32), ("child_mark", C.c_uint64),
                ("gathers", C.c_uint32), ("reserved", C.c_uint32)]


class tg_rec_stats(C.Structure):
    _fields_ = [("size", C.c_uint32), ("peak_nodes", C.c_uint32), ("child_pool_size", C.c_uint64),
                ("peak_children", C.c_uint64), ("peak_arena_bytes", C.c_uint64), ("max_arity", C.c_uint32),
                ("n_params", C.c_uint32)]


class tg_model_args(C.Structure):
    _fields_ = [("dims", C.c_uint32 * 8), ("dtype", C.c_int)]


class tg_program_info(C.Structure):
    _fields_ = [
        ("n_params", C.c_uint32), ("n_inputs", C.c_uint32), ("n_index_inputs", C.c_uint32),
        ("n_sample_nodes", C.c_uint32), ("n_uniform_nodes", C.c_uint32),
        ("n_dense_groups", C.c_uint32), ("n_fwd_instr", C.c_uint32), ("n_bwd_instr", C.c_uint32),
        ("n_edges", C.c_uint64), ("tile_samples", C.c_uint32), ("smem_bytes", C.c_uint32),
        ("storage", C.c_uint32), ("dtype", C.c_int), ("n_attn_heads", C.c_uint32), ("n_layer_norms", C.c_uint32),
        ("fused_mlp", C.c_uint32),
    ]


class TgError(RuntimeError):
    """A tg_status other than TG_OK; .status holds the enum name."""

    def __init__(self, status: int, message: str):
        self.status = STATUS.get(status, str(status))
        super().__init__(f"{self.status}: {message}")


class DomainError(TgError, ValueError):
    """Per-sample operator domain violation (reference std::domain_error)."""


class InvalidArgument(TgError, ValueError):
    """Reference std::invalid_argument."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
            "there is no CPU fallback for the gradient-oracle path")
    lib = C.CDLL(LIB_PATH)
    P, u8, u32, u64, i32, i64, sz = C.c_void_p, C.c_uint8, C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_size_t
    st = C.c_int
    sig = {
        "tg_last_error": (C.c_char_p, []),
        "tg_status_name": (C.c_char_p, [st]),
        "tg_op_name": (C.c_char_p, [u8]),
        "tg_recorder_new": (st, [st, sz, C.POINTER(P)]),
        "tg_recorder_free": (None, [P]),
        "tg_rec_param": (st, [P, C.c_double, C.POINTER(u32)]),
        "tg_rec_input": (st, [P, u32, C.c_double, C.POINTER(u32)]),
        "tg_rec_const": (st, [P, C.c_double, C.POINTER(u32)]),
        "tg_rec_gather": (st, [P, u32, u32, u32, u32, u32, i32, C.POINTER(u32)]),
        "tg_rec_op": (st, [P, u8, C.POINTER(u32), u32, C.c_double, C.POINTER(u32)]),
        "tg_rec_value": (st, [P, u32, C.POINTER(C.c_double)]),
        "tg_rec_set_root": (st, [P, u32]),
        "tg_rec_describe": (st, [P, C.POINTER(tg_tape_desc)]),
        "tg_recorder_new_fixed": (st, [st, sz, sz, C.POINTER(P)]),
        "tg_rec_checkpoint": (st, [P, C.POINTER(tg_checkpoint)]),
        "tg_rec_rewind": (st, [P, C.POINTER(tg_checkpoint)]),
        "tg_rec_get_stats": (st, [P, C.POINTER(tg_rec_stats)]),
        "tg_build_model": (st, [st, C.POINTER(tg_model_args), u64, C.POINTER(P)]),
        "tg_synth_batch": (st, [st, C.POINTER(tg_model_args), u64, sz, P, C.POINTER(i32)]),
        "tg_synth_ctr": (st, [st, C.POINTER(tg_model_args), u64, u64, sz, P, C.POINTER(i32)]),
        "tg_synth_ctr_device": (st, [st, C.POINTER(tg_model_args), u64, u64, sz, P, C.POINTER(i32), P]),
        "tg_compile": (st, [C.POINTER(tg_tape_desc), C.POINTER(P)]),
        "tg_program_info_get": (st, [P, C.POINTER(tg_program_info)]),
        "tg_program_order": (st, [P, C.POINTER(C.POINTER(u32)), C.POINTER(u32)]),
        "tg_workspace_size": (st, [P, sz, C.POINTER(sz)]),
        "tg_set_memory_budget": (st, [P, sz]),
        "tg_chunk_samples": (st, [P, sz, C.POINTER(sz)]),
        "tg_forward_backward": (st, [P, P, P, sz, P, P, P, P, P, sz, P]),
        "tg_gd_update": (st, [P, P, P, C.c_double, sz, P]),
        "tg_train_step": (st, [P, P, P, sz, P, P, P, C.c_double, P, sz, P]),
        "tg_check_device_error": (st, [P, P, C.POINTER(i64), C.POINTER(u32)]),
        "tg_launch_count": (u64, [P]),
        "tg_gemm": (st, [st, C.c_int, u32, u32, u32, P, sz, C.c_int, P, sz, C.c_int, P, sz, C.c_int, P]),
        "tg_program_jit": (st, [P, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p), C.POINTER(C.c_double)]),
        "tg_profile_enable": (st, [P, C.c_int]),
        "tg_profile_read": (st, [P, C.POINTER(C.c_double), C.POINTER(u64)]),
        "tg_program_free": (None, [P]),
        "tg_pipeline_new": (st, [P, sz, P, P, C.POINTER(P)]),
        "tg_pipeline_step": (st, [P, P, P, P, C.c_double]),
        "tg_pipeline_join": (st, [P, P]),
        "tg_pipeline_sync": (st, [P]),
        "tg_pipeline_grad_sum": (st, [P, C.POINTER(P)]),
        "tg_pipeline_free": (None, [P]),
        "tg_host_alloc": (st, [sz, C.POINTER(P)]),
        "tg_host_free": (None, [P]),
        "tg_range_bytes": (sz, [st, sz, C.c_int]),
        "tg_save_range": (st, [st, P, P, sz, P, sz, C.POINTER(sz)]),
        "tg_load_range": (st, [st, P, P, sz, P, sz]),
        "tg_snapshot_bytes": (sz, [st, sz, C.c_int]),
        "tg_save_snapshot": (st, [st, P, P, sz, P, sz, C.POINTER(sz)]),
        "tg_load_snapshot": (st, [P, sz, C.c_int, P, P, sz, C.POINTER(sz), C.POINTER(C.c_int)]),
        "tg_nccl_get_unique_id": (st, [P]),
        "tg_nccl_comm_init": (st, [C.c_int, P, C.c_int, C.POINTER(P)]),
        "tg_nccl_comm_destroy": (st, [P]),
        "tg_nccl_version": (C.c_int, []),
        "tg_allreduce_gd_step": (st, [P, P, P, C.c_double, sz, P, P]),
        "tg_window_create": (st, [P, st, sz, C.c_int, C.POINTER(P)]),
        "tg_window_destroy": (st, [P]),
        "tg_window_buffer": (P, [P]),
        "tg_window_multimem": (C.c_int, [P]),
        "tg_window_allreduce_gd": (st, [P, P, C.c_double, sz, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    if status == 0:
        return
    msg = lib.tg_last_error().decode()
    if status == 5:
        raise DomainError(status, msg)
    if status == 1:
        raise InvalidArgument(status, msg)
    raise TgError(status, msg)


def header_symbols() -> list[str]:
    """Function names declared in include/tg_abi.h."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "tg_abi.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(tg_\w+)\s*\(", text, re.M)))
