"""B200-native Multiverse Attention hot path (host bindings over the C-ABI in include/multiverse_b200.h).

The product is libmvb200.so (CUDA kernels for sm_100a + the C-ABI). This package only binds
it with ctypes and mirrors the reference's proj/core interface names for this path:

    dag.build_visibility  <- multiverse::dag::build_visibility / build_mask (dag.hpp:104-110)
    kv.PagedStore         <- multiverse::kv::RadixStore (kvcache.hpp:60-101)
    attention.decode      <- attention core of ToyModel::step (toy_model.cpp:121-157)
    attention.prefill     <- attention inside ToyModel::forward (toy_model.cpp:174-202)
    toy.ToyModel          <- ToyModel forward / engine::run_forced around those kernels (configs[0])
    interp.TagInterpreter <- the engine's per-lane feed_interpreter (engine.cpp:323-415)

There is no CPU fallback: importing fails loudly when the library is missing, and every
call runs on the GPU.
"""
from __future__ import annotations

import ctypes
import os
import pathlib

PKG = pathlib.Path(__file__).resolve().parent
LIB_PATH = pathlib.Path(os.environ["MV_LIB"]) if os.environ.get("MV_LIB") else PKG / "libmvb200.so"  # MV_LIB: A/B builds


class MvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class CacheError(MvError):
    """kv::CacheError (kvcache.hpp:32-41). kind in {UnknownHandle, DoubleRelease, CapacityExceeded,
    BranchNotDescendant}."""

    KINDS = {1: "UnknownHandle", 2: "DoubleRelease", 3: "CapacityExceeded", 4: "BranchNotDescendant"}

    @property
    def kind(self) -> str:
        return self.KINDS[self.status]


class ParseError(MvError):
    """grammar::ParseError (grammar.hpp:136-152). kind in {MalformedStructure, CountMismatch}."""

    KINDS = {5: "MalformedStructure", 6: "CountMismatch"}

    @property
    def kind(self) -> str:
        return self.KINDS[self.status]


# mv_engine_label_fn: token id of a path index label text
LABEL_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_char_p)


def _load():
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback for the Multiverse hot path)")
    L = ctypes.CDLL(str(LIB_PATH))
    P, i32, i64, u64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t
    sigs = {
        "mv_last_error": ([], ctypes.c_char_p),
        "mv_version": ([], ctypes.c_char_p),
        "mv_visibility_workspace_size": ([P, i32], sz),
        "mv_visibility": ([P, P, i32, i32, P, P, P, P, P, sz, P], ctypes.c_int),
        "mv_training_batch": ([P, P, i32, i32, i32, P, P, P, P, P, P, sz, P], ctypes.c_int),
        "mv_mask_packed": ([P, i32, i32, i32, i32, P, P], ctypes.c_int),
        "mv_tile_map": ([P, i32, i32, i32, P, P, P, P], ctypes.c_int),
        "mv_kv_store_create": ([P, P], ctypes.c_int),
        "mv_kv_store_destroy": ([P], ctypes.c_int),
        "mv_kv_set_stream": ([P, P], ctypes.c_int),
        "mv_kv_planes": ([P, i32, P, P], ctypes.c_int),
        "mv_kv_create": ([P, P], ctypes.c_int),
        "mv_kv_extend": ([P, u64, P, i64, P, P], ctypes.c_int),
        "mv_kv_fork": ([P, u64, i32, P], ctypes.c_int),
        "mv_kv_merge": ([P, u64, P, i32, P], ctypes.c_int),
        "mv_kv_release": ([P, u64], ctypes.c_int),
        "mv_kv_length": ([P, u64, P], ctypes.c_int),
        "mv_kv_stats_get": ([P, P], ctypes.c_int),
        "mv_kv_resolve": ([P, u64, P], ctypes.c_int),
        "mv_kv_resolve_payloads": ([P, u64, P], ctypes.c_int),
        "mv_kv_resolve_slots": ([P, u64, P], ctypes.c_int),
        "mv_kv_append": ([P, P, i32, P, P, i32, P, P], ctypes.c_int),
        "mv_kv_write_last": ([P, P, i32, P, i32, P, P], ctypes.c_int),
        "mv_kv_append_many": ([P, u64, i64, P, P, i32, P, P], ctypes.c_int),
        "mv_kv_gather_kv": ([P, u64, i32, P, P], ctypes.c_int),
        "mv_attn_decode": ([P, i32, P, i32, i32, P, P, P, i32], ctypes.c_int),
        "mv_attn_decode_plan_info": ([P, P], ctypes.c_int),
        "mv_attn_decode_kernel_timing": ([P, i32, P, P], ctypes.c_int),
        "mv_prefill_workspace_size": ([i32, i32, i32], sz),
        "mv_attn_prefill": ([P, P, P, P, P, i32, i32, i32, i32, ctypes.c_double, P, i32, P, sz, P], ctypes.c_int),
        "mv_prefill_workspace_size_hd": ([i32, i32, i32, i32], sz),
        "mv_attn_prefill_hd": ([P, P, P, P, P, i32, i32, i32, i32, i32, ctypes.c_double, P, i32, P, sz, P],
                               ctypes.c_int),
        "mv_attn_head_dim": ([i32], i32),
        "mv_kv_write_range": ([P, u64, i64, i64, P, i32, P, P], ctypes.c_int),
        "mv_toy_weight_count": ([P], sz),
        "mv_toy_create": ([P, P, P], ctypes.c_int),
        "mv_toy_destroy": ([P], ctypes.c_int),
        "mv_toy_get_config": ([P, P], ctypes.c_int),
        "mv_toy_vocab": ([P], i32),
        "mv_toy_step": ([P, P, P, i32, P, P, P, P, P], ctypes.c_int),
        "mv_toy_load_context": ([P, P, u64, P, i64], ctypes.c_int),
        "mv_toy_forward": ([P, P, i32, P, P, i32, P, P, P], ctypes.c_int),
        "mv_argmax_rows": ([P, i32, i32, P, P], ctypes.c_int),
        "mv_engine_run_forced": ([P, P, i32, P, P, P, P, i64, P], ctypes.c_int),
        "mv_engine_run_batch": ([P, P, P, i32, P, P, P, P, i64, P], ctypes.c_int),
        "mv_engine_run_free": ([P, P, i32, i32, P, LABEL_FN, P, P, P, i64, P], ctypes.c_int),
        "mv_interp_init": ([P, i32, P, P], ctypes.c_int),
        "mv_interp_feed": ([P, i32, P, i32, P, P, P, P, P], ctypes.c_int),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


lib = _load()

# C-ABI symbols declared in include/multiverse_b200.h (checked by tests/test_capi.py)
EXPORTED = (
    "mv_last_error", "mv_version", "mv_visibility_workspace_size", "mv_visibility", "mv_training_batch",
    "mv_mask_packed", "mv_tile_map",
    "mv_kv_store_create", "mv_kv_store_destroy", "mv_kv_set_stream", "mv_kv_planes", "mv_kv_create", "mv_kv_extend",
    "mv_kv_fork", "mv_kv_merge", "mv_kv_release", "mv_kv_length", "mv_kv_stats_get", "mv_kv_resolve",
    "mv_kv_resolve_payloads", "mv_kv_resolve_slots", "mv_kv_append", "mv_kv_write_last", "mv_kv_append_many",
    "mv_kv_gather_kv", "mv_attn_decode", "mv_attn_decode_plan_info",
    "mv_attn_decode_kernel_timing", "mv_prefill_workspace_size", "mv_attn_prefill",
    "mv_prefill_workspace_size_hd", "mv_attn_prefill_hd", "mv_attn_head_dim",
    "mv_interp_init", "mv_interp_feed", "mv_kv_write_range", "mv_toy_weight_count", "mv_toy_create", "mv_toy_destroy",
    "mv_toy_get_config", "mv_toy_vocab", "mv_toy_step", "mv_toy_load_context", "mv_toy_forward", "mv_argmax_rows",
    "mv_engine_run_forced", "mv_engine_run_batch", "mv_engine_run_free",
)


def check(status: int) -> None:
    if status == 0:
        return
    msg = lib.mv_last_error().decode(errors="replace")
    if status in CacheError.KINDS:
        raise CacheError(status, msg)
    if status in ParseError.KINDS:
        raise ParseError(status, msg)
    if status == 7:
        raise ValueError(msg)
    raise MvError(status, msg)


from . import dag, kv, attention, toy, interp  # noqa: E402,F401
