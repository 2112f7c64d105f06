"""Paged KV store with fork / zero-copy merge (K2): mirrors multiverse::kv::RadixStore (kvcache.hpp:60-154).

Handles are plain integer ids (SequenceHandle::id); lengths come from `length(h)`.
Errors raise CacheError with the reference's kinds.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import check, lib


class _Cfg(ctypes.Structure):
    _fields_ = [("num_pages", ctypes.c_int32), ("record_bytes", ctypes.c_int32), ("layers", ctypes.c_int32),
                ("kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("table_entries", ctypes.c_int64),
                ("rope_base", ctypes.c_double)]


class _Stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in ("physical_tokens_stored", "logical_tokens_reachable",
                                               "bytes_copied_on_last_op", "live_handles", "node_count",
                                               "total_refcount", "free_pages")]


class _PlanInfo(ctypes.Structure):
    _fields_ = [("units", ctypes.c_int32), ("chunks", ctypes.c_int32), ("work_items", ctypes.c_int32),
                ("partial_slots", ctypes.c_int32), ("unique_kv_tokens", ctypes.c_int64),
                ("naive_kv_tokens", ctypes.c_int64)]


@dataclass
class StorageStats:
    physical_tokens_stored: int
    logical_tokens_reachable: int
    bytes_copied_on_last_op: int
    live_handles: int
    node_count: int
    total_refcount: int
    free_pages: int


def handle_array(hs) -> np.ndarray:
    """Handles as a contiguous uint64 array: pass it (instead of a list) to the per-step calls
    (append, write_last, attention.decode) to skip the per-call list -> C array conversion."""
    return np.ascontiguousarray(np.asarray([int(h) for h in hs], dtype=np.uint64))


def _u64_array(hs):
    if isinstance(hs, np.ndarray) and hs.dtype == np.uint64 and hs.flags["C_CONTIGUOUS"]:
        return ctypes.c_void_p(hs.ctypes.data)  # zero-copy view
    return (ctypes.c_uint64 * len(hs))(*[int(h) for h in hs])


class PagedStore:
    def __init__(self, num_pages: int, record_bytes: int = 0, layers: int = 0, kv_heads: int = 0,
                 head_dim: int = 128, table_entries: int = 0, rope_base: float = 10000.0):
        cfg = _Cfg(num_pages, record_bytes, layers, kv_heads, head_dim if kv_heads else 0, table_entries, rope_base)
        self._h = ctypes.c_void_p()
        check(lib.mv_kv_store_create(ctypes.byref(cfg), ctypes.byref(self._h)))
        self.record_bytes = record_bytes
        self.layers, self.kv_heads, self.head_dim = layers, kv_heads, head_dim
        self.set_stream(torch.cuda.current_stream())

    def close(self):
        if self._h:
            lib.mv_kv_store_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream: torch.cuda.Stream):
        check(lib.mv_kv_set_stream(self._h, ctypes.c_void_p(stream.cuda_stream)))

    # ---- RadixStore API ----
    def create(self) -> int:
        out = ctypes.c_uint64()
        check(lib.mv_kv_create(self._h, ctypes.byref(out)))
        return out.value

    def extend(self, h: int, tokens, payloads: bytes | None = None) -> int:
        toks = np.ascontiguousarray(tokens, dtype=np.int32)
        out = ctypes.c_uint64()
        pl = None
        if payloads is not None and self.record_bytes > 0 and len(toks) > 0:
            assert len(payloads) == len(toks) * self.record_bytes, "payload byte count does not match token count"
            pl = ctypes.c_char_p(bytes(payloads))
        check(lib.mv_kv_extend(self._h, h, toks.ctypes.data_as(ctypes.c_void_p), len(toks), pl,
                               ctypes.byref(out)))
        return out.value

    def fork(self, h: int, n: int) -> list[int]:
        out = (ctypes.c_uint64 * max(n, 1))()
        check(lib.mv_kv_fork(self._h, h, n, out))
        return list(out)[:n]

    def merge(self, prefix: int, branches) -> int:
        out = ctypes.c_uint64()
        check(lib.mv_kv_merge(self._h, prefix, _u64_array(branches), len(branches), ctypes.byref(out)))
        return out.value

    def release(self, h: int) -> None:
        check(lib.mv_kv_release(self._h, h))

    def length(self, h: int) -> int:
        out = ctypes.c_int64()
        check(lib.mv_kv_length(self._h, h, ctypes.byref(out)))
        return out.value

    def stats(self) -> StorageStats:
        s = _Stats()
        check(lib.mv_kv_stats_get(self._h, ctypes.byref(s)))
        return StorageStats(*[getattr(s, f) for f, _ in _Stats._fields_])

    def resolve(self, h: int) -> list[int]:
        n = self.length(h)
        out = np.zeros(max(n, 1), np.int32)
        check(lib.mv_kv_resolve(self._h, h, out.ctypes.data_as(ctypes.c_void_p)))
        return out[:n].tolist()

    def resolve_payloads(self, h: int) -> bytes:
        n = self.length(h) * self.record_bytes
        out = np.zeros(max(n, 1), np.uint8)
        check(lib.mv_kv_resolve_payloads(self._h, h, out.ctypes.data_as(ctypes.c_void_p)))
        return out[:n].tobytes()

    def resolve_slots(self, h: int) -> list[int]:
        n = self.length(h)
        out = np.zeros(max(n, 1), np.uint32)
        check(lib.mv_kv_resolve_slots(self._h, h, out.ctypes.data_as(ctypes.c_void_p)))
        return out[:n].tolist()

    # ---- device fast path ----
    def append(self, handles, tokens: torch.Tensor, positions: torch.Tensor | None = None, layer: int = 0,
               k: torch.Tensor | None = None, v: torch.Tensor | None = None) -> None:
        check(lib.mv_kv_append(self._h, _u64_array(handles), len(handles), _p(tokens), _p(positions), layer, _p(k),
                               _p(v)))

    def write_last(self, handles, positions: torch.Tensor, layer: int, k: torch.Tensor, v: torch.Tensor) -> None:
        check(lib.mv_kv_write_last(self._h, _u64_array(handles), len(handles), _p(positions), layer, _p(k), _p(v)))

    def append_many(self, h: int, tokens: torch.Tensor | None, positions: torch.Tensor | None = None,
                    layer: int = 0, k: torch.Tensor | None = None, v: torch.Tensor | None = None,
                    n: int | None = None) -> None:
        n = n if n is not None else (len(tokens) if tokens is not None else len(positions))
        check(lib.mv_kv_append_many(self._h, h, n, _p(tokens), _p(positions), layer, _p(k), _p(v)))

    def gather_kv(self, h: int, layer: int = 0):
        n = self.length(h)
        k = torch.empty((n, self.kv_heads, 128), dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        check(lib.mv_kv_gather_kv(self._h, h, layer, _p(k), _p(v)))
        return k, v

    def decode_kernel_timing(self, max_calls: int) -> list[float]:
        """Durations (ms) of the decode_tc launches recorded since the last call, then record the next
        max_calls mv_attn_decode calls (0 = off)."""
        ms = (ctypes.c_float * 1024)()
        n = ctypes.c_int32(0)
        check(lib.mv_attn_decode_kernel_timing(self._h, min(max_calls, 1024), ms, ctypes.byref(n)))
        return [float(ms[i]) for i in range(n.value)]

    def plan_info(self) -> dict:
        s = _PlanInfo()
        check(lib.mv_attn_decode_plan_info(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in _PlanInfo._fields_}

    @property
    def handle(self):
        return self._h


def _p(t):
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)
