"""CPU oracle for the Multiverse hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs import this package, and only as the checker or the timed CPU baseline. The
product package (paper_2506_09991_b200) never imports it.

`libmvoracle.so` is built from oracle/mv_oracle.c (a restatement of the reference's
dag.cpp / toy_model.cpp algorithms, citing file:line) by `build()`; parity of the
restatement itself is pinned against the patched reference's own outputs in
tests/golden/ (see tests/test_oracle_golden.py).
"""
from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB = HERE / "libmvoracle.so"

ERR_NAMES = {0: "ok", 1: "MalformedStructure", 2: "CountMismatch"}


def build(force: bool = False) -> pathlib.Path:
    src = HERE / "mv_oracle.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", str(LIB), str(src), "-lm", "-lpthread"],
                       check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        i32, i64, f64, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64
        L.mvo_build_dag.argtypes = [P, ctypes.c_int, P, P, P, P]
        L.mvo_mask_packed.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
        L.mvo_fill_symmetric.argtypes = [u64, f64, P, i64]
        L.mvo_rope.argtypes = [P, i64, ctypes.c_int, ctypes.c_int, P, f64]
        L.mvo_attn_decode.argtypes = [P, P, P, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, ctypes.c_int]
        L.mvo_attn_prefill.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.c_int, P, i64, P,
                                       ctypes.c_int]
        L.mvo_attn_prefill_mask.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, i64, P, i64, P,
                                            ctypes.c_int]
        L.mvo_batch_targets.argtypes = [P, ctypes.c_int, ctypes.c_int, P, P]
        L.mvo_toy_new.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, u64, f64, f64]
        L.mvo_toy_new.restype = P
        L.mvo_toy_free.argtypes = [P]
        L.mvo_toy_weight.argtypes = [P, ctypes.c_int, ctypes.c_int]
        L.mvo_toy_weight.restype = ctypes.POINTER(ctypes.c_double)
        L.mvo_toy_step.argtypes = [P, P, i64, ctypes.c_int, ctypes.c_int, P, P, P]
        L.mvo_toy_forward.argtypes = [P, P, P, P, i64, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def threads() -> int:
    return int(os.environ.get("MV_ORACLE_THREADS", os.cpu_count() or 1))


def build_dag(tokens):
    """(err, positions, seg_id, seg_kind). err: 0 ok, 1 MalformedStructure, 2 CountMismatch."""
    t = np.ascontiguousarray(tokens, dtype=np.int32)
    n = len(t)
    pos = np.zeros(n, np.int32)
    seg = np.zeros(n, np.int32)
    kind = np.zeros(n, np.int32)
    ns = np.zeros(1, np.int32)
    err = lib().mvo_build_dag(_p(t), n, _p(pos), _p(seg), _p(kind), _p(ns))
    return err, pos, seg, kind


def batch_targets(tokens, tag_loss: bool = True):
    """(err, target_ids, loss_mask) of build_training_batch (dag.cpp:326-357), restated over segments."""
    t = np.ascontiguousarray(tokens, dtype=np.int32)
    n = len(t)
    tgt = np.full(max(n, 1), -1, np.int32)
    loss = np.zeros(max(n, 1), np.uint8)
    err = lib().mvo_batch_targets(_p(t), n, int(bool(tag_loss)), _p(tgt), _p(loss))
    return err, tgt[:n], loss[:n]


def mask_packed(tokens, row0: int = 0, row1: int | None = None) -> np.ndarray:
    t = np.ascontiguousarray(tokens, dtype=np.int32)
    n = len(t)
    row1 = n if row1 is None else row1
    out = np.zeros(((row1 - row0) * n + 7) // 8, np.uint8)
    err = lib().mvo_mask_packed(_p(t), n, row0, row1, _p(out))
    if err:
        raise ValueError(f"oracle parse error {ERR_NAMES.get(err, err)}")
    return out


def mask_dense(tokens) -> np.ndarray:
    n = len(tokens)
    return np.unpackbits(mask_packed(tokens))[: n * n].reshape(n, n).astype(bool)


def fill_symmetric(seed: int, r: float, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().mvo_fill_symmetric(seed, r, _p(out), n)
    return out


def rope(x: np.ndarray, pos, base: float = 10000.0) -> np.ndarray:
    """Interleaved rotary (toy_model.cpp:30-41) in fp64; x [rows, heads, dh]."""
    y = np.ascontiguousarray(x, dtype=np.float64).copy()
    p = np.ascontiguousarray(pos, dtype=np.int32)
    lib().mvo_rope(_p(y), y.shape[0], y.shape[1], y.shape[2], _p(p), base)
    return y


def attn_decode(q, K, V, ctx_lists, nthreads: int | None = None) -> np.ndarray:
    """q [B,Hq,D], K/V [N,Hkv,D] (post-RoPE, fp64); ctx_lists[b] = context row ids in order."""
    q = np.ascontiguousarray(q, np.float64)
    K = np.ascontiguousarray(K, np.float64)
    V = np.ascontiguousarray(V, np.float64)
    B, hq, dh = q.shape
    hkv = K.shape[1]
    ptr = np.zeros(B + 1, np.int64)
    ptr[1:] = np.cumsum([len(c) for c in ctx_lists])
    idx = np.ascontiguousarray(np.concatenate([np.asarray(c, np.int64) for c in ctx_lists]) if B else
                               np.zeros(0, np.int64))
    out = np.zeros_like(q)
    lib().mvo_attn_decode(_p(q), _p(K), _p(V), B, hq, hkv, dh, _p(ptr), _p(idx), _p(out), nthreads or threads())
    return out


def attn_prefill(q_rows, K, V, excl, rows, nthreads: int | None = None) -> np.ndarray:
    """q_rows [len(rows),Hq,D] (post-RoPE queries of the sampled rows), K/V [n,Hkv,D] post-RoPE fp64;
    excl [n,D_excl,2] int32; rows: the sampled query row indices. Returns [len(rows),Hq,D]."""
    q = np.ascontiguousarray(q_rows, np.float64)
    K = np.ascontiguousarray(K, np.float64)
    V = np.ascontiguousarray(V, np.float64)
    ex = np.ascontiguousarray(excl, np.int32)
    r = np.ascontiguousarray(rows, np.int32)
    _, hq, dh = q.shape
    out = np.zeros((len(r), hq, dh), np.float64)
    lib().mvo_attn_prefill(_p(q), _p(K), _p(V), hq, K.shape[1], dh, _p(ex), ex.shape[1], _p(r), len(r), _p(out),
                           nthreads or threads())
    return out


def attn_prefill_tokens(q_rows, K, V, tokens, rows, nthreads: int | None = None) -> np.ndarray:
    """The prefill oracle with the mask built from the tag stream by the oracle's own build_mask restatement
    (segment ancestry, dag.cpp:227-263; no interval form): independent of the device K1 builder."""
    q = np.ascontiguousarray(q_rows, np.float64)
    K = np.ascontiguousarray(K, np.float64)
    V = np.ascontiguousarray(V, np.float64)
    r = np.ascontiguousarray(rows, np.int32)
    n = len(tokens)
    bits = np.concatenate([np.unpackbits(mask_packed(tokens, int(i), int(i) + 1))[:n] for i in r]) if len(r) else \
        np.zeros(0, np.uint8)
    packed = np.ascontiguousarray(np.packbits(bits))
    _, hq, dh = q.shape
    out = np.zeros((len(r), hq, dh), np.float64)
    lib().mvo_attn_prefill_mask(_p(q), _p(K), _p(V), hq, K.shape[1], dh, _p(packed), n, _p(r), len(r), _p(out),
                                nthreads or threads())
    return out


class Toy:
    """Restated ToyModel (toy_model.cpp:45-202); weights drawn exactly as the reference."""

    def __init__(self, layers=2, heads=2, model_dim=32, vocab=256, seed=0, init=0.05, rope=10000.0):
        self.layers, self.heads, self.d, self.vocab = layers, heads, model_dim, vocab
        self.h = lib().mvo_toy_new(layers, heads, model_dim, vocab, seed, init, rope)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().mvo_toy_free(self.h)
                self.h = None
        except Exception:  # interpreter shutdown
            pass

    @property
    def rec(self):
        return 2 * self.layers * self.d

    def weight(self, which: str, layer: int = 0) -> np.ndarray:
        codes = {"emb": 0, "unemb": 1, "wq": 2, "wk": 3, "wv": 4, "wo": 5, "up": 6, "down": 7}
        d, H, V = self.d, 4 * self.d, self.vocab
        shape = {"emb": (V, d), "unemb": (V, d), "wq": (d, d), "wk": (d, d), "wv": (d, d), "wo": (d, d),
                 "up": (H, d), "down": (d, H)}[which]
        ptr = lib().mvo_toy_weight(self.h, codes[which], layer)
        return np.ctypeslib.as_array(ptr, shape=shape).copy()

    def step(self, ctx: np.ndarray, token: int, position: int):
        ctx = np.ascontiguousarray(ctx, np.float64).reshape(-1)
        n = len(ctx) // self.rec
        logits = np.zeros(self.vocab)
        hidden = np.zeros(self.d)
        kv = np.zeros(self.rec)
        lib().mvo_toy_step(self.h, _p(ctx), n, token, position, _p(logits), _p(hidden), _p(kv))
        return logits, hidden, kv

    def forward(self, ids, pos, mask: np.ndarray) -> np.ndarray:
        ids = np.ascontiguousarray(ids, np.int32)
        pos = np.ascontiguousarray(pos, np.int32)
        m = np.ascontiguousarray(mask, np.uint8)
        n = len(ids)
        out = np.zeros((n, self.vocab))
        lib().mvo_toy_forward(self.h, _p(ids), _p(pos), _p(m), n, _p(out))
        return out
