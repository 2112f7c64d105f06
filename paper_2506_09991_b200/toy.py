"""The reference's toy transformer and its engine on the device (BASELINE configs[0]).

Binds three parts of libmvb200 (include/multiverse_b200.h):

* `ToyModel` <- toy::ToyModel (toy_model.hpp:71-92): `mv_toy_*`, every layer op on the GPU (fp32
  projections / tanh MLP / unembed, fp64 RoPE at the Multiverse position, attention through K3 / K4).
  `forward(ids)` is ToyModel::forward over a whole tag stream (K1 positions + exclusion intervals, one
  masked prefill per layer).
* `run_forced(ids)` / `run_free(prompt)` <- engine::run_forced / run_free (engine.cpp:928-950): the C++
  engine of `mv_engine_*` (engine.cu): one batched device pass per step for every active lane, the K5 tag
  interpreter on the device, fork / zero-copy merge of the paged store on spawn / reduce.

Head dims 64 and 128 run on native attention kernels; other head dims ride the 128-wide kernels
zero-padded (toy.cu, mv_attn_head_dim).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import LABEL_FN, check, dag, lib


class _ToyCfg(ctypes.Structure):
    _fields_ = [("layers", ctypes.c_int32), ("heads", ctypes.c_int32), ("model_dim", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("rope_base", ctypes.c_double)]


class _EngineOpts(ctypes.Structure):
    _fields_ = [("max_worker_tokens", ctypes.c_int32), ("max_request_tokens", ctypes.c_int32),
                ("num_pages", ctypes.c_int32)]


class _Report(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("failure", ctypes.c_int32), ("failure_detail", ctypes.c_char * 256),
                ("steps", ctypes.c_int64), ("total_tokens", ctypes.c_int64), ("merges", ctypes.c_int64),
                ("spawns", ctypes.c_int64), ("lanes", ctypes.c_int64), ("events", ctypes.c_int64)]


class _Event(ctypes.Structure):
    _fields_ = [("step", ctypes.c_int64), ("request", ctypes.c_int32), ("lane", ctypes.c_int32),
                ("kind", ctypes.c_int32), ("token", ctypes.c_int32), ("source", ctypes.c_int32)]


EVENT_KINDS = {0: "Decode", 1: "Prefill", 2: "Spawn", 3: "ZombieEnter", 4: "Merge", 6: "Done", 7: "Failed"}
FAILURES = {0: "None", 1: "GrammarViolationDuringDecode", 2: "LimitExceeded"}


def flat_weights(weights: dict, layers: int) -> np.ndarray:
    """ToyModelWeights order (toy_model.cpp:58-68): embedding; per layer wq wk wv wo w_up w_down; unembed."""
    parts = [np.asarray(weights["emb"], np.float64).ravel()]
    for layer in range(layers):
        for k in ("wq", "wk", "wv", "wo", "up", "down"):
            parts.append(np.asarray(weights[k][layer], np.float64).ravel())
    parts.append(np.asarray(weights["unemb"], np.float64).ravel())
    return np.ascontiguousarray(np.concatenate(parts))


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class ToyModel:
    def __init__(self, weights: dict, layers: int, heads: int, model_dim: int, vocab: int, rope_base: float = 1e4,
                 device="cuda"):
        """weights: emb [V, D], unemb [V, D], and per layer lists wq, wk, wv, wo [D, D], up [4D, D], down [D, 4D]
        (row-major as in ToyModelWeights, toy_model.hpp:33-47), host fp64."""
        self.L, self.H, self.D, self.V = layers, heads, model_dim, vocab
        self.dev = torch.device(device)
        self._cfg = _ToyCfg(layers, heads, model_dim, vocab, rope_base)
        w = flat_weights(weights, layers)
        assert w.size == lib.mv_toy_weight_count(ctypes.byref(self._cfg)), "weight count"
        self._h = ctypes.c_void_p()
        check(lib.mv_toy_create(ctypes.byref(self._cfg), w.ctypes.data_as(ctypes.c_void_p), ctypes.byref(self._h)))

    def __del__(self):
        try:
            if self._h:
                lib.mv_toy_destroy(self._h)
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def forward(self, ids) -> torch.Tensor:
        """ToyModel::forward (toy_model.cpp:174-202): logits fp32 [n, V] on the device."""
        ids = [int(i) for i in ids]
        spec = dag.build_visibility(ids)
        n = len(ids)
        tok = torch.tensor(ids, dtype=torch.int32, device=self.dev)
        logits = torch.empty(n, self.V, dtype=torch.float32, device=self.dev)
        check(lib.mv_toy_forward(self._h, _p(tok), n, _p(spec.positions), _p(spec.excl), spec.max_depth, _p(logits),
                                 None, _stream()))
        return logits

    def step(self, store, handles, tokens: torch.Tensor, positions: torch.Tensor, hidden=False, kv=False):
        """ToyModel::step for every lane in `handles` at once (engine.cpp:603-641 batched)."""
        n = len(handles)
        from .kv import _u64_array
        logits = torch.empty(n, self.V, dtype=torch.float32, device=self.dev)
        hid = torch.empty(n, self.D, dtype=torch.float32, device=self.dev) if hidden else None
        rec = torch.empty(n, 2 * self.L * self.D, dtype=torch.float32, device=self.dev) if kv else None
        check(lib.mv_toy_step(self._h, store.handle, _u64_array(handles), n, _p(tokens), _p(positions), _p(logits),
                              _p(hid), _p(rec)))
        return logits, hid, rec

    def run_forced(self, ids, num_pages: int = 4096, max_worker_tokens: int = 0, max_request_tokens: int = 0):
        """engine::run_forced with record_logits: (logits [n, V] fp32 by source index, report dict)."""
        ids = np.ascontiguousarray([int(i) for i in ids], dtype=np.int32)
        n = len(ids)
        logits = np.zeros((max(n, 1), self.V), np.float32)
        cap = 8 * n + 64
        events = (_Event * cap)()
        rep = _Report()
        opts = _EngineOpts(max_worker_tokens, max_request_tokens, num_pages)
        check(lib.mv_engine_run_forced(self._h, ids.ctypes.data_as(ctypes.c_void_p), n, ctypes.byref(opts), _stream(),
                                       logits.ctypes.data_as(ctypes.c_void_p), events, cap, ctypes.byref(rep)))
        return torch.from_numpy(logits[:n]), _report(rep, events, cap)

    def run_batch(self, streams, num_pages: int = 4096, max_worker_tokens: int = 0, max_request_tokens: int = 0):
        """engine::run_batch (with the toy model attached): every step one device pass over the active lanes
        of ALL requests.  Returns ([logits [n_r, V] per request], report dict; events carry the request)."""
        streams = [np.ascontiguousarray([int(i) for i in s_], dtype=np.int32) for s_ in streams]
        offs = np.zeros(len(streams) + 1, np.int64)
        offs[1:] = np.cumsum([len(s_) for s_ in streams])
        flat = np.ascontiguousarray(np.concatenate(streams) if offs[-1] else np.zeros(1, np.int32))
        logits = np.zeros((max(int(offs[-1]), 1), self.V), np.float32)
        cap = 8 * int(offs[-1]) + 64 * len(streams)
        events = (_Event * cap)()
        rep = _Report()
        opts = _EngineOpts(max_worker_tokens, max_request_tokens, num_pages)
        check(lib.mv_engine_run_batch(self._h, flat.ctypes.data_as(ctypes.c_void_p),
                                      offs.ctypes.data_as(ctypes.c_void_p), len(streams), ctypes.byref(opts),
                                      _stream(), logits.ctypes.data_as(ctypes.c_void_p), events, cap,
                                      ctypes.byref(rep)))
        out = [torch.from_numpy(logits[offs[r]:offs[r + 1]]) for r in range(len(streams))]
        return out, _report(rep, events, cap)

    def run_free(self, prompt, label_token=None, max_steps: int = 0, num_pages: int = 4096,
                 max_worker_tokens: int = 0, max_request_tokens: int = 0):
        """engine::run_free (greedy): the report dict, with the emitted tokens per event."""
        prompt = np.ascontiguousarray([int(i) for i in prompt], dtype=np.int32)
        cap = 4 * (len(prompt) + max(max_steps, 4096)) + 64
        events = (_Event * cap)()
        rep = _Report()
        opts = _EngineOpts(max_worker_tokens, max_request_tokens, num_pages)
        fn = LABEL_FN(lambda ctx, text: int(label_token(text.decode()))) if label_token else LABEL_FN(0)
        check(lib.mv_engine_run_free(self._h, prompt.ctypes.data_as(ctypes.c_void_p), len(prompt), max_steps,
                                     ctypes.byref(opts), fn, None, _stream(), events, cap, ctypes.byref(rep)))
        return _report(rep, events, cap)


def _report(rep: _Report, events, cap) -> dict:
    ev = [(events[i].step, events[i].lane, EVENT_KINDS.get(events[i].kind, events[i].kind), events[i].token,
           events[i].source, events[i].request) for i in range(min(rep.events, cap))]
    return {"status": "Failed" if rep.status else "Done", "failure": FAILURES.get(rep.failure, rep.failure),
            "failure_detail": rep.failure_detail.decode(), "steps": rep.steps, "total_tokens": rep.total_tokens,
            "merges": rep.merges, "spawns": rep.spawns, "lanes": rep.lanes, "events": ev}


def _p(t):
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)
