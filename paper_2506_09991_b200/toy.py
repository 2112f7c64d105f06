"""GPU toy transformer around the hot path (BASELINE configs[0] parity).

The reference's ToyModel (toy_model.cpp:45-202) is a pre-norm-free transformer: x = emb[id];
per layer q, k, v = W x, interleaved RoPE per head at the token's Multiverse position
(toy_model.cpp:30-41), attention over the visible context then self (:121-157),
x += Wo attn, x += down(tanh(up x)); logits = unemb x.  Here the layer algebra (projections,
MLP, unembed) is plain GEMMs in fp64 on the GPU and the attention is this package's kernels:

* `ToyModel.forward(ids)` — ToyModel::forward (toy_model.cpp:174-202): one masked prefill per
  layer over the whole tag stream, with the K1 positions / exclusion intervals.
* `ToyModel.run_forced(ids)` — engine::run_forced (engine.cpp:928-939, lanes :498-582): a lane
  per Process-stage path, all active lanes stepped together (one append + one decode per layer
  for the whole batch), fork at a block's first `<Path>` (spawn_children, :679-725), zero-copy
  merge when every path lane finished (maybe_merge, :767-802), KV in the paged store.

The kernels are built for head_dim 128.  A smaller head (C1: 4 heads x 64) is zero-padded to
128 lanes: zero q/k dims add nothing to q.k, zero v dims give zero outputs that are dropped,
and q is pre-scaled by sqrt(128 / dh) so the kernels' 1/sqrt(128) becomes 1/sqrt(dh).  RoPE
frequencies depend on dh (theta = pos * base^(-2t/dh)), so q and k are rotated here, in fp64,
and the kernels are called with position 0 (the identity rotation; positions only feed RoPE in
both attention entry points).
"""
from __future__ import annotations

import math

import torch

from . import attention, dag
from .host.tokenize import PATH_CLOSE, PATH_OPEN
from .kv import PagedStore

KDIM = 128  # the kernels' head dim


class ToyModel:
    def __init__(self, weights: dict, layers: int, heads: int, model_dim: int, vocab: int, rope_base: float = 1e4,
                 device="cuda"):
        """weights: emb [V, D], unemb [V, D], and per layer lists wq, wk, wv, wo [D, D], up [4D, D],
        down [D, 4D] (row-major as in ToyModelWeights, toy_model.hpp:33-47)."""
        self.L, self.H, self.D, self.V = layers, heads, model_dim, vocab
        self.dh = model_dim // heads
        if self.dh > KDIM or model_dim % heads:
            raise ValueError("head_dim must divide model_dim and be <= 128")
        self.rope_base = rope_base
        self.dev = torch.device(device)
        f64 = lambda t: torch.as_tensor(t, dtype=torch.float64).to(self.dev)  # noqa: E731
        self.emb, self.unemb = f64(weights["emb"]), f64(weights["unemb"])
        self.w = {k: [f64(m) for m in weights[k]] for k in ("wq", "wk", "wv", "wo", "up", "down")}
        t = torch.arange(self.dh // 2, dtype=torch.float64, device=self.dev)
        self.inv_freq = rope_base ** (-2.0 * t / self.dh)

    # ---- pieces ----
    def _rotate(self, x: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        """x [n, H, dh] fp64, pos [n]: interleaved pairs (2t, 2t+1) by pos * base^(-2t/dh)."""
        th = pos.to(torch.float64)[:, None] * self.inv_freq[None, :]  # [n, dh/2]
        c, s = torch.cos(th)[:, None, :], torch.sin(th)[:, None, :]
        a, b = x[..., 0::2], x[..., 1::2]
        out = torch.empty_like(x)
        out[..., 0::2] = a * c - b * s
        out[..., 1::2] = a * s + b * c
        return out

    def _pad(self, x: torch.Tensor, scale: float = 1.0) -> torch.Tensor:
        n, h, dh = x.shape
        out = torch.zeros(n, h, KDIM, dtype=torch.bfloat16, device=self.dev)
        out[..., :dh] = (x * scale).to(torch.bfloat16)
        return out.contiguous()

    def _qkv(self, x: torch.Tensor, layer: int, pos: torch.Tensor):
        n = x.shape[0]
        q = (x @ self.w["wq"][layer].T).view(n, self.H, self.dh)
        k = (x @ self.w["wk"][layer].T).view(n, self.H, self.dh)
        v = (x @ self.w["wv"][layer].T).view(n, self.H, self.dh)
        q, k = self._rotate(q, pos), self._rotate(k, pos)
        return self._pad(q, math.sqrt(KDIM / self.dh)), self._pad(k), self._pad(v)

    def _finish_layer(self, x: torch.Tensor, attn: torch.Tensor, layer: int) -> torch.Tensor:
        n = x.shape[0]
        a = attn[..., : self.dh].to(torch.float64).reshape(n, self.D)
        x = x + a @ self.w["wo"][layer].T
        return x + torch.tanh(x @ self.w["up"][layer].T) @ self.w["down"][layer].T

    # ---- ToyModel::forward over the masked layout (one prefill launch per layer) ----
    def forward(self, ids) -> torch.Tensor:
        ids = [int(i) for i in ids]
        spec = dag.build_visibility(ids)
        n = len(ids)
        x = self.emb[torch.tensor([i % self.V for i in ids], device=self.dev)]
        zero = torch.zeros(n, dtype=torch.int32, device=self.dev)
        for layer in range(self.L):
            q, k, v = self._qkv(x, layer, spec.positions)
            attn = attention.prefill(q, k, v, zero, spec.excl, out_dtype=torch.float32)
            x = self._finish_layer(x, attn, layer)
        return x @ self.unemb.T

    # ---- engine::run_forced: lanes, fork / merge, batched decode steps ----
    def run_forced(self, ids, num_pages: int = 4096):
        """Returns (logits [n, V] in layout order, stats) for a forced tag stream."""
        ids = [int(i) for i in ids]
        n = len(ids)
        spec = dag.build_visibility(ids)  # K1: positions (bit-exact with assign_positions)
        pos = spec.positions.to(self.dev)
        program, end = _parse_program(ids, 0, stop_at_path_close=False)
        assert end == n
        st = PagedStore(num_pages=num_pages, layers=self.L, kv_heads=self.H)
        logits = torch.empty(n, self.V, dtype=torch.float64, device=self.dev)
        root = _Lane(st.create(), program, None)
        lanes = [root]
        steps = forks = merges = 0
        while not root.done():
            batch = []
            for lane in list(lanes):
                if lane.waiting or lane.done():
                    continue
                op = lane.ops[lane.pc]
                if op[0] == "block":  # spawn_children: one forked lane per path
                    kids = st.fork(lane.handle, len(op[1]))
                    forks += 1
                    lane.children = [_Lane(h, p, lane) for h, p in zip(kids, op[1])]
                    lane.waiting = True
                    lane.pc += 1
                    lanes.extend(lane.children)
                    continue
                batch.append((lane, op[1]))
            if batch:
                self._step(st, batch, ids, pos, logits)
                steps += 1
                for lane, _ in batch:
                    lane.pc += 1
            # maybe_merge: parents whose path lanes all finished
            for lane in list(lanes):
                if lane.waiting and all(c.done() for c in lane.children):
                    merged = st.merge(lane.handle, [c.handle for c in lane.children])
                    merges += 1
                    for h in [lane.handle] + [c.handle for c in lane.children]:
                        st.release(h)
                    for c in lane.children:
                        lanes.remove(c)
                    lane.handle, lane.children, lane.waiting = merged, [], False
        stats = {"steps": steps, "forks": forks, "merges": merges, "tokens": n, "length": st.length(root.handle),
                 "store": st.stats()}
        st.release(root.handle)
        return logits, stats

    def _step(self, st: PagedStore, batch, ids, pos, logits):
        """One engine step for every lane in `batch`: append each lane's next token, attend."""
        idx = torch.tensor([t for _, t in batch], device=self.dev)
        handles = [lane.handle for lane, _ in batch]
        tok = torch.tensor([ids[t] for _, t in batch], dtype=torch.int32, device=self.dev)
        x = self.emb[torch.tensor([ids[t] % self.V for _, t in batch], device=self.dev)]
        p = pos[idx]
        zero = torch.zeros(len(batch), dtype=torch.int32, device=self.dev)
        for layer in range(self.L):
            q, k, v = self._qkv(x, layer, p)
            if layer == 0:
                st.append(handles, tok, zero, 0, k, v)
            else:
                st.write_last(handles, zero, layer, k, v)
            attn = attention.decode(st, handles, q, zero, layer=layer, out_dtype=torch.float32)
            x = self._finish_layer(x, attn, layer)
        logits[idx] = x @ self.unemb.T


class _Lane:
    def __init__(self, handle, ops, parent):
        self.handle, self.ops, self.parent = handle, ops, parent
        self.pc, self.waiting, self.children = 0, False, []

    def done(self):
        return not self.waiting and self.pc >= len(self.ops)


def _parse_program(ids, i, stop_at_path_close):
    """A lane program: ('tok', index) ops, and ('block', [path programs]) where a block's first
    <Path> starts (the lane forks there; the lane after the merge continues with the rest)."""
    ops = []
    n = len(ids)
    while i < n:
        t = ids[i]
        if t == PATH_OPEN:
            paths = []
            while i < n and ids[i] == PATH_OPEN:
                start = i
                body, i = _parse_program(ids, i + 1, stop_at_path_close=True)
                paths.append([("tok", start)] + body)
            ops.append(("block", paths))
            continue
        ops.append(("tok", i))
        i += 1
        if t == PATH_CLOSE and stop_at_path_close:
            return ops, i
    return ops, i
