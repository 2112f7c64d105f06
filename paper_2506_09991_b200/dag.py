"""Device mask / position builder (K1): mirrors multiverse::dag::build_visibility (dag.hpp:104-110).

`build_visibility(tokens)` takes tag-stream token ids (tok::Tokenizer ids: 0..9 tags, >= 10 text)
and returns positions, segment ids and exclusion intervals computed by the CUDA kernel.
The dense legacy `Mask` (dag.hpp:59-73) is expanded on the device from the intervals.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import ParseError, check, lib

DEFAULT_MAX_DEPTH = 4


def _ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@dataclass
class VisibilitySpec:
    positions: torch.Tensor   # int32 [n]           (assign_positions)
    seg_id: torch.Tensor      # int32 [n]           (GenerationDag segment id per layout row)
    excl: torch.Tensor        # int32 [n, D, 2]     (compact build_mask)
    max_depth: int

    @property
    def n(self) -> int:
        return int(self.positions.shape[0])

    def mask_packed(self, row0: int = 0, row1: int | None = None) -> torch.Tensor:
        row1 = self.n if row1 is None else row1
        out = torch.empty(((row1 - row0) * self.n + 7) // 8, dtype=torch.uint8, device=self.excl.device)
        check(lib.mv_mask_packed(_ptr(self.excl), self.n, self.max_depth, row0, row1, _ptr(out), _stream()))
        return out

    def mask(self) -> torch.Tensor:
        """Dense bool [n, n] (small n only)."""
        n = self.n
        bits = self.mask_packed()
        shifts = torch.arange(7, -1, -1, device=bits.device, dtype=torch.uint8)
        dense = ((bits.unsqueeze(1) >> shifts) & 1).reshape(-1)[: n * n]
        return dense.reshape(n, n).bool()


def build_visibility_batch(token_lists, max_depth: int = DEFAULT_MAX_DEPTH, device="cuda"):
    """Runs the K1 kernel over several tag streams in one launch.

    Returns (list of VisibilitySpec-or-ParseError, status tensor)."""
    lens = [len(t) for t in token_lists]
    offs = [0]
    for L in lens:
        offs.append(offs[-1] + L)
    total = offs[-1]
    h_offs = (ctypes.c_int64 * len(offs))(*offs)
    if lens and all(isinstance(t, torch.Tensor) for t in token_lists):  # no host round trip per token
        flat = torch.cat([t.reshape(-1).to(device=device, dtype=torch.int32) for t in token_lists])
        if flat.numel() == 0:
            flat = torch.zeros(1, dtype=torch.int32, device=device)
    else:
        flat = torch.tensor([int(x) for t in token_lists for x in t] or [0], dtype=torch.int32, device=device)
    pos = torch.empty(max(total, 1), dtype=torch.int32, device=device)
    seg = torch.empty(max(total, 1), dtype=torch.int32, device=device)
    excl = torch.empty((max(total, 1), max_depth, 2), dtype=torch.int32, device=device)
    status = torch.empty(len(lens), dtype=torch.int32, device=device)
    ws_bytes = lib.mv_visibility_workspace_size(h_offs, len(lens))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=device)
    check(lib.mv_visibility(_ptr(flat), h_offs, len(lens), max_depth, _ptr(pos), _ptr(seg), _ptr(excl),
                            _ptr(status), _ptr(ws), ws_bytes, _stream()))
    st = status.cpu().tolist()
    out = []
    for s, (a, b) in enumerate(zip(offs[:-1], offs[1:])):
        if st[s] != 0:
            out.append(st[s])
        else:
            out.append(VisibilitySpec(pos[a:b], seg[a:b], excl[a:b], max_depth))
    return out, st


MAX_DEPTH_LIMIT = 64  # the mask consumers' interval capacity (K3, tile maps)


def build_visibility(tokens, max_depth: int = DEFAULT_MAX_DEPTH, device="cuda") -> VisibilitySpec:
    """Positions + compact mask of one tag stream; raises ParseError like grammar::parse.  The interval
    capacity grows (doubling, up to MAX_DEPTH_LIMIT) when the stream nests deeper than `max_depth`."""
    toks = tokens if isinstance(tokens, torch.Tensor) else list(tokens)
    res, st = build_visibility_batch([toks], max_depth, device)
    while st[0] == 9 and max_depth < MAX_DEPTH_LIMIT:  # MV_ERR_DEPTH: more nesting than interval slots
        max_depth = min(2 * max_depth, MAX_DEPTH_LIMIT)
        res, st = build_visibility_batch([toks], max_depth, device)
    if st[0] != 0:
        check(st[0]) if st[0] not in ParseError.KINDS else None
        raise ParseError(st[0], f"tag stream rejected: {ParseError.KINDS.get(st[0], st[0])}")
    return res[0]


def tile_map(spec: VisibilitySpec, tile: int = 128):
    """(count[n_qt], list[n_qt, n_qt], visible_pairs) — tiles to compute for masked prefill."""
    n = spec.n
    n_qt = (n + tile - 1) // tile
    dev = spec.excl.device
    count = torch.empty(n_qt, dtype=torch.int32, device=dev)
    lst = torch.empty((n_qt, n_qt), dtype=torch.int32, device=dev)
    vis = torch.zeros(1, dtype=torch.int64, device=dev)
    check(lib.mv_tile_map(_ptr(spec.excl), n, spec.max_depth, tile, _ptr(count), _ptr(lst), _ptr(vis), _stream()))
    return count, lst, vis


@dataclass
class TrainingBatch:
    """dag::TrainingBatch (dag.hpp:124-139) on the device; the mask in its compact interval form."""
    token_ids: torch.Tensor   # int32 [n] (layout order = stream order)
    positions: torch.Tensor   # int32 [n]
    excl: torch.Tensor        # int32 [n, D, 2]
    target_ids: torch.Tensor  # int32 [n], -1 where a row has no next-token target
    loss_mask: torch.Tensor   # uint8 [n]
    max_depth: int


def build_training_batch(tokens, tag_loss: bool = True, max_depth: int = DEFAULT_MAX_DEPTH,
                         device="cuda") -> TrainingBatch:
    """dag::build_training_batch (dag.cpp:314-359) for one tag stream, in one K1 launch pair;
    raises ParseError like grammar::parse."""
    flat = (tokens.reshape(-1).to(device=device, dtype=torch.int32) if isinstance(tokens, torch.Tensor)
            else torch.tensor([int(x) for x in tokens] or [0], dtype=torch.int32, device=device))
    n = len(tokens)
    h_offs = (ctypes.c_int64 * 2)(0, n)
    m = max(n, 1)
    pos = torch.empty(m, dtype=torch.int32, device=device)
    excl = torch.empty((m, max_depth, 2), dtype=torch.int32, device=device)
    tgt = torch.empty(m, dtype=torch.int32, device=device)
    loss = torch.empty(m, dtype=torch.uint8, device=device)
    status = torch.empty(1, dtype=torch.int32, device=device)
    ws_bytes = lib.mv_visibility_workspace_size(h_offs, 1)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=device)
    check(lib.mv_training_batch(_ptr(flat), h_offs, 1, max_depth, int(bool(tag_loss)), _ptr(pos), _ptr(excl),
                                _ptr(tgt), _ptr(loss), _ptr(status), _ptr(ws), ws_bytes, _stream()))
    st = int(status.item())
    if st != 0:
        check(st) if st not in ParseError.KINDS else None
        raise ParseError(st, f"tag stream rejected: {ParseError.KINDS.get(st, st)}")
    return TrainingBatch(flat[:n], pos[:n], excl[:n], tgt[:n], loss[:n], max_depth)
