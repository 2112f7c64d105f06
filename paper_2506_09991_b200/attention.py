"""Branch-parallel paged decode (K4) and branch-masked prefill (K3) attention on the device."""
from __future__ import annotations

import ctypes

import torch

from . import check, lib
from .kv import PagedStore, _p, _u64_array


def decode(store: PagedStore, handles, q: torch.Tensor, positions: torch.Tensor, layer: int = 0,
           out: torch.Tensor | None = None, out_dtype: torch.dtype = torch.bfloat16) -> torch.Tensor:
    """q: bf16 [n, Hq, d] pre-RoPE queries of the tokens just appended to `handles` (d = the store's head_dim,
    64 or 128).
    out_dtype float32 returns the kernel's fp32 result (no bf16 store rounding)."""
    assert q.dtype == torch.bfloat16 and q.is_cuda and q.is_contiguous()
    n, hq, d = q.shape
    if d != store.head_dim:
        raise ValueError(f"decode: q head dim {d} != the store's head_dim {store.head_dim}")
    if out is None:
        out = torch.empty(q.shape, dtype=out_dtype, device=q.device)
    code = {torch.bfloat16: 0, torch.float32: 1}[out.dtype]
    check(lib.mv_attn_decode(store.handle, layer, _u64_array(handles), n, hq, _p(q), _p(positions), _p(out), code))
    return out


def prefill(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, positions: torch.Tensor, excl: torch.Tensor,
            rope_base: float = 10000.0, out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
            out_dtype: torch.dtype = torch.bfloat16):
    """q bf16 [n, Hq, d]; k, v bf16 [n, Hkv, d] (pre-RoPE; d = 64 or 128); excl int32 [n, D, 2] from
    dag.build_visibility."""
    n, hq, d = q.shape
    hkv = k.shape[1]
    if out is None:
        out = torch.empty(q.shape, dtype=out_dtype, device=q.device)
    code = {torch.bfloat16: 0, torch.float32: 1}[out.dtype]
    ws_bytes = lib.mv_prefill_workspace_size_hd(n, hq, hkv, d)
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=q.device)
    check(lib.mv_attn_prefill_hd(_p(q), _p(k), _p(v), _p(positions), _p(excl), excl.shape[1], n, hq, hkv, d, rope_base,
                              _p(out), code, _p(workspace), ws_bytes,
                              ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out
