"""Device tag interpreter (K5): mirrors the engine's per-lane feed_interpreter (engine.cpp:323-415,
BUG-2 fixed) and the merge-completion reset (engine.cpp:793) over all lanes in one launch.

    it = TagInterpreter(n_lanes, is_child)         # LaneRuntime::parent >= 0 for worker lanes
    action, arg = it.feed(token_ids)               # [n_lanes] or [n_steps, n_lanes], int32 on the device
    it.feed(events) with MERGED for lanes whose paths were just merged

action is InterpAction::Kind (NONE, SPAWN, WORKER_DONE, VIOLATION); arg is the spawn count
(outlines of the closing <Goal>) or a VIOLATIONS code. Nothing is read back to the host unless the
caller asks (`spawns=True` also returns a compacted (step, lane, count) list on the device).
"""
from __future__ import annotations

import ctypes

import torch

from . import check, lib

STATE_WORDS = 2
IDLE, MERGED = -1, -2
NONE, SPAWN, WORKER_DONE, VIOLATION = range(4)
TAGS = ("<Parallel>", "</Parallel>", "<Goal>", "</Goal>", "<Outline>", "</Outline>", "<Path>", "</Path>",
        "<Conclusion>", "</Conclusion>")
# MV_VIOL_* -> the reference's InterpAction::detail text ({tag}: the offending token's literal)
VIOLATIONS = {
    1: "</Path> outside any path",
    2: "unexpected {tag} in sequential decode",
    3: "expected <Goal> after <Parallel>",
    4: "text between outlines",
    5: "nested <Outline>",
    6: "</Outline> without <Outline>",
    7: "</Goal> inside <Outline>",
    8: "</Goal> with zero outlines",
    9: "unexpected {tag} inside <Goal>",
    10: "token while waiting for paths",
    11: "expected <Conclusion> after merge",
    12: "unexpected {tag} inside <Conclusion>",
    13: "expected </Parallel> after </Conclusion>",
    14: "merge without an open block",
}


def violation_text(code: int, token: int) -> str:
    return VIOLATIONS[code].format(tag=TAGS[token] if 0 <= token < 10 else f"w{token}")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class TagInterpreter:
    def __init__(self, n_lanes: int, is_child=None, device="cuda"):
        self.n = int(n_lanes)
        self.device = torch.device(device)
        self.state = torch.empty((max(self.n, 1), STATE_WORDS), dtype=torch.int32, device=self.device)
        ch = None
        if is_child is not None:
            ch = torch.as_tensor(is_child, dtype=torch.int32).to(self.device).reshape(-1)
            if ch.numel() != self.n:
                raise ValueError("is_child must have one entry per lane")
        check(lib.mv_interp_init(_ptr(self.state), self.n, _ptr(ch), _stream()))

    def feed(self, events, spawns: bool = False):
        ev = torch.as_tensor(events, dtype=torch.int32).to(self.device)
        one = ev.dim() == 1
        ev = (ev.reshape(-1, self.n) if self.n else ev.reshape(ev.shape[0] if ev.dim() == 2 else 1, 0)).contiguous()
        steps = ev.shape[0]
        action = torch.empty_like(ev)
        arg = torch.empty_like(ev)
        sp = cnt = None
        if spawns:
            sp = torch.empty((max(ev.numel(), 1), 3), dtype=torch.int32, device=self.device)
            cnt = torch.zeros(1, dtype=torch.int32, device=self.device)
        check(lib.mv_interp_feed(_ptr(self.state), self.n, _ptr(ev), steps, _ptr(action), _ptr(arg), _ptr(sp),
                                 _ptr(cnt), _stream()))
        if one:
            action, arg = action[0], arg[0]
        return (action, arg, sp, cnt) if spawns else (action, arg)

    def lanes(self) -> torch.Tensor:
        """[n, 5] = depth, phase, outlines, in_outline, after_outline (zeros when no frame is open)."""
        s = self.state[: self.n]
        depth = s[:, 0] & 0xFF
        f = torch.where(depth > 0, s[:, 1], torch.zeros_like(s[:, 1]))
        return torch.stack([depth, f & 7, f >> 8, (f >> 3) & 1, (f >> 4) & 1], 1)
