"""CPU oracle for the per-lane tag interpreter (K5) — TEST INFRASTRUCTURE ONLY.

A pure-Python restatement of feed_interpreter (engine.cpp:323-415, with the BUG-2 fix of
oracle/ref_patch.py) and the merge-completion reset (engine.cpp:793), one lane at a time.
Pinned against the reference's own interpreter in tests/golden/interp.jsonl.gz
(tests/golden/gen_interp_golden.py, oracle/interp_drv.cpp); only tests import it.
"""
from __future__ import annotations

from dataclasses import dataclass

TAGS = ("<Parallel>", "</Parallel>", "<Goal>", "</Goal>", "<Outline>", "</Outline>", "<Path>", "</Path>",
        "<Conclusion>", "</Conclusion>")
P_OPEN, P_CLOSE, G_OPEN, G_CLOSE, O_OPEN, O_CLOSE, PATH, PATH_C, C_OPEN, C_CLOSE = range(10)
AWAIT_GOAL, GOAL, WAIT, AWAIT_CONCLUSION, CONCLUSION, AWAIT_CLOSE = range(6)  # InterpFrame::Phase
NONE, SPAWN, WORKER_DONE, VIOLATION = range(4)  # InterpAction::Kind
IDLE, MERGED = -1, -2


@dataclass
class Lane:
    child: bool
    depth: int = 0  # frames.size() (never above 1: frames are pushed only when empty, engine.cpp:335)
    phase: int = AWAIT_GOAL
    outlines: int = 0
    in_outline: bool = False
    after_outline: bool = False

    def row(self, kind, arg):
        """[kind, arg, depth, phase, outlines, in_outline, after_outline] (interp_drv's line)."""
        if self.depth == 0:
            return [kind, arg, 0, 0, 0, 0, 0]
        return [kind, arg, 1, self.phase, self.outlines, int(self.in_outline), int(self.after_outline)]


def feed(lane: Lane, ev: int):
    """Returns (kind, spawn_count, violation text or None)."""
    if ev == IDLE:
        return NONE, 0, None
    if ev == MERGED:
        if lane.depth == 0:
            return VIOLATION, 0, "merge without an open block"
        lane.phase = AWAIT_CONCLUSION
        return NONE, 0, None
    tag = ev < 10
    txt = TAGS[ev] if tag else f"w{ev}"
    if lane.depth == 0:  # engine.cpp:332-349
        if not tag:
            return NONE, 0, None
        if ev == P_OPEN:
            lane.depth, lane.phase, lane.outlines, lane.in_outline, lane.after_outline = 1, AWAIT_GOAL, 0, False, False
            return NONE, 0, None
        if ev == PATH and lane.child:
            return NONE, 0, None
        if ev == PATH_C:
            return (WORKER_DONE, 0, None) if lane.child else (VIOLATION, 0, "</Path> outside any path")
        return VIOLATION, 0, f"unexpected {txt} in sequential decode"
    ph = lane.phase
    if ph == AWAIT_GOAL:
        if ev == G_OPEN:
            lane.phase = GOAL
            return NONE, 0, None
        return VIOLATION, 0, "expected <Goal> after <Parallel>"
    if ph == GOAL:
        if not tag:
            if lane.after_outline and not lane.in_outline:
                return VIOLATION, 0, "text between outlines"
            return NONE, 0, None
        if ev == O_OPEN:
            if lane.in_outline:
                return VIOLATION, 0, "nested <Outline>"
            lane.in_outline = True
            lane.outlines += 1
            return NONE, 0, None
        if ev == O_CLOSE:
            if not lane.in_outline:
                return VIOLATION, 0, "</Outline> without <Outline>"
            lane.in_outline, lane.after_outline = False, True
            return NONE, 0, None
        if ev == G_CLOSE:
            if lane.in_outline:
                return VIOLATION, 0, "</Goal> inside <Outline>"
            if lane.outlines == 0:
                return VIOLATION, 0, "</Goal> with zero outlines"
            lane.phase = WAIT
            return SPAWN, lane.outlines, None
        return VIOLATION, 0, f"unexpected {txt} inside <Goal>"
    if ph == WAIT:
        return VIOLATION, 0, "token while waiting for paths"
    if ph == AWAIT_CONCLUSION:
        if ev == C_OPEN:
            lane.phase = CONCLUSION
            return NONE, 0, None
        return VIOLATION, 0, "expected <Conclusion> after merge"
    if ph == CONCLUSION:
        if not tag:
            return NONE, 0, None
        if ev == C_CLOSE:
            lane.phase = AWAIT_CLOSE
            return NONE, 0, None
        return VIOLATION, 0, f"unexpected {txt} inside <Conclusion>"
    if ev == P_CLOSE:  # AWAIT_CLOSE
        lane.depth = 0
        return NONE, 0, None
    return VIOLATION, 0, "expected </Parallel> after </Conclusion>"


def run(child: bool, events):
    """(rows, details) for one lane stream, in interp_drv's format."""
    lane = Lane(bool(child))
    rows, details = [], {}
    for i, ev in enumerate(events):
        kind, arg, text = feed(lane, int(ev))
        rows.append(lane.row(kind, arg))
        if text is not None:
            details[i] = text
    return rows, details
