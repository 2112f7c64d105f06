#!/usr/bin/env python3
"""Writes tests/golden/interp.jsonl.gz: the reference's own per-lane tag interpreter
(feed_interpreter, engine.cpp:323-415, BUG-2 patched; driven by oracle/interp_drv.cpp) over
lane event streams.

Run in the build container (where /root/reference exists):
    ./oracle/ref_build.sh && python tests/golden/gen_interp_golden.py

Streams: the engine's lane split of the reference-generated trajectories in dag.jsonl.gz (the
root lane sees everything outside its paths, with the merge completion before <Conclusion>;
each worker lane sees its <Path> ... </Path> with its own inner paths split off the same way),
the same streams with a few random edits (violations), and short random tag soups.
Each line: {"child": 0|1, "events": [...], "out": [[kind, arg, depth, phase, outlines,
in_outline, after_outline], ...], "detail": {event index: violation text}}.
"""
import gzip
import json
import pathlib
import subprocess
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
DRV = REPO / "oracle" / "_ref" / "interp_drv"
PATH_OPEN, PATH_CLOSE, CONC_OPEN = 6, 7, 8
IDLE, MERGED = -1, -2


def lane_streams(toks, i0, i1, child, out):
    """The engine's lanes over toks[i0:i1] (a child range starts with <Path>, ends with </Path>)."""
    ev = []
    i = i0
    if child:
        ev.append(toks[i0])
        i, i1 = i0 + 1, i1 - 1
    while i < i1:
        t = toks[i]
        if t == PATH_OPEN:
            depth, j = 0, i
            while True:
                depth += {PATH_OPEN: 1, PATH_CLOSE: -1}.get(toks[j], 0)
                if depth == 0:
                    break
                j += 1
            lane_streams(toks, i, j + 1, True, out)
            i = j + 1
            continue
        if t == CONC_OPEN:
            ev.append(MERGED)
        ev.append(t)
        i += 1
    if child:
        ev.append(toks[i1])
    out.append((int(child), ev))


def mutate(ev, rng):
    ev = list(ev)
    for _ in range(int(rng.integers(1, 4))):
        k = int(rng.integers(0, len(ev) + 1))
        r = rng.random()
        new = int(rng.choice([*range(10), 10 + int(rng.integers(0, 50)), MERGED, IDLE]))
        if r < 0.4 and k < len(ev):
            ev[k] = new
        elif r < 0.7:
            ev.insert(k, new)
        elif k < len(ev):
            del ev[k]
    return ev


def main():
    if not DRV.exists():
        sys.exit("build oracle/_ref first: ./oracle/ref_build.sh")
    rng = np.random.default_rng(2506)
    with gzip.open(HERE / "dag.jsonl.gz", "rt") as f:
        dags = [json.loads(line) for line in f if line.strip()]
    cases = []
    for d in dags:
        if d["error"] != -1:
            continue
        lanes = []
        lane_streams([int(t) for t in d["tokens"]], 0, len(d["tokens"]), False, lanes)
        cases += lanes
        if len(cases) > 900:
            break
    valid = list(cases)
    for k in range(600):
        child, ev = valid[int(rng.integers(0, len(valid)))]
        cases.append((child if rng.random() < 0.8 else 1 - child, mutate(ev, rng)))
    for k in range(300):
        n = int(rng.integers(1, 40))
        ev = [int(rng.choice([*range(10), 10, 11, 12, MERGED, IDLE])) for _ in range(n)]
        cases.append((int(rng.integers(0, 2)), ev))
    cases = [(c, ev) for c, ev in cases if ev]
    stdin = "".join(f"{c} {len(ev)} {' '.join(map(str, ev))}\n" for c, ev in cases)
    res = subprocess.run([str(DRV)], input=stdin, text=True, capture_output=True, check=True).stdout.splitlines()
    lines, pos = [], 0
    for c, ev in cases:
        out, detail = [], {}
        while res[pos] != "end":
            if res[pos].startswith("#"):
                detail[len(out) - 1] = res[pos][1:]
            else:
                out.append([int(x) for x in res[pos].split()])
            pos += 1
        pos += 1
        assert len(out) == len(ev)
        lines.append(json.dumps({"child": c, "events": ev, "out": out, "detail": detail}, separators=(",", ":")))
    raw = ("\n".join(lines) + "\n").encode()
    (HERE / "interp.jsonl.gz").write_bytes(gzip.compress(raw, compresslevel=9, mtime=0))
    n_viol = sum(1 for line in lines if '"detail":{}' not in line)
    print(f"interp.jsonl.gz: {len(lines)} streams ({n_viol} with violations), {len(raw)} bytes raw")


if __name__ == "__main__":
    main()
