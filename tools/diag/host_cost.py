#!/usr/bin/env python3
"""Host-side cost per decode step (bench C2 workload): time spent in each API call while
enqueueing (no syncs), to see what bounds the step when the GPU is faster than the host."""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import bench  # noqa: E402
import paper_2506_09991_b200 as mv  # noqa: E402
from paper_2506_09991_b200.kv import _u64_array  # noqa: E402


def main(steps=300):
    dev = torch.device("cuda", 0)
    st, handles, pos0, rnd = bench.build_workload(mv, torch, 16, dev, 0, steps_total=steps + 20)
    n = len(handles)
    q, k, v = rnd(n, 40, 128), rnd(n, 8, 128), rnd(n, 8, 128)
    toks = torch.full((n,), 13, dtype=torch.int32, device=dev)
    out = torch.empty(n, 40, 128, dtype=torch.bfloat16, device=dev)
    base = torch.tensor(pos0, dtype=torch.int32, device=dev)
    pos = [base + i for i in range(steps + 10)]
    for i in range(5):
        st.append(handles, toks, pos[i], 0, k, v)
        mv.attention.decode(st, handles, q, pos[i], out=out)
    torch.cuda.synchronize()
    t = {"u64_array": [], "append": [], "decode": [], "event": []}
    ev = torch.cuda.Event(enable_timing=True)
    for s in range(5, steps):
        a = time.perf_counter()
        _u64_array(handles)
        b = time.perf_counter()
        st.append(handles, toks, pos[s], 0, k, v)
        c = time.perf_counter()
        mv.attention.decode(st, handles, q, pos[s], out=out)
        d = time.perf_counter()
        ev.record()
        e = time.perf_counter()
        t["u64_array"].append(b - a)
        t["append"].append(c - b)
        t["decode"].append(d - c)
        t["event"].append(e - d)
        if s % 50 == 0:
            torch.cuda.synchronize()  # keep the GPU queue short so we time the host, not back-pressure
    for kk, vv in t.items():
        print(f"{kk:10s} median {np.median(vv) * 1e6:8.1f} us  p90 {np.percentile(vv, 90) * 1e6:8.1f} us")


if __name__ == "__main__":
    main()
