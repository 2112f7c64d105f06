#!/usr/bin/env python3
"""Host-side cost of one decode step's API calls when the GPU is idle (the e2e setting: the
caller synchronises every step), on the bench C2 workload."""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import bench  # noqa: E402
import paper_2506_09991_b200 as mv  # noqa: E402


def main(steps=200):
    dev = torch.device("cuda", 0)
    st, handles, pos0, rnd = bench.build_workload(mv, torch, 16, dev, 0, steps_total=steps + 20)
    n = len(handles)
    if os.environ.get("MV_HANDLE_ARRAY", "1") == "1":
        handles = mv.kv.handle_array(handles)
    q, k, v = rnd(n, 40, 128), rnd(n, 8, 128), rnd(n, 8, 128)
    toks = torch.full((n,), 13, dtype=torch.int32, device=dev)
    out = torch.empty(n, 40, 128, dtype=torch.bfloat16, device=dev)
    base = torch.tensor(pos0, dtype=torch.int32, device=dev)
    pos = [base + i for i in range(steps + 10)]
    for i in range(5):
        st.append(handles, toks, pos[i], 0, k, v)
        mv.attention.decode(st, handles, q, pos[i], out=out)
    torch.cuda.synchronize()
    t = {"append": [], "decode": [], "sync": []}
    for s in range(5, steps):
        a = time.perf_counter()
        st.append(handles, toks, pos[s], 0, k, v)
        b = time.perf_counter()
        mv.attention.decode(st, handles, q, pos[s], out=out)
        c = time.perf_counter()
        torch.cuda.synchronize()
        d = time.perf_counter()
        t["append"].append(b - a)
        t["decode"].append(c - b)
        t["sync"].append(d - c)
    for kk, vv in t.items():
        print(f"{kk:8s} median {np.median(vv) * 1e6:8.1f} us  p90 {np.percentile(vv, 90) * 1e6:8.1f} us")


if __name__ == "__main__":
    main()
