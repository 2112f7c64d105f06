"""Host cost of one C4 decode step (2048 branches): time of the st.append and attention.decode calls
(enqueue only, and with a sync after each), over 40 steps."""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import bench  # noqa: E402


def main():
    import paper_2506_09991_b200 as mv
    wl = bench.WORKLOADS["c4"]
    dev = torch.device("cuda")
    R = wl["total_requests"]
    st, handles, pos0, rnd = bench.build_workload(mv, torch, R, dev, 0, wl["prefix"], wl["branches"], wl["branch_len"],
                                                  80)
    n = len(handles)
    handles = mv.kv.handle_array(handles)
    q = rnd(n, 40, 128)
    k = rnd(n, 8, 128)
    v = rnd(n, 8, 128)
    toks = torch.full((n,), 13, dtype=torch.int32, device=dev)
    out = torch.empty(n, 40, 128, dtype=torch.bfloat16, device=dev)
    base = torch.tensor(pos0, dtype=torch.int32, device=dev)
    ta, td, tas, tds = [], [], [], []
    for i in range(40):
        p = base + i
        torch.cuda.synchronize()
        a = time.perf_counter()
        st.append(handles, toks, p, 0, k, v)
        b = time.perf_counter()
        mv.attention.decode(st, handles, q, p, out=out)
        c = time.perf_counter()
        torch.cuda.synchronize()
        d = time.perf_counter()
        ta.append(b - a)
        td.append(c - b)
        tds.append(d - a)
    ta, td, tds = (np.array(x[5:]) * 1e3 for x in (ta, td, tds))
    print(f"append enqueue {ta.mean():.3f} ms, decode enqueue {td.mean():.3f} ms, step with sync {tds.mean():.3f} ms")


if __name__ == "__main__":
    main()
