#!/usr/bin/env python3
"""CTA 0's timeline of one decode launch (run against tools/ab/trace/libmvb200.so, see ab_decode.py):
MV_LIB=tools/ab/trace/libmvb200.so python tools/experiments/decode_timeline.py c2|c4 out.npy"""
import ctypes
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import bench  # noqa: E402
import paper_2506_09991_b200 as mv  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1]]
dev = torch.device("cuda", 0)
R = 16 if sys.argv[1] == "c2" else 64
st, hs, pos0, rnd = bench.build_workload(mv, torch, R, dev, 0, wl["prefix"], wl["branches"], wl["branch_len"], 16)
n = len(hs)
hs = mv.kv.handle_array(hs)
q, k, v = rnd(n, 40, 128), rnd(n, 8, 128), rnd(n, 8, 128)
tok = torch.full((n,), 13, dtype=torch.int32, device=dev)
base = torch.tensor(pos0, dtype=torch.int32, device=dev)
for i in range(6):
    st.append(hs, tok, base + i, 0, k, v)
    mv.attention.decode(st, hs, q, base + i)
torch.cuda.synchronize()
buf = np.zeros(24 * 256, np.uint64)
assert mv.lib.mv_debug_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
np.save(sys.argv[2], buf.reshape(24, 256))
print("saved", sys.argv[2], st.plan_info())
