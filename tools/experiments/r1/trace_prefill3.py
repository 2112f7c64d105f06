#!/usr/bin/env python3
"""Prefill v3 timeline of CTA 0 (tools/ab_build.sh trace3 -DMV_PF_TRACE=1; run with
MV_LIB=tools/ab/trace3/libmvb200.so MV_PREFILL_TRACE=file).  Per processed k tile g (clock64):
[0] issuer saw P(g), [1] issued PV(g) + QK(g+2), [2] softmax c0 saw S(g), [3] S in registers,
[4] row max exchanged, [5] c0 released P, [6] softmax c1 saw S, [7] c1 released P."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64).reshape(-1, 8)
n = int((t[:, 1] > 0).sum())
t = t[:n]


def stat(name, x):
    x = x[(x > 0) & (x < 1e6)]
    if len(x):
        print(f"{name:40s} mean {x.mean():8.0f}  p50 {np.median(x):8.0f}  p90 {np.percentile(x, 90):8.0f}  n={len(x)}")


stat("softmax c0: S seen -> P (busy)", t[:, 5] - t[:, 2])
stat("softmax c1: S seen -> P (busy)", t[:, 7] - t[:, 6])
stat("  c0: S seen -> in registers", t[:, 3] - t[:, 2])
stat("  c0: registers -> max exchanged", t[:, 4] - t[:, 3])
stat("  c0: exchanged -> P released", t[:, 5] - t[:, 4])
stat("issuer: P seen -> PV + QK issued", t[:, 1] - t[:, 0])
stat("issuer: P released (c0/c1 max) -> seen", t[:, 0] - np.maximum(t[:, 5], t[:, 7]))
stat("softmax idle: P(g) -> S(g+1) seen", t[1:, 2] - t[:-1, 5])
stat("S(g+2) seen - QK(g+2) issued", t[2:, 2] - t[:-2, 1])
stat("tile period (P seen g -> g+1)", np.diff(t[:, 0]))
print("tiles", n)
if len(sys.argv) > 2:
    b = t[t > 0].min()
    for g in range(min(n, int(sys.argv[2]))):
        print(g, " ".join(f"{(v - b) if v else -1:8d}" for v in t[g]))
