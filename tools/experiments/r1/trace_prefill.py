#!/usr/bin/env python3
"""Prefill timeline of CTA 0 (build with tools/ab_build.sh trace -DMV_PF_TRACE=1, run with
MV_PREFILL_TRACE=file).  Per k step g (clock64 cycles): [0] issuer saw P_A, [1] issued P_A.V +
next Q_A.K^T, [2] saw P_B, [3] issued P_B.V + next Q_B.K^T, [4]/[5] softmax A saw S / released P,
[6]/[7] softmax B saw S / released P (0 when the half skipped the tile)."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64).reshape(-1, 16)
n = int((t[:, 3] > 0).sum())
t = t[:n]
base = t[t > 0].min()


def stat(name, x):
    x = x[(x > 0) & (x < 1e6)]
    if len(x):
        print(f"{name:44s} mean {x.mean():8.0f} cyc  p50 {np.median(x):8.0f}  p90 {np.percentile(x, 90):8.0f}  n={len(x)}")


okA, okB = (t[:, 4] > 0) & (t[:, 5] > 0), (t[:, 6] > 0) & (t[:, 7] > 0)
stat("softmax A busy (S seen -> P released)", (t[:, 5] - t[:, 4])[okA])
stat("softmax B busy", (t[:, 7] - t[:, 6])[okB])
stat("issuer: P_A seen -> A MMAs issued", (t[:, 1] - t[:, 0])[t[:, 0] > 0])
stat("issuer: P_B seen -> B MMAs issued", (t[:, 3] - t[:, 2])[t[:, 2] > 0])
stat("issuer: A issued -> P_B seen (waits)", (t[:, 2] - t[:, 1])[t[:, 2] > 0])
stat("k-step period (step end -> step end)", np.diff(t[:, 3]))
stat("S_A(g+1) seen - A issued(g)", (t[1:, 4] - t[:-1, 1])[(t[1:, 4] > 0)])
stat("S_B(g+1) seen - B issued(g)", (t[1:, 6] - t[:-1, 3])[(t[1:, 6] > 0)])
for x, nm in ((0, "A"), (1, "B")):
    o = 8 + 3 * x
    ok = (t[:, o] > 0) & (t[:, o + 2] > 0)
    stat(f"softmax {nm}: S seen -> S in registers", (t[:, o] - t[:, 4 + 2 * x])[ok])
    stat(f"softmax {nm}: max / mask / rescale", (t[:, o + 1] - t[:, o])[ok])
    stat(f"softmax {nm}: exp + P stores", (t[:, o + 2] - t[:, o + 1])[ok])
    stat(f"softmax {nm}: wait st + arrive", (t[:, 5 + 2 * x] - t[:, o + 2])[ok])
print(f"steps {n}, span {(t[:, 3].max() - base) / 1e3:.1f} kcyc")
if len(sys.argv) > 2:
    for g in range(min(n, int(sys.argv[2]))):
        print(g, " ".join(f"{(v - base) if v else -1:8d}" for v in t[g][:8]))
