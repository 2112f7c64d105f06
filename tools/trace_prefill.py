#!/usr/bin/env python3
"""Prefill timeline (MV_PREFILL_TRACE=file, prefill_tc.cu): head-0 CTA of each q-tile pair.
per k step j: [0] MMA got P_A, [1] MMA issued PV_A + QK_A(j+1), [2] MMA got P_B, [3] MMA issued
PV_B + QK_B(j+1), [4]/[5] softmax A saw S / released P, [6]/[7] softmax B saw S / released P."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64).reshape(-1, 272)
t = t[t[:, 0] > 0]
steps = t[:, 16:].reshape(len(t), 32, 8)


def stat(name, x):
    x = x[(x > 0) & (x < 1e7)]
    if len(x):
        print(f"{name:40s} mean {x.mean()/1e3:7.3f} us  p50 {np.median(x)/1e3:7.3f}  p90 {np.percentile(x, 90)/1e3:7.3f}")


ok = steps[:, :, 3] > 0
stat("softmax A busy (S seen -> P)", (steps[:, :, 5] - steps[:, :, 4])[ok])
stat("softmax B busy", (steps[:, :, 7] - steps[:, :, 6])[ok])
stat("MMA: P_A ready -> issued A's MMAs", (steps[:, :, 1] - steps[:, :, 0])[ok])
stat("MMA: waits for P_B", (steps[:, :, 2] - steps[:, :, 1])[ok])
stat("MMA: P_B ready -> issued B's MMAs", (steps[:, :, 3] - steps[:, :, 2])[ok])
okn = ok[:, 1:] & ok[:, :-1]
stat("k-step period (MMA got P_A j -> j+1)", (steps[:, 1:, 0] - steps[:, :-1, 0])[okn])
stat("softmax A idle (P_A(j) -> S_A(j+1))", (steps[:, 1:, 4] - steps[:, :-1, 5])[okn])
stat("MMA waits P_A (B issued -> P_A next)", (steps[:, 1:, 0] - steps[:, :-1, 3])[okn])
print("CTA durations (us):", np.round(np.sort((steps[:, :, 3].max(1) - t[:, 0]) / 1e3)[-5:], 1), "k tiles:", t[:, 1].min(), t[:, 1].max())
