#!/usr/bin/env python3
"""Analyse a decode timeline (MV_DECODE_TRACE=file, decode.cu kTraceWords layout):
per global block g<64: [0+g] softmax saw S, [64+g] softmax released P, [128+g] MMA starts the
QK of g (waits for its pages), [192+g] QK of g committed; per unit i<32: [256+i] epilogue start,
[288+i] epilogue end, [320+i] stager claim."""
import sys

import numpy as np

W = 864
t = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
t = t.reshape(-1, W)
valid = t[:, 320] > 0
t = t[valid]
t0 = t[:, 320].min()
sm_seen, sm_rel, qk_s, qk_e = t[:, 0:64], t[:, 64:128], t[:, 128:192], t[:, 192:256]
ep_s, ep_e, claim = t[:, 256:288], t[:, 288:320], t[:, 320:352]


def stat(name, x):
    x = x[(x > -1e9) & (x < 1e9)]
    if len(x):
        print(f"{name:42s} mean {x.mean()/1e3:7.3f} us  p50 {np.median(x)/1e3:7.3f}  p90 {np.percentile(x, 90)/1e3:7.3f}")


def pairs(a, b):
    m = (a > 0) & (b > 0)
    return (b - a)[m]


stat("softmax busy (saw S -> released P)", pairs(sm_seen, sm_rel))
stat("softmax idle (released g-1 -> saw S g)", pairs(sm_rel[:, :-1], sm_seen[:, 1:]))
stat("MMA QK page wait (start -> commit)", pairs(qk_s, qk_e))
stat("QK commit -> softmax saw S", pairs(qk_e, sm_seen))
stat("block period (softmax seen g -> g+1)", pairs(sm_seen[:, :-1], sm_seen[:, 1:]))
qw = t[:, 352:416].astype(np.float64) / 1.965
stat("MMA QK issue (data ready) ns @1965MHz", qw[qk_e > 0] * 1.0)
ow = t[:, 416:480].astype(np.float64) / 1.965
stat("MMA PV issue ns @1965MHz", ow[sm_rel > 0] * 1.0)
tw = t[:, 608:672].astype(np.float64) / 1.965
stat("TMA issue per block ns (after empty)", tw[t[:, 544:608] > 0] * 1.0)
stat("TMA block issue -> QK commit", pairs(t[:, 544:608], qk_e))
for nm, o in (("softmax: masks+ld+exp (fast path) ns", 672), ("softmax: P store+wait ns", 736), ("softmax: compute total ns", 800)):
    x = t[:, o:o + 64].astype(np.float64) / 1.965
    stat(nm, x[x > 0] * 1.0)
stat("epilogue (incl. combine)", pairs(ep_s, ep_e))
stat("unit period (claim i -> i+1)", pairs(claim[:, :-1], claim[:, 1:]))
stat("first S after first claim", sm_seen[:, 0] - claim[:, 0])
last = np.max(np.where(ep_e > 0, ep_e, 0), axis=1)
print(f"CTA last epilogue end after t0: min {((last - t0).min())/1e3:.1f} med {np.median(last - t0)/1e3:.1f} "
      f"max {((last - t0).max())/1e3:.1f} us; units/CTA {int((claim > 0).sum(1).min())}..{int((claim > 0).sum(1).max())}")

if len(sys.argv) > 2:
    c = int(sys.argv[2])
    base = claim[c, 0]
    print(f"CTA {c} timeline (us after first claim): g | TMA start | S seen | P released | MMA got P | QK start | QK commit")
    for g in range(40):
        row = [t[c, 544 + g], t[c, g], t[c, 64 + g], t[c, 480 + g], t[c, 128 + g], t[c, 192 + g]]
        print(f"  {g:2d} " + " ".join(f"{(x - base) / 1e3:8.3f}" if x > 0 else "       -" for x in row))
