#!/usr/bin/env python3
"""Analyse a decode per-item trace (MV_DECODE_TRACE=file): per CTA timeline of items."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(148, 64, 4).astype(np.int64)
start = t[:, 0, 0]
t0 = start[start > 0].min()
ends, items, busy, epi, gaps = [], [], [], [], []
for c in range(148):
    it = t[c, 1:63]
    n, last = 0, None
    for k in range(62):
        if it[k, 0] == 0 or it[k, 2] == 0:
            break
        n += 1
        busy.append(it[k, 2] - it[k, 0])
        epi.append(it[k, 3] - it[k, 2])
        if last is not None:
            gaps.append(it[k, 0] - last)
        last = it[k, 3]
    items.append(n)
    ends.append(last - t0 if last else 0)
ends = np.array(ends)
print(f"CTA end min/med/max {ends.min()/1e3:.1f}/{np.median(ends)/1e3:.1f}/{ends.max()/1e3:.1f} us; "
      f"items/CTA {min(items)}..{max(items)}; start skew {(start.max()-start.min())/1e3:.1f} us")
print(f"item pages-phase mean {np.mean(busy)/1e3:.2f} us (p90 {np.percentile(busy,90)/1e3:.2f}); "
      f"epilogue mean {np.mean(epi)/1e3:.2f}; gap to next item mean {np.mean(gaps)/1e3:.2f} max {np.max(gaps)/1e3:.2f}")
first = np.array([t[c, 1, 0] - t[c, 0, 0] for c in range(148)])
print(f"first item ready after CTA start: mean {first.mean()/1e3:.2f} us, max {first.max()/1e3:.2f}")
