"""Diagnostic: random 16K-lane case, sentinel outputs, per library build variant."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from oracle import interp as o
import paper_2506_09991_b200 as mv
from paper_2506_09991_b200.interp import _ptr, _stream

rng = np.random.default_rng(11)
n, steps = 16384, 48
pool = np.array([*range(10), 10, 11, 12, 13, -1, -2], np.int32)
w = np.array([3, 1, 3, 2, 4, 4, 2, 2, 2, 2, 3, 3, 3, 3, 2, 1], np.float64)
ev = rng.choice(pool, size=(steps, n), p=w / w.sum()).astype(np.int32)
child = rng.integers(0, 2, n).astype(np.int32)
want = np.stack([np.array(o.run(child[j], ev[:, j])[0])[:, 0] for j in range(n)], 1)
for name in ("main",):
    L = mv.lib if name == "main" else ctypes.CDLL(f"tools/debug/libinterp_{name}.so")
    for chunks in ((48,), (20, 28), (1,) * 48):
        st = torch.empty((n, 2), dtype=torch.int32, device="cuda")
        assert L.mv_interp_init(_ptr(st), n, _ptr(torch.from_numpy(child).cuda()), _stream()) == 0
        acts, s0 = [], 0
        for c in chunks:
            d = torch.from_numpy(ev[s0:s0 + c].copy()).cuda()
            a = torch.full_like(d, -7)
            r = torch.full_like(d, -7)
            assert L.mv_interp_feed(_ptr(st), n, _ptr(d), c, _ptr(a), _ptr(r), _ptr(None), _ptr(None), _stream()) == 0
            acts.append(a)
            s0 += c
        a = torch.cat(acts).cpu().numpy()
        unw = int((a == -7).sum())
        bad = np.argwhere(a != want)
        print(name, chunks[:2], "unwritten", unw, "mismatch", len(bad), bad[:4].tolist())
