"""Diagnostic: sentinel-filled outputs, one launch; reports unwritten / wrong (step, lane)."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, "tests")
from conftest import load_jsonl
from test_interp import lanes_matrix
import paper_2506_09991_b200 as mv
from paper_2506_09991_b200.interp import _ptr, _stream

g = load_jsonl("interp.jsonl.gz")
ev, child = lanes_matrix(g)
n = len(g)
it = mv.interp.TagInterpreter(n, child)
d_ev = torch.from_numpy(ev).cuda()
act = torch.full_like(d_ev, -7)
arg = torch.full_like(d_ev, -7)
torch.cuda.synchronize()
mv.check(mv.lib.mv_interp_feed(_ptr(it.state), n, _ptr(d_ev), ev.shape[0], _ptr(act), _ptr(arg), _ptr(None), _ptr(None), _stream()))
torch.cuda.synchronize()
a = act.cpu().numpy()
print("unwritten", np.argwhere(a == -7)[:10].tolist(), int((a == -7).sum()))
for j, x in enumerate(g):
    want = np.array([r[0] for r in x["out"]])
    d = np.nonzero(a[: len(want), j] != want)[0]
    if d.size:
        print("lane", j, "first bad step", int(d[0]), "got", a[d[0]: d[0] + 3, j].tolist(), "want", want[d[0]: d[0] + 3].tolist())
print("events equal after", bool((d_ev.cpu().numpy() == ev).all()))
