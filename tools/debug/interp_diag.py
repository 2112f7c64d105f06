"""Diagnostic: where the multi-step device interpreter diverges from the restatement."""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests")
from conftest import load_jsonl
from test_interp import lanes_matrix
from oracle import interp as o
import paper_2506_09991_b200 as mv

g = load_jsonl("interp.jsonl.gz")
ev, child = lanes_matrix(g)
print("steps", ev.shape)
for spawns in (False, True):
    for chunk in (ev.shape[0], 16, 1):
        it = mv.interp.TagInterpreter(len(g), child)
        acts = []
        for s0 in range(0, ev.shape[0], chunk):
            r = it.feed(torch.from_numpy(ev[s0:s0 + chunk]), spawns=spawns)
            acts.append(r[0].reshape(-1, len(g)))
        a = torch.cat(acts).cpu().numpy()
        bad = []
        for j, x in enumerate(g):
            want = np.array([r[0] for r in x["out"]])
            d = np.nonzero(a[: len(want), j] != want)[0]
            if d.size:
                bad.append((j, int(d[0]), len(want)))
        print("spawns", spawns, "chunk", chunk, "bad lanes", len(bad), bad[:8])
        if bad:
            j, s, n = bad[0]
            print("  events", ev[max(0, s - 4): s + 2, j].tolist(), "got", a[max(0, s - 4): s + 2, j].tolist(),
                  "want", [r[0] for r in g[j]["out"]][max(0, s - 4): s + 2])
