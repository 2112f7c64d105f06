import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, gzip, json
import paper_2506_09991_b200 as mv
import test_toy_gpu as T
import oracle
from paper_2506_09991_b200.host.tokenize import tokenize
gold = {json.loads(l)["name"]: json.loads(l) for l in gzip.open("tests/golden/toy.jsonl.gz", "rt")}
c = gold["t1_c1"]
ref, toy = T.gpu_toy(mv, c)
ids = tokenize(T.c1_text())
err, pos, _, _ = oracle.build_dag(ids)
want = ref.forward(ids, pos, oracle.mask_dense(ids))
import time, torch
f = toy.forward(ids).cpu().numpy(); t0 = time.perf_counter(); f = toy.forward(ids).cpu().numpy(); t1 = time.perf_counter()
r, st = toy.run_forced(ids); r = r.cpu().numpy(); t2 = time.perf_counter()
print("n", len(ids), "forward max err", np.abs(f - want).max(), "run_forced max err", np.abs(r - want).max(), "steps", st["steps"], "logit scale", np.abs(want).max())
print("forward s", t1 - t0, "run_forced s", t2 - t1)
