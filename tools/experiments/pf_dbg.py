"""debug: per-row error of the prefill vs the oracle on fixture t1 (sum-guard experiment)"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import oracle
import paper_2506_09991_b200 as mv
from conftest import load_jsonl
from mvtest import bf16_to_f64, sym_bf16
t1 = next(c for c in load_jsonl("dag.jsonl.gz") if c["name"] == "fixture:t1.txt")
tokens = t1["tokens"]; n = len(tokens); hq, hkv = 8, 2
spec = mv.dag.build_visibility(tokens)
q = sym_bf16(31, (n, hq, 128)); k = sym_bf16(32, (n, hkv, 128)); v = sym_bf16(33, (n, hkv, 128))
out = mv.attention.prefill(q.cuda(), k.cuda(), v.cuda(), spec.positions, spec.excl, out_dtype=torch.float32)
torch.cuda.synchronize()
_, pos, _, _ = oracle.build_dag(tokens)
rows = np.arange(n)
ref = oracle.attn_prefill_tokens(oracle.rope(bf16_to_f64(q), pos), oracle.rope(bf16_to_f64(k), pos), bf16_to_f64(v), tokens, rows)
got = out.cpu().numpy()
e = np.abs(got - ref)
print("n", n, "D", spec.max_depth, "max err", e.max())
er = e.max(axis=(1, 2)); bad = np.nonzero(er > 2e-3)[0]
print("bad rows", len(bad), bad[:40])
eh = e.max(axis=(0, 2)); print("per head", eh)
ed = e.max(axis=(0, 1)); print("dims bad", np.nonzero(ed > 2e-3)[0][:40])
if len(bad): r = bad[0]; print("row", r, "got", got[r, 0, :6], "ref", ref[r, 0, :6])
