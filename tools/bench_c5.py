#!/usr/bin/env python3
"""Reduce-merge stress (BASELINE configs[4]): prefix 4,096; 16 rounds of
{fork 128; append 64 tokens per branch; merge in ordinal order; append 16 Reduce tokens}; then
256 decode steps over the merged context (final 135,424 tokens + 256).

Reports per-op latency (host wall clock around each call + device sync: what an engine waits)
for fork / append / merge / release, that fork and merge moved 0 KV bytes, and the decode HBM
rate over the merged KV (CUDA events).  The reference arm (oracle/_ref/refdrv c5, the patched
reference RadixStore, 1 thread, 16-byte records) is timed on a bounded number of rounds because
its bookkeeping grows quadratically; its round count is printed."""
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main(rounds=16, B=128, path=64, red=16, prefix=4096, decode_steps=256, ref_rounds=6):
    import paper_2506_09991_b200 as mv
    hq, hkv = 40, 8
    total = prefix + rounds * (B * path + red)
    pages = total // 16 + rounds * B * 2 + decode_steps // 16 + 4096
    st = mv.kv.PagedStore(num_pages=pages, layers=1, kv_heads=hkv, table_entries=1 << 23)
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    rnd = lambda *s: (torch.rand(*s, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)  # noqa: E731
    pool_k, pool_v = rnd(B * path, hkv, 128), rnd(B * path, hkv, 128)
    tok = torch.full((B * path,), 11, dtype=torch.int32, device="cuda")
    t = {"fork": [], "append": [], "merge": [], "release": [], "reduce_append": []}
    copied = 0

    def timed(key, fn):
        torch.cuda.synchronize()
        a = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        t[key].append((time.perf_counter() - a) * 1e6)
        return r

    cur = st.create()
    st.append_many(cur, tok[:1].expand(prefix).contiguous(), torch.arange(prefix, dtype=torch.int32, device="cuda"), 0,
                   rnd(prefix, hkv, 128), rnd(prefix, hkv, 128))
    L = prefix
    pos_path = torch.arange(L, L + path, dtype=torch.int32, device="cuda")
    for r in range(rounds):
        kids = timed("fork", lambda: st.fork(cur, B))
        copied += st.stats().bytes_copied_on_last_op
        pos_path = torch.arange(L, L + path, dtype=torch.int32, device="cuda")
        for k, h in enumerate(kids):
            timed("append", lambda: st.append_many(h, tok[:path], pos_path, 0, pool_k[k * path:(k + 1) * path],
                                                   pool_v[k * path:(k + 1) * path]))
        m = timed("merge", lambda: st.merge(cur, kids))
        copied += st.stats().bytes_copied_on_last_op
        for h in [cur] + kids:
            timed("release", lambda: st.release(h))
        L += path
        timed("reduce_append", lambda: st.append_many(m, tok[:red], torch.arange(L, L + red, dtype=torch.int32,
                                                                                  device="cuda"), 0, pool_k[:red],
                                                      pool_v[:red]))
        L += red
        cur = m
    assert st.length(cur) == total
    # decode over the merged KV
    qs, ks, vs = rnd(2, hq, 128), rnd(2, hkv, 128), rnd(2, hkv, 128)
    tok1 = torch.tensor([13], dtype=torch.int32, device="cuda")
    poss = [torch.tensor([L + s], dtype=torch.int32, device="cuda") for s in range(decode_steps + 3)]
    for s in range(3):
        st.append([cur], tok1, poss[s], 0, ks[s % 2:s % 2 + 1], vs[s % 2:s % 2 + 1])
        mv.attention.decode(st, [cur], qs[s % 2:s % 2 + 1], poss[s])
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for s in range(3, decode_steps + 3):
        st.append([cur], tok1, poss[s], 0, ks[s % 2:s % 2 + 1], vs[s % 2:s % 2 + 1])
        mv.attention.decode(st, [cur], qs[s % 2:s % 2 + 1], poss[s])
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / decode_steps
    ctx = total + 3 + decode_steps / 2
    gbs = ctx * hkv * 128 * 2 * 2 / (ms / 1e3) / 1e9
    res = {"workload": "configs[4]: prefix 4096, 16 rounds x {fork 128, 64 tokens per branch, ordinal merge, "
                       "16 Reduce tokens}, then 256 decode steps (40q/8kv, d128, bf16)",
           "final_context": total, "kv_bytes_copied_by_fork_and_merge": int(copied),
           "ours_us_per_op": {k: float(np.median(v)) for k, v in t.items()},
           "decode_ms_per_step": ms, "decode_hbm_gbs": gbs}
    ref = os.path.join(REPO, "oracle", "_ref", "refdrv")
    if os.path.exists(ref):
        out = subprocess.run([ref, "c5", str(ref_rounds), "16"], capture_output=True, text=True, timeout=600).stdout
        res["reference_cpu_1thread"] = json.loads(out.strip().splitlines()[-1])
    print(json.dumps(res))
    return res


if __name__ == "__main__":
    main()
