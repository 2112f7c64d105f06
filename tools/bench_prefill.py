#!/usr/bin/env python3
"""Branch-masked prefill benchmark (BASELINE configs[2]): 16K nested structured sequence,
40 q / 8 kv heads, d128, bf16. Reports achieved TFLOP/s counting VISIBLE pairs only
(4 * 128 * Hq * popcount(mask)) against the measured bf16 peak."""
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main(iters=10):
    import paper_2506_09991_b200 as mv
    from tools.workloads import nested_16k
    toks = nested_16k()
    n, hq, hkv = len(toks), 40, 8
    g = torch.Generator(device="cuda").manual_seed(0)
    rnd = lambda *s: (torch.rand(*s, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)  # noqa: E731
    q, k, v = rnd(n, hq, 128), rnd(n, hkv, 128), rnd(n, hkv, 128)
    spec = mv.dag.build_visibility(toks)
    _, _, vis = mv.dag.tile_map(spec, 64)
    pairs = int(vis.item())
    out = torch.empty_like(q)
    ws = torch.empty(mv.lib.mv_prefill_workspace_size(n, hq, hkv), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        mv.attention.prefill(q, k, v, spec.positions, spec.excl, out=out, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        mv.attention.prefill(q, k, v, spec.positions, spec.excl, out=out, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    flops = 4.0 * 128 * hq * pairs
    try:
        peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except Exception:
        peak = 1590.0
    res = {"workload": "configs[2]: n=16384 nested 4x4 Parallel, 40q/8kv, d128, bf16", "visible_pairs": pairs,
           "density": pairs / (n * n), "ms": ms, "tflops": flops / ms / 1e9, "peak_tflops": peak,
           "frac": flops / ms / 1e9 / peak}
    print(json.dumps(res))
    return res


if __name__ == "__main__":
    main()
