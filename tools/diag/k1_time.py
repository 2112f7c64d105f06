#!/usr/bin/env python3
"""K1 timing: dag.build_visibility on the C3 16K nested stream (CUDA events, warm)."""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
import paper_2506_09991_b200 as mv  # noqa: E402
from tools.workloads import nested_16k  # noqa: E402

toks = nested_16k()
t = torch.tensor(toks, dtype=torch.int32, device="cuda")
for _ in range(3):
    mv.dag.build_visibility(t)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    mv.dag.build_visibility(t)
e1.record()
torch.cuda.synchronize()
print(f"build_visibility n={len(toks)}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per call (incl. allocations)")

import cProfile  # noqa: E402
import pstats  # noqa: E402
import time  # noqa: E402

a = time.perf_counter()
for _ in range(20):
    mv.dag.build_visibility(t)
torch.cuda.synchronize()
print(f"wall per call {(time.perf_counter() - a) / 20 * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    mv.dag.build_visibility(t)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
