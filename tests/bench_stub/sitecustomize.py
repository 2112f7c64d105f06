"""Test-only stand-in for the CUDA library, loaded through PYTHONPATH by tests/test_bench_multirank.py:
registers a host-side `paper_2506_09991_b200` (page-table bookkeeping in Python, no kernels) so that
bench.py's multi-rank plumbing (torchrun relaunch, sharding, max-over-ranks timing, per-GPU arithmetic)
runs on CPU under gloo.  Never used by the product or the GPU tests."""
import importlib.util
import pathlib
import sys
import time
import types

import numpy as np

REPO = pathlib.Path(__file__).resolve().parents[2]

pkg = types.ModuleType("paper_2506_09991_b200")
pkg.__path__ = []
spec = importlib.util.spec_from_file_location("paper_2506_09991_b200.shard", REPO / "paper_2506_09991_b200" / "shard.py")
shard = importlib.util.module_from_spec(spec)
sys.modules["paper_2506_09991_b200.shard"] = shard
spec.loader.exec_module(shard)


class PagedStore:
    def __init__(self, num_pages, layers=0, kv_heads=0, table_entries=0, **_):
        self.len, self.next, self.lineage = {}, 1, {}

    def create(self):
        h = self.next
        self.next += 1
        self.len[h] = 0
        return h

    def append_many(self, h, tokens, positions=None, layer=0, k=None, v=None, n=None):
        self.len[h] += len(tokens) if tokens is not None else n

    def append(self, handles, tokens, positions=None, layer=0, k=None, v=None):
        for h in handles:
            self.len[int(h)] += 1

    def fork(self, h, n):
        kids = []
        for _ in range(n):
            c = self.create()
            self.len[c] = self.len[h]
            self.lineage[c] = h
            kids.append(c)
        return kids

    def release(self, h):
        self.len.pop(h)

    def decode_kernel_timing(self, max_calls):
        done, self.timed = getattr(self, "timed", 0), max_calls
        return [2.0] * done  # the stub's fixed "kernel" time

    def plan_info(self):
        roots = {}
        for c, p in self.lineage.items():
            if c in self.len:
                roots.setdefault(p, []).append(c)
        uniq = 0
        for p, kids in roots.items():
            shared = min(self.len[c] for c in kids) if kids else 0
            uniq += shared // 1  # prefix once
            uniq += sum(self.len[c] for c in kids) - len(kids) * shared
        return {"units": 0, "chunks": 0, "work_items": 0, "partial_slots": 0, "unique_kv_tokens": uniq,
                "naive_kv_tokens": sum(self.len.values())}


def handle_array(hs):
    return np.asarray([int(h) for h in hs], dtype=np.uint64)


def decode(store, handles, q, positions, layer=0, out=None, out_dtype=None):
    store.timed = getattr(store, "timed", 0)
    time.sleep(0.002)  # a fixed "kernel" time per step: the per-GPU arithmetic is then predictable
    return out


pkg.kv = types.SimpleNamespace(PagedStore=PagedStore, handle_array=handle_array)
pkg.attention = types.SimpleNamespace(decode=decode)
pkg.shard = shard
sys.modules["paper_2506_09991_b200"] = pkg
