"""Synthetic workload generators shared by bench.py and the tests (host-only, no GPU).

nested_16k: BASELINE configs[2], a 16,384-token structured tag stream with
nested Parallel blocks, in tokenizer ids (tokenizer.cpp:56-63: 0..9 tags, >= 10 text).
"""
from __future__ import annotations

import numpy as np


def nested_16k(seed=0, n_target=16384):
    """BASELINE configs[2]: prefix 2048, an outer block of 4 paths, each path = head text + an
    inner block of 4 paths + continuation; word counts chosen so n == 16384 exactly."""
    rng = np.random.default_rng(seed)
    words = lambda k: list(10 + rng.integers(0, 4000, size=k))  # noqa: E731
    P_OPEN, P_CLOSE, G_OPEN, G_CLOSE, O_OPEN, O_CLOSE, PATH, PATH_C, C_OPEN, C_CLOSE = range(10)

    def block(path_bodies, outline_words=6, concl=24):
        t = [P_OPEN, G_OPEN]
        for _ in path_bodies:
            t += [O_OPEN] + words(outline_words) + [O_CLOSE]
        t += [G_CLOSE]
        for body in path_bodies:
            t += [PATH] + body + [PATH_C]
        return t + [C_OPEN] + words(concl) + [C_CLOSE, P_CLOSE]

    def build(inner_len):
        outer_paths = []
        for _ in range(4):
            inner = block([words(inner_len) for _ in range(4)])
            outer_paths.append(words(256) + inner + words(64))
        return words(2048) + block(outer_paths)

    lo, hi = 1, 2000
    while lo < hi:  # largest inner path length with n <= target
        mid = (lo + hi + 1) // 2
        if len(build(mid)) <= n_target:
            lo = mid
        else:
            hi = mid - 1
    toks = build(lo)
    toks = words(n_target - len(toks)) + toks  # pad the prefix to hit n exactly
    return [int(x) for x in toks]
