"""K5 timing: one decode step of the device tag interpreter over L lanes (CUDA events, 1 GPU).

Lanes = C2 (16 requests x 9 lanes), C4 (64 requests x 33 lanes) and 16K; events are a seeded
tag / text mix. Prints one JSON line per size: microseconds per step (launch-bound, not a
roofline kernel) and the bytes it touches (events + action + arg + state read/write)."""
import json

import numpy as np
import torch

import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import paper_2506_09991_b200 as mv  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    for lanes in (144, 2112, 16384):
        steps = 200
        ev = torch.from_numpy(rng.choice(np.array([*range(10), 10, 11, 12, 13, -1], np.int32),
                                         size=(steps, lanes)).astype(np.int32)).cuda()
        it = mv.interp.TagInterpreter(lanes, rng.integers(0, 2, lanes))
        for s in range(10):
            it.feed(ev[s])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for s in range(steps):
            it.feed(ev[s])
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / steps
        print(json.dumps({"kernel": "interp_kernel", "lanes": lanes, "us_per_step": us,
                          "bytes_per_step": lanes * (4 + 8 + 16), "note": "includes the per-call host path "
                          "(tensor allocation + ctypes); launch-bound"}))


if __name__ == "__main__":
    main()
