#!/usr/bin/env python3
"""Round-1 K5 report, re-examined: build tools/experiments/k5_multistep.cu (multi-step loop, switch dispatch)
at -O3 / -O1 / -G and compare every action of 16K random lanes x 48 steps with the oracle restatement
(oracle/interp.py).  build: python tools/experiments/k5_multistep.py build; run (GPU): ... run"""
import ctypes
import pathlib
import subprocess
import sys

import numpy as np

REPO = pathlib.Path(__file__).resolve().parents[2]
OUT = REPO / "tools" / "ab" / "k5"
VARIANTS = {"O3_opaque": ["-O3"], "O3": ["-O3"], "O1": ["-O1", "-Xptxas", "-O1"], "G": ["-G"], "O3_noptxopt": ["-O3", "-Xptxas", "-O0"]}


def build():
    OUT.mkdir(parents=True, exist_ok=True)
    for name, fl in VARIANTS.items():
        cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-shared",
               "-Xcompiler", "-fPIC", "-lineinfo" if name != "G" else "-g", f"-I{REPO / 'include'}",
               f"-I{REPO / 'paper_2506_09991_b200' / 'csrc'}", *fl, str(REPO / ("tools/experiments/k5_multistep_opaque.cu" if name == "O3_opaque" else "tools/experiments/k5_multistep.cu")),
               "-o", str(OUT / f"k5_{name}.so")]
        subprocess.run(cmd, check=True)
        print("built", name)


def run(only=None, single=False, uniform=False):
    import torch
    sys.path.insert(0, str(REPO))
    from oracle import interp as o
    rng = np.random.default_rng(11)
    n, steps = 16384, 48
    pool = np.array([*range(10), 10, 11, 12, 13, -1, -2], np.int32)
    w = np.array([3, 1, 3, 2, 4, 4, 2, 2, 2, 2, 3, 3, 3, 3, 2, 1], np.float64)
    ev = rng.choice(pool, size=(steps, n), p=w / w.sum()).astype(np.int32)
    child = rng.integers(0, 2, n).astype(np.int32)
    if uniform:  # every lane the same stream: the phase dispatch never diverges inside a warp
        ev[:] = ev[:, :1]
        child[:] = child[0]
    want = np.stack([np.array(o.run(child[j], ev[:, j])[0])[:, 0] for j in range(n)], 1)
    for name in ([only] if only else VARIANTS):
        L = ctypes.CDLL(str(OUT / f"k5_{name}.so"))
        st = torch.zeros((n, 2), dtype=torch.int32, device="cuda")
        st[:, 0] = torch.from_numpy(child).cuda() << 8
        d = torch.from_numpy(ev).cuda()
        a = torch.full_like(d, -7)
        r = torch.full_like(d, -7)
        P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        if single:  # one step per launch, the same binary
            rc = 0
            for k in range(steps):
                rc |= L.k5x_run(P(st), n, P(d[k:k + 1]), 1, P(a[k:k + 1]), P(r[k:k + 1]))
        else:
            rc = L.k5x_run(P(st), n, P(d), steps, P(a), P(r))
        a = a.cpu().numpy()
        bad = np.argwhere(a != want)
        unw = int((a == -7).sum())
        first = bad[0].tolist() if len(bad) else None
        warps = sorted({int(x) // 32 for x in bad[:, 1]})[:8] if len(bad) else []
        print(f"{name}{' single-step launches' if single else ''}{' uniform lanes' if uniform else ''}: rc {rc} unwritten {unw} mismatches {len(bad)} first {first} lanes' warps {warps}", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        mode = sys.argv[3] if len(sys.argv) > 3 else ""
        run(sys.argv[2] if len(sys.argv) > 2 else None, mode == "single", mode == "uniform")
