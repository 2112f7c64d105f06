#!/usr/bin/env python3
"""Regenerates the golden fixtures in this directory from the *patched reference core*.

Run in the build container (where /root/reference exists):
    ./oracle/ref_build.sh && python tests/golden/gen_golden.py

Every fixture is the verbatim JSON-lines output of oracle/_ref/refdrv (see
oracle/refdrv.cpp for what each mode calls in the reference), gzip-compressed.
The GPU box never regenerates these; tests only read them.
"""
import gzip
import pathlib
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
DRV = REPO / "oracle" / "_ref" / "refdrv"
FIX = pathlib.Path("/root/reference/proj/data/fixtures")


def run(args, name):
    out = subprocess.run([str(DRV)] + args, check=True, capture_output=True).stdout
    (HERE / name).write_bytes(gzip.compress(out, compresslevel=9, mtime=0))
    print(f"{name}: {len(out)} bytes raw")


def main():
    if not DRV.exists():
        sys.exit("build oracle/_ref first: ./oracle/ref_build.sh")
    run(["dag", str(FIX)], "dag.jsonl.gz")
    run(["batch", str(FIX)], "batch.jsonl.gz")
    run(["toy"], "toy.jsonl.gz")
    run(["free"], "free.jsonl.gz")
    logs = []
    for seed in range(1, 7):
        for rec in (0, 8):
            logs.append((seed * 10 + rec, 400, rec))
    logs.append((777, 3000, 8))
    for seed, ops, rec in logs:
        run(["kv", str(seed), str(ops), str(rec)], f"kv_{seed}_{ops}_{rec}.jsonl.gz")


if __name__ == "__main__":
    main()
