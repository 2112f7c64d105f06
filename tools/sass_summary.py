#!/usr/bin/env python3
"""SASS evidence per kernel of the built library: tcgen05 MMAs (UTCHMMA / UTCQMMA), TMA loads / stores (UTMALDG / UTMASTG),
bulk copies (UBLKCP), TMEM loads / stores (LDTM / STTM), tcgen05 commits (UTCBAR), MUFU.EX2, legacy
HMMA (mma.sync) and local-memory traffic (LDL / STL).  usage: sass_summary.py [lib.so] > out.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2506_09991_b200/libmvb200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
keys = ["UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "UTCBAR", "UTCCP", "MUFU.EX2", "HMMA", "LDL", "STL",
        "SYNCS.PHASECHK", "ELECT"]
cur, counts, order = None, {}, []
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        order.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(2)
    counts[cur]["_total"] += 1
    for k in keys:
        if op == k or op.startswith(k + ".") or (k in ("LDTM", "STTM") and op.startswith(k)):
            counts[cur][k] += 1


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    d = d.replace("(anonymous namespace)::", "").replace("void ", "")
    return re.sub(r"\(.*", "", d)


print(f"# SASS summary of {lib} (cuobjdump -sass; static instruction counts per kernel)")
print(f"{'kernel':44s} {'total':>6s} " + " ".join(f"{k:>9s}" for k in keys))
for f in order:
    c = counts[f]
    print(f"{short(f)[:44]:44s} {c['_total']:6d} " + " ".join(f"{c[k]:9d}" for k in keys))
