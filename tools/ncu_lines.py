#!/usr/bin/env python3
"""Stall samples of an ncu report aggregated per CUDA source line (needs -lineinfo), plus the
top SASS addresses with their source line.  usage: ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kfilt = ["--kernel-name", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *kfilt, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, line, src = None, None, None
per_line, per_addr = {}, []
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No"):
        continue
    try:
        samples = int(row[4])
    except (ValueError, IndexError):
        continue
    if row[0]:
        line, src = int(row[0]), row[1].strip()
        per_line[(fname, line)] = (samples, src)
    elif row[2].startswith("0x"):
        per_addr.append((samples, row[2][-5:], row[3][:60], f"{fname}:{line}"))
tot = sum(s for s, _ in per_line.values()) or 1
print(f"per source line ({tot} samples):")
for (f, l), (s, src) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"  {100.0 * s / tot:5.1f}% {f}:{l:<5d} {src[:90]}")
print("top SASS:")
for s, a, ins, where in sorted(per_addr, reverse=True)[:top]:
    print(f"  {100.0 * s / tot:5.1f}% {a} {ins:60s} {where}")
