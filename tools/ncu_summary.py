#!/usr/bin/env python3
"""Summarise an ncu report: key raw metrics + top stall sites (source page)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
kfilt = ["--kernel-name", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
raw = subprocess.run(["ncu", "-i", rep, *kfilt, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
print("kernel:", v[h.index("Kernel Name")][:90] if "Kernel Name" in h else "?")
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_utchmma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg"]
for name in want:
    if name in h:
        i = h.index(name)
        print(f"{name:80s} {v[i]} {u[i]}")
st = []
for i, name in enumerate(h):
    if "pcsamp_warps_issue_stalled" in name and not name.endswith("not_issued"):
        try:
            st.append((float(v[i].replace(",", "")), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
print("stalls:", ", ".join(f"{n}={int(x)}" for x, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, *kfilt, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
if len(rows) > 2:
    hdr = rows[1]
    iS, iA, iAd = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Address")
    data = []
    for k, row in enumerate(rows[2:]):
        try:
            data.append((int(row[iA]), row[iAd][-5:], row[iS][:100]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    print(f"top stall sites ({tot} samples):")
    for d in sorted(data, reverse=True)[:top]:
        print(f"  {100.0 * d[0] / tot:5.1f}% {d[1]} {d[2]}")
