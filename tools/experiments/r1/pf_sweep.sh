#!/bin/bash
# decode L2-prefetch sweep: time (bench, 64 steps) for head/tail settings
for cfg in "32 1" "0 0" "16 0" "32 0" "64 0" "8 1"; do
  set -- $cfg
  MV_DECODE_PF_HEAD=$1 MV_DECODE_PF_TAIL=$2 timeout 200 python bench.py --steps 64 --warmup 5 --cpu-seconds 0.2 > gpurun_out/pf_$1_$2.log 2>&1
  python - "$1" "$2" <<'PY'
import json, sys
l = json.loads(open(f"gpurun_out/pf_{sys.argv[1]}_{sys.argv[2]}.log").read().strip().splitlines()[-1])
print("head", sys.argv[1], "tail", sys.argv[2], "att_ms", round(l["roofline"]["launch_ms"], 4), "GB/s", round(l["roofline"]["achieved"]))
PY
done
