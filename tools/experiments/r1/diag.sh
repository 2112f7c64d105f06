#!/bin/bash
# decode pipeline diagnostics: 0 normal, 1 skip math (pipeline only), 2 skip loads (math only)
for d in 0 1 2; do
  MV_DECODE_DIAG=$d timeout 200 python bench.py --steps 20 --warmup 5 --cpu-seconds 0.2 > gpurun_out/diag_$d.log 2>&1
  python - "$d" <<'PY'
import json, sys
d = sys.argv[1]
l = json.loads(open(f"gpurun_out/diag_{d}.log").read().strip().splitlines()[-1])
print("diag", d, "attn_ms", round(l["roofline"]["launch_ms"], 4), "GB/s", round(l["roofline"]["achieved"]))
PY
done
