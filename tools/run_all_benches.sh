#!/bin/bash
# Runs every configs[] measurement of this repo on one GPU and writes profiles/r01_summary.json:
#   configs[0] C1 toy parity (tests/test_toy_gpu.py), configs[1] C2 decode (bench.py),
#   configs[2] C3 prefill (tools/bench_prefill.py), configs[3] C4 wide decode (bench.py --workload c4),
#   configs[4] C5 reduce-merge stress (tools/bench_c5.py), and the reference CPU arm.
set -e
cd "$(dirname "$0")/.."
out=${1:-gpurun_out/summary}
mkdir -p "$out"
python bench.py > "$out/c2.json" 2> "$out/c2.err"
python bench.py --workload c4 --steps 100 --cpu-seconds 0 > "$out/c4.json" 2> "$out/c4.err"
python tools/bench_prefill.py > "$out/c3.json" 2> "$out/c3.err"
python tools/bench_c5.py > "$out/c5.json" 2> "$out/c5.err"
python bench.py --impl reference --steps 3 --warmup 3 > "$out/ref.json" 2> "$out/ref.err"
python -m pytest tests/test_toy_gpu.py -q > "$out/c1.txt" 2>&1 || true
python - "$out" <<'PY'
import json, sys
o = sys.argv[1]
last = lambda f: json.loads(open(f"{o}/{f}").read().strip().splitlines()[-1])
c2, c4, c3, c5, ref = last("c2.json"), last("c4.json"), last("c3.json"), last("c5.json"), last("ref.json")
s = {
  "C1_toy_parity": open(f"{o}/c1.txt").read().strip().splitlines()[-1],
  "C2_decode": {"tokens_per_s": c2["value"], "frac_hbm": c2["roofline"]["frac"], "e2e_tokens_per_s": c2["e2e"]["value"],
                "ms_per_step": c2["ms_per_step"], "clocks": c2["clocks"]},
  "C2_reference_cpu": {"tokens_per_s": ref["value"], "cores": ref["cpu_baseline"]["cores"]},
  "C3_prefill": {"tflops": c3["tflops"], "frac_bf16": c3["frac"], "ms": c3["ms"]},
  "C4_decode": {"tokens_per_s": c4["value"], "frac_hbm": c4["roofline"]["frac"]},
  "C5_stress": {"us_per_op": c5["ours_us_per_op"], "decode_ms_per_step": c5["decode_ms_per_step"],
                "decode_hbm_gbs": c5["decode_hbm_gbs"], "kv_bytes_copied": c5["kv_bytes_copied_by_fork_and_merge"],
                "reference": c5.get("reference_cpu_1thread")},
}
json.dump(s, open(f"{o}/summary.json", "w"), indent=1)
print(json.dumps(s, indent=1))
PY
