#!/bin/bash
# Interleaved A/B of prefill builds: ab_run_prefill.sh <out> <variant>...  (tools/bench_prefill.py, 3 rounds)
o=gpurun_out/$1; shift; mkdir -p $o
for r in 1 2 3; do for v in "$@"; do
  MV_LIB=tools/ab/$v/libmvb200.so python tools/bench_prefill.py > $o/${v}_$r.json 2> $o/${v}_$r.err
done; done
