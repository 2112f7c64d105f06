#!/bin/bash
# Interleaved A/B of tools/ab/<variant>/libmvb200.so builds (tools/experiments/ab_files.py):
#   ab_run_files.sh <out> <variant>...   (two rounds, bench.py C2 + the c4 sub-record)
o=gpurun_out/$1; shift; mkdir -p $o
for r in 1 2; do for v in "$@"; do
  MV_LIB=tools/ab/$v/libmvb200.so python bench.py --gpus 1 --steps 20 --warmup 5 --extras c4 --cpu-seconds 0 > $o/${v}_$r.json 2> $o/${v}_$r.err
done; done
