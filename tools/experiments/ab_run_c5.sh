#!/bin/bash
# Interleaved A/B of the C5 sub-record (decode over the merged 135K context): ab_run_c5.sh <out> <variant>...
o=gpurun_out/$1; shift; mkdir -p $o
for r in 1 2 3; do for v in "$@"; do
  MV_LIB=tools/ab/$v/libmvb200.so python bench.py --gpus 1 --steps 5 --warmup 3 --extras c5 --cpu-seconds 0 > $o/${v}_$r.json 2> $o/${v}_$r.err
done; done
