#!/bin/bash
# ncu --set full (source-correlated) of decode_tc on C2 and C4 and of prefill_tc3 on C3, for tools/ncu_lines.py
o=gpurun_out/${1:-lines}; mkdir -p $o
ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 15 -c 1 -o $o/c2_decode \
    python bench.py --steps 20 --warmup 5 --extras none --cpu-seconds 0 > $o/c2.log 2>&1; echo "c2 rc=$?" >> $o/rc.txt
ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 3 -c 1 -o $o/c4_decode \
    python bench.py --workload c4 --steps 3 --warmup 3 --extras none --cpu-seconds 0 > $o/c4.log 2>&1; echo "c4 rc=$?" >> $o/rc.txt
ncu --set full --clock-control none --import-source on -k regex:prefill_tc3 -s 2 -c 1 -o $o/c3_prefill \
    python tools/bench_prefill.py > $o/c3.log 2>&1; echo "c3 rc=$?" >> $o/rc.txt
