#!/bin/bash
# Round-2 evidence on one GPU (each ncu pass only after the same command ran clean without ncu):
#   bench lines (the driver's command), the configs[] summary (run_all_benches.sh), the decode launch
#   list with DRAM bytes at the bench's own contexts (roofline.traffic), the C4 decode_tc DRAM bytes,
#   ncu --set full of decode_tc and of prefill_tc3, the GPU test suite and smoke().
cd "$(dirname "$0")/.."
o=gpurun_out/${1:-r02}
mkdir -p $o
python bench.py --gpus 1 --steps 20 --warmup 5 > $o/bench_s20w5.json 2> $o/bench_s20w5.err; echo "bench_s20w5 rc=$?" >> $o/rc.txt
bash tools/run_all_benches.sh $o/summary > $o/summary.log 2>&1; echo "summary rc=$?" >> $o/rc.txt
python bench.py --steps 20 --warmup 5 --extras none > $o/plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"decode_tc|k_append_one|rope_q_tile|combine" -c 120 --csv --log-file $o/decode_launches.csv \
      python bench.py --steps 20 --warmup 5 --extras none > $o/ncu_launches.log 2>&1; echo "launches rc=$?" >> $o/rc.txt
python bench.py --workload c4 --steps 3 --warmup 3 --extras none --cpu-seconds 0 > $o/c4_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:decode_tc -c 6 --csv --log-file $o/c4_decode_tc_traffic.csv \
      python bench.py --workload c4 --steps 3 --warmup 3 --extras none --cpu-seconds 0 > $o/ncu_c4.log 2>&1; echo "c4 traffic rc=$?" >> $o/rc.txt
ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 15 -c 1 -o $o/decode_tc_full \
    python bench.py --steps 20 --warmup 5 --extras none > $o/ncu_decode.log 2>&1; echo "decode full rc=$?" >> $o/rc.txt
python tools/bench_prefill.py > $o/prefill_plain.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:prefill_tc3 -s 2 -c 1 -o $o/prefill_tc3_full \
      python tools/bench_prefill.py > $o/ncu_prefill.log 2>&1; echo "prefill full rc=$?" >> $o/rc.txt
timeout 1800 python -m pytest tests -m gpu -q > $o/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $o/rc.txt
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; echo "smoke rc=$?" >> $o/rc.txt
