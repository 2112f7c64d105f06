o=gpurun_out/r02i; mkdir -p $o
python bench.py --gpus 1 --steps 20 --warmup 5 > $o/bench_s20w5.json 2> $o/bench_s20w5.err; echo "bench rc=$?" >> $o/rc.txt
bash tools/run_all_benches.sh $o/summary > $o/summary.log 2>&1; echo "summary rc=$?" >> $o/rc.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"decode_tc|k_append_one|rope_q_tile|combine" -c 120 --csv --log-file $o/decode_launches.csv \
    python bench.py --steps 20 --warmup 5 --extras none --cpu-seconds 0 > $o/ncu_launches.log 2>&1; echo "launches rc=$?" >> $o/rc.txt
ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 15 -c 1 -o $o/decode_tc_full \
    python bench.py --steps 20 --warmup 5 --extras none --cpu-seconds 0 > $o/ncu_decode.log 2>&1; echo "decode full rc=$?" >> $o/rc.txt
timeout 1500 python -m pytest tests -m gpu -q > $o/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $o/rc.txt
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; echo "smoke rc=$?" >> $o/rc.txt
python tools/sass_summary.py > $o/sass_summary.txt 2>&1
