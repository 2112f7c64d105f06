o=gpurun_out/r02g2; mkdir -p $o
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"decode_tc|k_append_one|rope_q_tile|combine" -c 120 --csv --log-file $o/decode_launches.csv \
    python bench.py --steps 20 --warmup 5 --extras none --cpu-seconds 0 > $o/ncu_launches.log 2>&1; echo "launches rc=$?" >> $o/rc.txt
python tools/sass_summary.py > $o/sass_summary.txt 2>&1; echo "sass rc=$?" >> $o/rc.txt
