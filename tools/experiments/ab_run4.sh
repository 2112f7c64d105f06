for v in base sb3 sb4 base sb4; do
  if [ $v = base ]; then L=""; else L="MV_LIB=tools/ab/$v/libmvb200.so"; fi
  env $L python bench.py --steps 100 --warmup 10 --extras none --cpu-seconds 0.5 > gpurun_out/ab4_c2_${v}_$RANDOM.log 2>&1
  env $L python bench.py --workload c4 --steps 10 --warmup 3 --extras none --cpu-seconds 0.5 > gpurun_out/ab4_c4_${v}_$RANDOM.log 2>&1
done
