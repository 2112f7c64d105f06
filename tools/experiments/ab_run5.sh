for v in base poly0 poly8 poly2; do
  if [ $v = base ]; then L=""; else L="MV_LIB=tools/ab/$v/libmvb200.so"; fi
  env $L python bench.py --steps 100 --warmup 10 --extras none --cpu-seconds 0.5 > gpurun_out/ab5_c2_${v}.log 2>&1
  env $L python bench.py --workload c4 --steps 10 --warmup 3 --extras none --cpu-seconds 0.5 > gpurun_out/ab5_c4_${v}.log 2>&1
done
