# poly clamp + prefill sum guard vs HEAD: decode C2/C4 and prefill C3
for v in base new base new; do
  if [ $v = base ]; then L="MV_LIB=tools/ab/base/libmvb200.so"; else L=""; fi
  env $L python bench.py --steps 100 --warmup 10 --extras none --cpu-seconds 0.5 > gpurun_out/ab8_c2_${v}_$RANDOM.log 2>&1
  env $L python bench.py --workload c4 --steps 10 --warmup 3 --extras none --cpu-seconds 0.5 > gpurun_out/ab8_c4_${v}_$RANDOM.log 2>&1
  env $L timeout 300 python tools/bench_prefill.py > gpurun_out/ab8_pf_${v}_$RANDOM.log 2>&1
done
