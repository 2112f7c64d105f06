# decode issuers converged vs base
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_toy_gpu.py -q -x > gpurun_out/ab10_test.log 2>&1
echo "tests exit $?" >> gpurun_out/ab10_test.log
for v in base new base new; do
  if [ $v = base ]; then L="MV_LIB=tools/ab/base/libmvb200.so"; else L=""; fi
  env $L python bench.py --steps 100 --warmup 10 --extras none --cpu-seconds 0.5 > gpurun_out/ab10_c2_${v}_$RANDOM.log 2>&1
  env $L python bench.py --workload c4 --steps 10 --warmup 3 --extras none --cpu-seconds 0.5 > gpurun_out/ab10_c4_${v}_$RANDOM.log 2>&1
done
