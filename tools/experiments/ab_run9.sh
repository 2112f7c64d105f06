# prefill parity-split softmax (ping-pong) vs base
timeout 600 python -m pytest tests/test_prefill_gpu.py -q -x > gpurun_out/ab9_test.log 2>&1
echo "tests exit $?" >> gpurun_out/ab9_test.log
for v in base new base new; do
  if [ $v = base ]; then L="MV_LIB=tools/ab/base/libmvb200.so"; else L=""; fi
  env $L timeout 300 python tools/bench_prefill.py > gpurun_out/ab9_pf_${v}_$RANDOM.log 2>&1
done
