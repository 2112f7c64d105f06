# prefill epilogue via TMA store: parity (bf16 + fp32 outputs) and timing vs base
timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_toy_gpu.py tests/test_refswap_gpu.py -q -x > gpurun_out/ab12_test.log 2>&1
echo "tests exit $?" >> gpurun_out/ab12_test.log
for v in base new base new; do
  if [ $v = base ]; then L="MV_LIB=tools/ab/base/libmvb200.so"; else L=""; fi
  env $L timeout 300 python tools/bench_prefill.py > gpurun_out/ab12_pf_${v}_$RANDOM.log 2>&1
done
