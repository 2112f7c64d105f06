# prefill poly share: 1 pair in 8 (base) vs 4/16 (poly4) vs 3/16 (poly5)
for v in base poly4 poly5 base poly4 poly5; do
  MV_LIB=tools/ab/$v/libmvb200.so timeout 300 python tools/bench_prefill.py > gpurun_out/ab11_${v}_$RANDOM.log 2>&1
done
MV_LIB=tools/ab/poly4/libmvb200.so timeout 600 python -m pytest tests/test_prefill_gpu.py -q -x > gpurun_out/ab11_test_poly4.log 2>&1
