set -x
for v in narrowF2 narrowF4; do
  MV_LIB=tools/ab/$v/libmvb200.so timeout 600 python -m pytest tests/test_decode_gpu.py -q -x > gpurun_out/ab2_test_$v.log 2>&1
done
for v in base narrowF2 narrowF4 base; do
  if [ $v = base ]; then L=""; else L="MV_LIB=tools/ab/$v/libmvb200.so"; fi
  env $L python bench.py --steps 100 --warmup 10 --extras none --cpu-seconds 0.5 > gpurun_out/ab2_c2_$v.log 2>&1
done
