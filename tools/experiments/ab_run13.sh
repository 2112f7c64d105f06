# decode tail split: 2 waves (base) vs 3 waves vs 2 + 1 passes; C2 (driver command) and C4
for v in base tail3 tail2p base tail3 tail2p; do
  MV_LIB=tools/ab/$v/libmvb200.so python bench.py --steps 20 --warmup 5 --extras none --cpu-seconds 0.5 > gpurun_out/ab13_c2_${v}_$RANDOM.log 2>&1
  MV_LIB=tools/ab/$v/libmvb200.so python bench.py --workload c4 --steps 10 --warmup 3 --extras none --cpu-seconds 0.5 > gpurun_out/ab13_c4_${v}_$RANDOM.log 2>&1
done
MV_LIB=tools/ab/tail2p/libmvb200.so timeout 900 python -m pytest tests/test_decode_gpu.py -q -x > gpurun_out/ab13_test.log 2>&1
