# prefill poly share after the split-O change: 1 pair in 8 (base) vs none / 1 in 16 / 1 in 4
for v in base poly0 poly16 poly4 base poly0 poly16 poly4; do
  MV_LIB=tools/ab/$v/libmvb200.so timeout 300 python tools/bench_prefill.py > gpurun_out/ab14_${v}_$RANDOM.log 2>&1
done
