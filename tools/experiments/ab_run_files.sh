o=gpurun_out/ab1; mkdir -p $o
for r in 1 2; do for v in base s3 dbl3; do
  MV_LIB=tools/ab/$v/libmvb200.so python bench.py --gpus 1 --steps 20 --warmup 5 --extras c4 --cpu-seconds 0 > $o/${v}_$r.json 2> $o/${v}_$r.err
done; done
