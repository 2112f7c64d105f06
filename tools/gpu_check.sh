#!/bin/bash
# One GPU pass over the current tree: the GPU test suite, smoke(), the default bench line and the C3 prefill
# bench.  Usage: tools/gpu_check.sh <out subdir of gpurun_out/>
o=gpurun_out/${1:-check}; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q -x > $o/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $o/rc.txt
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; echo "smoke rc=$?" >> $o/rc.txt
python bench.py --gpus 1 --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err; echo "bench rc=$?" >> $o/rc.txt
python tools/bench_prefill.py > $o/prefill.json 2>&1; echo "prefill rc=$?" >> $o/rc.txt
