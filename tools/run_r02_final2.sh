o=gpurun_out/${1:-r02j}; mkdir -p $o
python bench.py --gpus 1 --steps 20 --warmup 5 > $o/bench_s20w5.json 2> $o/bench_s20w5.err; echo "bench rc=$?" >> $o/rc.txt
bash tools/run_all_benches.sh $o/summary > $o/summary.log 2>&1; echo "summary rc=$?" >> $o/rc.txt
timeout 1500 python -m pytest tests -m gpu -q > $o/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $o/rc.txt
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; echo "smoke rc=$?" >> $o/rc.txt
python tools/sass_summary.py > $o/sass_summary.txt 2>&1
