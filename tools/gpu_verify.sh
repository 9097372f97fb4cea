set -x
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 400 python bench.py > $OUT/bench_c2.log 2>&1
timeout 400 python bench.py --config C3 --steps 20 --warmup 3 > $OUT/bench_c3.log 2>&1
timeout 400 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.log 2>&1
echo done
