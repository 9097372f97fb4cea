OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q > $OUT/pytest_batch.log 2>&1; echo "rc=$?" >> $OUT/pytest_batch.log
for c in C3 C4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.log 2>&1; done
timeout 300 python bench.py --config C3 --k 10000 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_k10000.log 2>&1
echo done
