OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host or e2e" > $OUT/pytest_host.log 2>&1; echo "rc=$?" >> $OUT/pytest_host.log
timeout 600 python bench.py > $OUT/bench_c2.log 2>&1
timeout 600 python bench.py --config C3 --steps 20 --warmup 3 > $OUT/bench_c3.log 2>&1
timeout 400 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.log 2>&1
echo done
