OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q > $OUT/pytest_batch.log 2>&1; echo "rc=$?" >> $OUT/pytest_batch.log
for c in C3 C4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/c3_launches.csv python bench.py --config C3 --profile --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 1500 python tools/sweep_c5.py > $OUT/c5_sweep.jsonl 2> $OUT/c5_sweep.err
echo done
