# batched-path iteration: parity tests for the batched path, C3/C4 bench lines, C3 launch list
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q > $OUT/pytest_batch.log 2>&1; echo "rc=$?" >> $OUT/pytest_batch.log
timeout 400 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3.log 2>&1
timeout 400 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/c3_launches.csv python bench.py --config C3 --profile --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
