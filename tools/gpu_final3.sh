OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench_c2.log 2>&1
timeout 600 python bench.py --config C3 --steps 20 --warmup 3 > $OUT/bench_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/c3_launches.csv python bench.py --config C3 --profile --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 1500 python tools/sweep_c5.py > $OUT/c5_sweep.jsonl 2> $OUT/c5_sweep.err
echo done
