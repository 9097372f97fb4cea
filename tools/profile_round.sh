#!/bin/bash
# One GPU call: bench (with clocks + cpu baseline), ncu launch list, ncu --set full of the top kernel.
set -x
OUT=gpurun_out
python bench.py > $OUT/bench_full.log 2>&1; tail -1 $OUT/bench_full.log > $OUT/bench_line.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv python bench.py --profile --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:small_kernel -s 5 -c 1 -o $OUT/prof_full python bench.py --profile --steps 6 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
