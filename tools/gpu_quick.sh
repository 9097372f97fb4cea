#!/bin/bash
# Quick iteration: batched-path GPU tests, then C3 bench (+ optional launch list).
OUT=gpurun_out
export EBR_SYNTH_CACHE=/tmp/ebr_synth
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q --timeout 600 > $OUT/pytest_batch.log 2>&1; echo "batch tests rc=$?"; tail -4 $OUT/pytest_batch.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --profile > $OUT/bench_quick.log 2>&1
tail -1 $OUT/bench_quick.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('C3 ms', l['ms_per_step'], 'score<1> ms', l['roofline']['kernel_ms'])" || tail -5 $OUT/bench_quick.log
if [ "$1" == "launches" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base -c 40 --csv --log-file $OUT/launches_quick.csv python bench.py --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; python tools/launch_table.py $OUT/launches_quick.csv 2>&1 | tail -14
fi
