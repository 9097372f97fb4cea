#!/bin/bash
# One parameterised GPU session: gpurun --timeout T -- 'bash tools/gpu_round.sh <what...>'
#   tests        pytest -m gpu (full suite)
#   bench:CFG    bench.py --config CFG (no cpu baseline)
#   launches:CFG ncu launch list (gpu__time_duration + dram bytes) of a short bench run
#   full:CFG:K   ncu --set full of kernel regex K in a short bench run
OUT=gpurun_out
export EBR_SYNTH_CACHE=/tmp/ebr_synth
mkdir -p $OUT
for w in "$@"; do
  IFS=: read -r what cfg kern <<< "$w"
  case $what in
    tests) timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log; tail -5 $OUT/pytest_gpu.log ;;
    testfile) timeout 1500 python -m pytest $cfg -q --timeout 600 > $OUT/pytest_file.log 2>&1; echo "rc=$?" >> $OUT/pytest_file.log; tail -15 $OUT/pytest_file.log ;;
    bench) timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline $kern > $OUT/bench_$cfg.log 2>&1; tail -c 3000 $OUT/bench_$cfg.log ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base -c 60 --csv --log-file $OUT/launches_$cfg.csv python bench.py --config $cfg --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; python tools/launch_table.py $OUT/launches_$cfg.csv 2>&1 | tail -40 ;;
    full) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$kern -s ${SKIP:-1} -c 1 -o $OUT/full_${cfg}_${kern} python bench.py --config $cfg --profile --steps 2 --warmup 3 --no-cpu-baseline > $OUT/full_${cfg}.log 2>&1; tail -3 $OUT/full_${cfg}.log ;;
  esac
done
