#!/bin/bash
# Round evidence (bench lines as the driver runs them, reference arm, launch lists, ncu full
# captures, device build timing, C5 sweep, compute-sanitizer).
OUT=gpurun_out
mkdir -p $OUT
export EBR_SYNTH_CACHE=/tmp/ebr_synth
timeout 900 python bench.py > $OUT/ev_bench_c3.log 2>&1; tail -c 600 $OUT/ev_bench_c3.log; echo
timeout 600 python bench.py --config C2 > $OUT/ev_bench_c2.log 2>&1; tail -c 300 $OUT/ev_bench_c2.log; echo
timeout 600 python bench.py --config C4 --no-cpu-baseline > $OUT/ev_bench_c4.log 2>&1; tail -c 300 $OUT/ev_bench_c4.log; echo
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/ev_bench_ref_c3.log 2>&1; tail -c 300 $OUT/ev_bench_ref_c3.log; echo
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base -c 40 --csv --log-file $OUT/ev_c3_launches.csv python bench.py --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py $OUT/ev_c3_launches.csv > $OUT/ev_c3_launch_table.txt 2>&1; head -8 $OUT/ev_c3_launch_table.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base -c 30 --csv --log-file $OUT/ev_c2_launches.csv python bench.py --config C2 --profile --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 1 -c 1 -o $OUT/ev_c3_score1 python bench.py --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_kernel -s 5 -c 1 -o $OUT/ev_c2_small python bench.py --config C2 --profile --steps 6 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 python tools/build_time.py C2 C3 C4 C5 > $OUT/ev_build_time.jsonl 2>&1; cat $OUT/ev_build_time.jsonl
timeout 1500 python tools/sweep_c5.py > $OUT/ev_c5_sweep.jsonl 2>&1; tail -3 $OUT/ev_c5_sweep.jsonl
echo done
