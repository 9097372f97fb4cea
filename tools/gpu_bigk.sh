OUT=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/c3_k10000_launches.csv python bench.py --config C3 --k 10000 --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/c4_launches.csv python bench.py --config C4 --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
