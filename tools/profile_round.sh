#!/bin/bash
# One GPU call for the round's evidence: gpu tests, smoke, bench lines (C2 default with cpu
# baseline, C3, C4, the reference arm), ncu launch lists (C2, C3) and ncu --set full of the C2 kernel.
OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench_c2.log 2>&1
timeout 600 python bench.py --config C3 --steps 20 --warmup 3 > $OUT/bench_c3.log 2>&1
timeout 400 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/c2_launches.csv python bench.py --profile --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/c3_launches.csv python bench.py --config C3 --profile --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:small_kernel -s 5 -c 1 -o $OUT/c2_full python bench.py --profile --steps 6 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
