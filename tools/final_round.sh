#!/bin/bash
# Final evidence of the round: gpu tests, smoke, bench lines, C3 launch list + ncu of gemm_kernel<1>.
OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench_c2.log 2>&1
timeout 600 python bench.py --config C3 --steps 20 --warmup 3 > $OUT/bench_c3.log 2>&1
timeout 400 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $OUT/c3_launches.csv python bench.py --config C3 --profile --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|wide_smem" -s 6 -c 3 -o $OUT/c3_final python bench.py --config C3 --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
