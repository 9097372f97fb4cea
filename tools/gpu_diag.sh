OUT=gpurun_out
for dg in 0 1 2; do
  EBR_DIAG=$dg timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_kernel -c 12 --csv --log-file $OUT/diag_$dg.csv python bench.py --config C3 --profile --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
EBR_HOT_KEYS=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_kernel -c 12 --csv --log-file $OUT/diag_nohot.csv python bench.py --config C3 --profile --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
EBR_HOT_KEYS=0 EBR_DIAG=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_kernel -c 12 --csv --log-file $OUT/diag_nohot2.csv python bench.py --config C3 --profile --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
