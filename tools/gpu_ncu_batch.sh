OUT=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"wide_smem|gemm_kernel" -s 6 -c 3 -o $OUT/c3_full python bench.py --config C3 --profile --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_c3.log 2>&1
echo done
