OUT=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|wide_smem" -s 6 -c 3 -o $OUT/c3_final2 python bench.py --config C3 --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
