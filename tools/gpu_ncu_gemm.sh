OUT=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel" -s 4 -c 2 -o $OUT/gemm_full python bench.py --config C3 --profile --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_gemm.log 2>&1
echo done
