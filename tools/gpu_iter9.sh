OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q > $OUT/pytest_batch.log 2>&1; echo "rc=$?" >> $OUT/pytest_batch.log
for L in cur ab/pf2.so ab/pf8.so; do
  if [ $L = cur ]; then E=""; else E=$PWD/$L; fi
  EBR_LIB=$E timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_kernel -c 8 --csv --log-file $OUT/pf_$(basename $L).csv python bench.py --config C3 --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  EBR_LIB=$E timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/pfb_$(basename $L).log 2>&1
done
echo done
