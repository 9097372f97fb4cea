OUT=gpurun_out
for L in cur ab/w16k384.so; do
  if [ $L = cur ]; then E=""; else E=$PWD/$L; fi
  EBR_LIB=$E timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wide_smem -c 4 --csv --log-file $OUT/w2_$(basename $L).csv python bench.py --config C3 --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  EBR_LIB=$E timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/w2b4_$(basename $L).log 2>&1
done
EBR_LIB=$PWD/ab/w16k384.so timeout 900 python -m pytest tests/test_gpu_batch.py -x -q > $OUT/pytest_w2.log 2>&1; echo "rc=$?" >> $OUT/pytest_w2.log
echo done
