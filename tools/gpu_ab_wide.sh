# A/B of wide-kernel range sizes (ab/*.so built with EBR_NVCC_DEFS) on one box
OUT=gpurun_out
for L in cur ab/r16k.so ab/r32k.so; do
  if [ $L = cur ]; then E=""; else E=$PWD/$L; fi
  EBR_LIB=$E timeout 600 python -m pytest tests/test_gpu_batch.py -x -q -k "exact or hot" > $OUT/ab_pytest_$(basename $L).log 2>&1; echo "rc=$?" >> $OUT/ab_pytest_$(basename $L).log
  for c in C3 C4; do
    EBR_LIB=$E timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ab_${c}_$(basename $L).log 2>&1
  done
done
timeout 300 python tools/phase_times.py C2 > $OUT/phase_c2.txt 2>&1
echo done
