OUT=gpurun_out
for L in cur ab/r24k.so ab/r16k.so; do
  if [ $L = cur ]; then E=""; else E=$PWD/$L; fi
  EBR_LIB=$E timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wide_smem -c 6 --csv --log-file $OUT/w_$(basename $L).csv python bench.py --config C3 --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
echo done
