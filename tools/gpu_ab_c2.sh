# C2 A/B of latency-path builds on one box, 3 interleaved repetitions (ms per step, roofline frac)
OUT=gpurun_out
: > $OUT/ab_c2.txt
for rep in 1 2 3; do
  for L in cur ab/s8.so ab/s4.so; do
    if [ $L = cur ]; then E=""; else E=$PWD/$L; fi
    EBR_LIB=$E timeout 200 python bench.py --steps 1000 --no-cpu-baseline 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],4))" >> $OUT/ab_c2.txt
  done
done
EBR_LIB=$PWD/ab/s8.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/pytest_s8.log 2>&1; echo "rc=$?" >> $OUT/pytest_s8.log
echo done
