#!/bin/bash
# Decomposition of score_kernel<1> on C3 by EBR_DIAG bits, with an alternative library (EBR_LIB):
#   1 no cold scatter, 2 no epilogue filter, 32 no TMEM read, 64 no TMEM store, 1024 no MMA issue,
#   2048 no hot one-hot writes.   bash tools/gpu_decomp.sh tools/bin/lib_diag.so 0 3 35 ...
OUT=gpurun_out
mkdir -p $OUT
export EBR_SYNTH_CACHE=/tmp/ebr_synth
lib=$1; shift
[ "$lib" != base ] && export EBR_LIB=/root/repo/$lib
for d in "$@"; do
  EBR_DIAG=$d timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile > $OUT/decomp_$d.log 2>&1
  echo "diag $d $(tail -1 $OUT/decomp_$d.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('ms', round(l['ms_per_step'],3), 'score1_ms', round(l['roofline']['kernel_ms'],3))" 2>/dev/null || tail -2 $OUT/decomp_$d.log)"
done
