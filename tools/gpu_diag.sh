#!/bin/bash
# Role / variant diagnosis of the batched path on C3 (EBR_DIAG bits of ebr_batch.cu):
#   4 = per-role cycle accounting, 1 = skip the cold scatter, 2 = skip the epilogue work;
#   EBR_HOT_BLOCKS = hot K blocks used (0..2).  Prints ms/step per variant.
OUT=gpurun_out
export EBR_SYNTH_CACHE=/tmp/ebr_synth
mkdir -p $OUT
CFG=${CFG:-C3}
for v in "${@:-base}"; do
  case $v in
    base) env=() ;;
    prof) env=(EBR_DIAG=4) ;;
    nocold) env=(EBR_DIAG=1) ;;
    noepi) env=(EBR_DIAG=2) ;;
    hot0) env=(EBR_HOT_BLOCKS=0) ;;
    hot1) env=(EBR_HOT_BLOCKS=1) ;;
    *) env=($v) ;;
  esac
  echo "== $v"
  tag=$(echo "$v" | tr '/= ' '___')
  env "${env[@]}" timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --profile > $OUT/diag_$tag.log 2>&1
  grep "ebr prof" $OUT/diag_$tag.log | tail -1
  tail -1 $OUT/diag_$tag.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('ms', l['ms_per_step'], 'kernel_ms', l['roofline']['kernel_ms'])" 2>/dev/null || tail -3 $OUT/diag_$v.log
done
