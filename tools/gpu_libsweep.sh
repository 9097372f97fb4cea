#!/bin/bash
# Per-kernel times (ncu launch list) of the C3 step for alternative builds of libebr.so:
#   bash tools/gpu_libsweep.sh tools/bin/libA.so tools/bin/libB.so ...   ("base" = the in-tree build)
OUT=gpurun_out
mkdir -p $OUT
export EBR_SYNTH_CACHE=/tmp/ebr_synth
for lib in "$@"; do
  tag=$(basename $lib .so)
  if [ "$lib" == "base" ]; then unset EBR_LIB; else export EBR_LIB=/root/repo/$lib; fi
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --print-units base -c 30 --csv --log-file $OUT/sweep_$tag.csv python bench.py --profile --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "== $tag"; python tools/launch_table.py $OUT/sweep_$tag.csv 2>&1 | grep -E "entry_|score_kernel<1" | head -3
done
