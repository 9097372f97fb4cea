# A/B of library builds / EBR_DIAG settings on one box (bench lines, C2).  Each ALTS entry is
# "<.so path or cur>:<EBR_DIAG>"; "cur" is the in-tree build.
ALTS=${ALTS:-"/root/repo/ab_libs_head.so:0 cur:0"}
for rep in 1 2 3; do
  for v in $ALTS; do
    lib=${v%%:*}; dg=${v##*:}
    if [ $lib = cur ]; then L=""; else L=$lib; fi
    EBR_LIB=$L EBR_DIAG=$dg timeout 200 python bench.py --steps 1000 --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib):$dg', round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/ab.txt
  done
done
