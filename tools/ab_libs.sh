# A/B of two library builds on one box (bench lines, C2): EBR_LIB=<alt .so> vs the in-tree build
ALT=${ALT:-/root/repo/ab_libs_head.so}
for rep in 1 2 3; do
  for v in alt cur; do
    if [ $v = alt ]; then L=$ALT; else L=""; fi
    EBR_LIB=$L timeout 200 python bench.py --steps 1000 --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/ab.txt
  done
done
