# A/B of EBR_DIAG variants on one box: phase stamps + bench lines (C2)
VARIANTS=${VARIANTS:-"16 0"}
for v in $VARIANTS; do EBR_DIAG=$v timeout 200 python tools/phase_times.py C2 > gpurun_out/phase_d$v.log 2>&1; done
for rep in 1 2; do for v in $VARIANTS; do EBR_DIAG=$v timeout 200 python bench.py --steps 1000 --no-cpu-baseline 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($v, round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],4), d['clocks'])" >> gpurun_out/ab.txt; done; done
