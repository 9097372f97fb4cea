bash tools/gpu_diag.sh "EBR_DIAG=103 EBR_HOT_BLOCKS=0" "EBR_DIAG=231 EBR_HOT_BLOCKS=0"
export EBR_SYNTH_CACHE=/tmp/ebr_synth
EBR_DIAG=99 EBR_HOT_BLOCKS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 1 -c 1 -o gpurun_out/full_hot0 python bench.py --profile --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_hot0.log 2>&1; tail -2 gpurun_out/ncu_hot0.log
