OUT=gpurun_out
timeout 1500 python tools/sweep_c5.py > $OUT/c5_sweep.jsonl 2> $OUT/c5_sweep.err
echo done
