#!/bin/bash
# Full round evidence: every gpu test, smoke, bench lines, launch lists, one ncu --set full.
OUT=gpurun_out
mkdir -p $OUT
export EBR_SYNTH_CACHE=/tmp/ebr_synth
t0=$(date +%s)
timeout 3000 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider > $OUT/pytest_gpu_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_full.log
echo "tests done in $(( $(date +%s) - t0 )) s"; tail -15 $OUT/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
