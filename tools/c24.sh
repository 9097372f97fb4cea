export EBR_SYNTH_CACHE=/tmp/ebr_synth
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/pytest_nopair.log 2>&1; echo "default tests rc=$?"; tail -2 gpurun_out/pytest_nopair.log
EBR_PAIR=1 timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/pytest_pair.log 2>&1; echo "pair tests rc=$?"; tail -2 gpurun_out/pytest_pair.log
bash tools/gpu_diag.sh base "EBR_PAIR=1" "EBR_PAIR=1 EBR_DIAG=4"
