export EBR_SYNTH_CACHE=/tmp/ebr_synth
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/pytest_b.log 2>&1; echo "default tests rc=$?"; tail -2 gpurun_out/pytest_b.log
EBR_PAIR=1 timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/pytest_bp.log 2>&1; echo "pair tests rc=$?"; tail -2 gpurun_out/pytest_bp.log
bash tools/gpu_diag.sh base "EBR_DIAG=4" "EBR_PAIR=1" "EBR_PAIR=1 EBR_DIAG=4" "EBR_DEEP_TMEM=1"
