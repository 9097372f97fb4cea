export EBR_SYNTH_CACHE=/tmp/ebr_synth
timeout 300 python -m pytest tests/test_gpu_batch.py -x -q -k "exact_bit_exact" > gpurun_out/pytest_pair.log 2>&1; echo "pair tests rc=$?"; tail -3 gpurun_out/pytest_pair.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile > gpurun_out/bench_pair.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_pair.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('ms', l['ms_per_step'], 'kernel_ms', l['roofline']['kernel_ms'])" || tail -3 gpurun_out/bench_pair.log
