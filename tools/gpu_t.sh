OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q -k "sharded" > $OUT/pytest_shard.log 2>&1; echo "rc=$?" >> $OUT/pytest_shard.log
echo done
