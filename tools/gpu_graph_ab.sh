OUT=gpurun_out
for rep in 1 2; do
timeout 300 python bench.py --no-cpu-baseline > $OUT/g_graph_$rep.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-graph > $OUT/g_direct_$rep.log 2>&1
done
echo done
