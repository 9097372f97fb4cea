for v in "0:256" "1:256" "3:256" "0:128" "1:128"; do
  IFS=: read d b <<< "$v"
  echo "== diag=$d batch=$b"; EBR_DIAG=$d timeout 300 python bench.py --config C3 --batch $b --steps 5 --warmup 3 --no-cpu-baseline --profile 2>&1 | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(l['ms_per_step'])"
done
echo "== hot 0"; EBR_HOT_BLOCKS=0 EBR_DIAG=1 timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline --profile 2>&1 | tail -c 300
