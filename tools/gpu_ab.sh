mkdir -p gpurun_out
for a in "" "--halves" "" "--halves" "--halves --streams 3" "--halves --split none"; do
  echo "== $a" >> gpurun_out/halves.log
  timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-batch1 $a 2>>gpurun_out/halves.err | python -c "import json,sys; p=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(p['value'], p['ms_per_step'], p['train_step']['value'])" >> gpurun_out/halves.log
done
