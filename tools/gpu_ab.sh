mkdir -p gpurun_out
for a in "--streams 4" "--streams 5" "--streams 6" "--streams 8" "--streams 4"; do
  echo "== $a" >> gpurun_out/streams.log
  timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-batch1 $a 2>>gpurun_out/streams.err | python -c "import json,sys; p=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(p['value'], p['ms_per_step'])" >> gpurun_out/streams.log
done
