mkdir -p gpurun_out
timeout 300 python tools/time_raster_ab.py bicycle 0 > gpurun_out/ab.log 2>&1
for a in "--split none" "--split bin-high" "--split raster-high" "--split same" "--split none --streams 4" "--split bin-high --streams 4" "--split raster-high --streams 4"; do
  echo "== $a" >> gpurun_out/split.log
  timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-batch1 $a 2>>gpurun_out/split.err | python -c "import json,sys; p=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(p['value'], p['ms_per_step'])" >> gpurun_out/split.log
done
