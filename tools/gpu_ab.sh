for v in default nb3; do
  if [ $v = default ]; then unset VKS_LIB_VARIANT; else export VKS_LIB_VARIANT=$v; fi
  for c in bicycle stress; do echo "$v $(timeout 600 python tools/time_raster_ab.py $c 0 2>&1 | grep records)"; done
done
unset VKS_LIB_VARIANT
run() { timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-batch1 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms']['raster_fwd'], d['stages_ms']['raster_bwd'], d['clocks']['sm_mhz'])"; }
for v in default nb3 default nb3; do
  if [ $v = default ]; then unset VKS_LIB_VARIANT; else export VKS_LIB_VARIANT=$v; fi
  echo "bench $v $(run)"
done
