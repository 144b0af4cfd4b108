python -m pytest tests/test_gpu_parity.py -x -q -k "batch or bicycle or tiny or sh_degrees or overwrite" 2>&1 | tail -1
for v in default dy default dy; do
  if [ $v = default ]; then unset VKS_LIB_VARIANT; else export VKS_LIB_VARIANT=$v; fi
  echo "$v $(timeout 600 python tools/time_batch.py bicycle 8)"
done
unset VKS_LIB_VARIANT
run() { timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-batch1 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms']['project_bwd'], d['clocks']['sm_mhz'])"; }
for v in default dy default dy; do
  if [ $v = default ]; then unset VKS_LIB_VARIANT; else export VKS_LIB_VARIANT=$v; fi
  echo "bench $v $(run)"
done
