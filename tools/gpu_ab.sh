python -m pytest tests/test_gpu_parity.py tests/test_gpu_bin_async.py -x -q -k "bin or sort or async or P2 or bicycle or tiny or mcmc" 2>&1 | tail -1
for v in default notrig default notrig; do
  if [ $v = default ]; then unset VKS_LIB_VARIANT; else export VKS_LIB_VARIANT=$v; fi
  echo "$v $(timeout 300 python tools/time_binsort.py bicycle)"
done
unset VKS_LIB_VARIANT
run() { timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms']['bin_sort'], d['batch1']['value'], d['clocks']['sm_mhz'])"; }
for v in default notrig default notrig; do
  if [ $v = default ]; then unset VKS_LIB_VARIANT; else export VKS_LIB_VARIANT=$v; fi
  echo "bench $v $(run)"
done
