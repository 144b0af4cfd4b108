python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
run() { timeout 300 python bench.py --steps 20 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['e2e_with_loss']['value'], d['batch1']['value'], d['stages_ms'], d['clocks']['sm_mhz'])"; }
for v in default nopdl default nopdl; do
  if [ $v = default ]; then unset VKS_LIB_VARIANT; else export VKS_LIB_VARIANT=$v; fi
  echo "bench $v $(run)"
done
