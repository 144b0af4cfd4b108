mkdir -p gpurun_out
: > gpurun_out/ab.log
for v in default pbwd3 default pbwd3; do
  if [ $v = default ]; then unset VKS_LIB_VARIANT; else export VKS_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --steps 20 > gpurun_out/ab_$v.json 2>/dev/null
  python - $v >> gpurun_out/ab.log <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
print(v, "value", d["value"], "e2e", d["e2e"]["value"], "stages", d["stages_ms"], "clk", d["clocks"]["sm_mhz"])
PY
done
cat gpurun_out/ab.log
