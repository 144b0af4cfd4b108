run() { timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-batch1 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms']['raster_bwd'], d['clocks']['sm_mhz'])"; }
for i in 1 2; do
for v in 4 6 8 2; do echo "sparse $v $(VKS_RASTER_SPARSE=$v run)"; done
done
