python -m pytest tests/test_gpu_parity.py -x -q -k "batch or bicycle or overwrite" 2>&1 | tail -1
for i in 1 2; do timeout 600 python tools/time_batch.py bicycle 8; done
run() { timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-batch1 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms']['project_bwd'], d['clocks']['sm_mhz'])"; }
echo "bench $(run)"; echo "bench $(run)"
