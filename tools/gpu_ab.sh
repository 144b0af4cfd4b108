mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_bin_async.py -x -q -k "bin or sort or async or P2 or bicycle or tiny" 2>&1 | tail -1
run() { timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-batch1 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms']['bin_sort'], d['clocks']['sm_mhz'])"; }
echo "bench $(run)"; echo "bench $(run)"
