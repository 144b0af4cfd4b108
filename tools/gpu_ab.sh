mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_bin_async.py tests/test_gpu_debug_checks.py -x -q -k "bin or sort or async or P2 or bicycle or tiny or debug or stress or ragged" 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"keys_" --csv python tools/time_binsort.py bicycle 1 2>/dev/null | grep -E "keys_" | head -4 | awk -F'","' '{print $5, $NF}' | cut -c1-40,100-
run() { timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-batch1 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms']['bin_sort'], d['clocks']['sm_mhz'])"; }
echo "bench $(run)"; echo "bench $(run)"
