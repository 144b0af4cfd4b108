python -m pytest tests/test_gpu_parity.py tests/test_gpu_bin_async.py -x -q -k "bin or sort or async or P2 or bicycle or tiny or mcmc or stress" 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/time_binsort.py bicycle; done
timeout 300 python tools/time_binsort.py stress
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"row_scan" --csv python tools/time_binsort.py bicycle 1 2>/dev/null | grep -E "row_scan" | awk -F'","' '{print $NF}' | head -8 | tr '\n' ' '; echo
run() { timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms']['bin_sort'], d['batch1']['value'], d['clocks']['sm_mhz'])"; }
echo "bench $(run)"; echo "bench $(run)"
