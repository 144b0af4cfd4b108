mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_bin_async.py -x -q -k "bin or sort or async or P2 or bicycle or tiny or mcmc or ragged or stress" 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/time_binsort.py bicycle; done
timeout 300 python tools/time_binsort.py stress
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:keys_count --csv python tools/time_binsort.py bicycle 1 2>/dev/null | grep -E "keys_count" | head -4 | cut -c1-60,200-
run() { timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-batch1 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms']['bin_sort'], d['clocks']['sm_mhz'])"; }
echo "bench $(run)"; echo "bench $(run)"
