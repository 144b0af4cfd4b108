python -m pytest tests/test_gpu_parity.py tests/test_gpu_bin_async.py -x -q -k "records or sparse or tiny or mcmc or bicycle or graph or ragged or culling" 2>&1 | tail -1
for c in bicycle mcmc stress; do timeout 600 python tools/time_raster_ab.py $c 0 VKS_RASTER_PERSIST 0 1 0 1 2>&1 | grep records; done
run() { timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-batch1 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms']['raster_bwd'], d['clocks']['sm_mhz'])"; }
for v in 0 1 0 1; do echo "bench persist=$v $(VKS_RASTER_PERSIST=$v run)"; done
