mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_bin_async.py -x -q -k "bin or sort or async or P2" 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/time_binsort.py bicycle; done
timeout 300 python tools/time_binsort.py stress
