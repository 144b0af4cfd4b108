mkdir -p gpurun_out
timeout 600 python tools/time_raster_ab.py bicycle 0 > gpurun_out/ab_addr.log 2>&1
timeout 600 python tools/time_raster_ab.py bicycle 0 >> gpurun_out/ab_addr.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "tiny or records or sparse" > gpurun_out/t_addr.log 2>&1; echo "rc=$?" >> gpurun_out/t_addr.log
