mkdir -p gpurun_out
timeout 300 python tools/time_raster_ab.py bicycle 0 VKS_RASTER_SPARSE 2 4 6 8 12 > gpurun_out/ab_sparse.log 2>&1
timeout 300 python tools/time_raster_ab.py mcmc 0 VKS_RASTER_SPARSE 4 8 >> gpurun_out/ab_sparse.log 2>&1
