mkdir -p gpurun_out
VKS_LIB_VARIANT=nb3 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "records or tiny or bicycle or culling" > gpurun_out/t_nb3.log 2>&1; echo "rc=$?" >> gpurun_out/t_nb3.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "records or tiny or culling" > gpurun_out/t_nb2.log 2>&1; echo "rc=$?" >> gpurun_out/t_nb2.log
for c in stress bicycle mcmc; do
timeout 600 python tools/time_raster_ab.py $c 0 >> gpurun_out/ab_nb.log 2>&1
VKS_LIB_VARIANT=nb3 timeout 600 python tools/time_raster_ab.py $c 0 >> gpurun_out/ab_nb.log 2>&1
done
