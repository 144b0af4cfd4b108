mkdir -p gpurun_out
for c in stress bicycle mcmc; do
timeout 600 python tools/time_raster_ab.py $c 0 >> gpurun_out/ab_ca.log 2>&1
VKS_LIB_VARIANT=cg timeout 600 python tools/time_raster_ab.py $c 0 >> gpurun_out/ab_ca.log 2>&1
done
