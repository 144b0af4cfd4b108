mkdir -p gpurun_out
for c in bicycle mcmc stress; do
VKS_TOOL_WORK_ORDER=1 timeout 600 python tools/time_raster_ab.py $c 0 2>&1 | grep -E "records|work" >> gpurun_out/worder.log
done
