mkdir -p gpurun_out
for c in bicycle stress; do
for v in "" "VKS_LIB_VARIANT=b9" "VKS_LIB_VARIANT=b8"; do
  echo "== $c $v" >> gpurun_out/ab_b.log
  env $v timeout 600 python tools/time_raster_ab.py $c 0 2>&1 | grep records >> gpurun_out/ab_b.log
done; done
