mkdir -p gpurun_out
for v in "" "VKS_LIB_VARIANT=items8" "VKS_LIB_VARIANT=items12"; do
  echo "== $v" >> gpurun_out/items.log
  env $v timeout 300 python tools/time_binsort.py bicycle 30 >> gpurun_out/items.log 2>&1
  env $v timeout 300 python tools/time_binsort.py stress 10 >> gpurun_out/items.log 2>&1
done
