mkdir -p gpurun_out
for v in "" "VKS_LIB_VARIANT=cs4" "VKS_LIB_VARIANT=cs8" ""; do
  echo "== $v" >> gpurun_out/cs.log
  env $v timeout 300 python tools/time_binsort.py bicycle 30 >> gpurun_out/cs.log 2>&1
  env $v timeout 300 python tools/time_binsort.py stress 10 >> gpurun_out/cs.log 2>&1
done
VKS_LIB_VARIANT=cs4 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "binning or tiny or bicycle" > gpurun_out/t_cs4.log 2>&1; echo "rc=$?" >> gpurun_out/t_cs4.log
