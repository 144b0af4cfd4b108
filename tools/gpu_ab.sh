mkdir -p gpurun_out
VKS_LIB_VARIANT=lossf32 timeout 600 python -m pytest tests/test_gpu_loss.py -q -p no:cacheprovider > gpurun_out/t_lossf32.log 2>&1; echo "rc=$?" >> gpurun_out/t_lossf32.log
VKS_LIB_VARIANT=lossf32 timeout 120 python tools/time_loss.py bicycle > gpurun_out/loss_time.log 2>&1
timeout 120 python tools/time_loss.py bicycle >> gpurun_out/loss_time.log 2>&1
