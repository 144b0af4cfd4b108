mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_loss.py -q -p no:cacheprovider > gpurun_out/t_loss3.log 2>&1; echo "rc=$?" >> gpurun_out/t_loss3.log
timeout 120 python tools/time_loss.py bicycle > gpurun_out/loss3.log 2>&1
timeout 120 python tools/time_loss.py bicycle >> gpurun_out/loss3.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:ssim -c 2 -o gpurun_out/loss3 python tools/time_loss.py > gpurun_out/ncu_loss3.log 2>&1
