mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_loss.py -x -q -p no:cacheprovider > gpurun_out/t_loss.log 2>&1; echo "rc=$?" >> gpurun_out/t_loss.log
timeout 120 python tools/time_loss.py bicycle > gpurun_out/loss_time.log 2>&1
timeout 300 python tools/time_raster_ab.py bicycle 0 VKS_RASTER_BWD_PPT 1 2 4 > gpurun_out/ab_bwd.log 2>&1
timeout 300 python tools/time_raster_ab.py bicycle 0 VKS_RASTER_FWD_PPT 1 2 4 > gpurun_out/ab_fwd.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ssim -c 2 -o gpurun_out/loss_full2 python tools/time_loss.py > gpurun_out/ncu_loss.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_loss.log
