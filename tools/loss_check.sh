mkdir -p gpurun_out
python -m pytest tests/test_gpu_loss.py -x -q > gpurun_out/loss_tests.log 2>&1; tail -3 gpurun_out/loss_tests.log
for i in 1 2; do python tools/time_loss.py bicycle; done > gpurun_out/loss_time.log 2>&1; cat gpurun_out/loss_time.log
timeout 300 ncu --set full --clock-control none -k regex:"ssim|combine" -c 2 -o gpurun_out/loss_full2 python tools/time_loss.py bicycle > gpurun_out/loss_ncu.log 2>&1
