set -x
mkdir -p gpurun_out
python tools/time_loss.py bicycle > gpurun_out/loss_time.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:ssim -c 2 -o gpurun_out/loss_full python tools/time_loss.py bicycle > gpurun_out/loss_ncu.log 2>&1
