mkdir -p gpurun_out
for v in "" "VKS_LIB_VARIANT=l4x512" "VKS_LIB_VARIANT=l2x256"; do
  echo "== $v" >> gpurun_out/loss_var.log
  env $v timeout 120 python tools/time_loss.py bicycle >> gpurun_out/loss_var.log 2>&1
  env $v timeout 120 python tools/time_loss.py bicycle >> gpurun_out/loss_var.log 2>&1
  env $v timeout 300 python -m pytest tests/test_gpu_loss.py -q -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/loss_var.log
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo "rc=$?" >> gpurun_out/torchrun1.err
