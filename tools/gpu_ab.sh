mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "project_bwd_batch or grad_overwrite or tiny" > gpurun_out/t_pb.log 2>&1; echo "rc=$?" >> gpurun_out/t_pb.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-batch1 > gpurun_out/bench_pb.json 2> gpurun_out/bench_pb.err
timeout 600 ncu --profile-from-start off --set full --clock-control none -k "regex:project_bwd_batch" -o gpurun_out/pb2 python tools/profile_bench_step.py > gpurun_out/ncu_pb.log 2>&1
