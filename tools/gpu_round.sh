# round-end evidence: GPU tests, smoke, bench line, launch list of two timed steps, full ncu capture
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "gputest_rc=$?" >> gpurun_out/gputest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?" >> gpurun_out/bench.err
VKS_NCU_RANGE=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-batch1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu1_rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:^(digit|keys|project|raster|rect|scan|scatter|tile)" -o gpurun_out/bench_step_full python tools/profile_bench_step.py > gpurun_out/ncu_full.log 2>&1; echo "ncu2_rc=$?" >> gpurun_out/ncu_full.log
