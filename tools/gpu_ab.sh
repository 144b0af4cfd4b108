mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
timeout 300 python tools/time_binsort.py bicycle 30 > gpurun_out/binsort.log 2>&1
timeout 300 python tools/time_binsort.py mcmc 30 >> gpurun_out/binsort.log 2>&1
timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_rec.json 2> gpurun_out/bench_rec.err; echo "rc=$?" >> gpurun_out/bench_rec.err
VKS_NCU_RANGE=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-batch1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu1_rc=$?" >> gpurun_out/ncu_launch.log
