mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
timeout 300 python tools/time_raster_ab.py bicycle 0 > gpurun_out/ab.log 2>&1
timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_rec.json 2> gpurun_out/bench_rec.err; echo "rc=$?" >> gpurun_out/bench_rec.err
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:^(raster)" -o gpurun_out/raster_f32x2 python tools/profile_bench_step.py > gpurun_out/ncu_full.log 2>&1; echo "ncu_rc=$?" >> gpurun_out/ncu_full.log
