# GPU check: whole -m gpu suite, raster A/B timing, bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
timeout 300 python tools/time_raster_ab.py bicycle 0 > gpurun_out/ab.log 2>&1; echo "rc=$?" >> gpurun_out/ab.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/bench_rec.json 2> gpurun_out/bench_rec.err; echo "rc=$?" >> gpurun_out/bench_rec.err
