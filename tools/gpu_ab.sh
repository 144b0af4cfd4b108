mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/bench_ca.json 2> gpurun_out/bench_ca.err
for c in mcmc garden stress; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/other_configs.jsonl 2>>gpurun_out/other_configs.err
done
