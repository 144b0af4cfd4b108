# final evidence of the round: bench line (defaults), other configs, GPU tests, smoke
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench_rc=$?" >> gpurun_out/bench_final.err
rm -f gpurun_out/other_final.jsonl
for c in mcmc garden stress; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/other_final.jsonl 2>>gpurun_out/other_final.err
done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_final.log 2>&1; echo "gputest_rc=$?" >> gpurun_out/gputest_final.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke_final.log
