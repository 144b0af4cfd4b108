mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-batch1 > gpurun_out/b_sync.json 2> gpurun_out/b_sync.err
timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-batch1 --binning async > gpurun_out/b_async.json 2> gpurun_out/b_async.err
timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-batch1 --binning async --graph > gpurun_out/b_graph.json 2> gpurun_out/b_graph.err
