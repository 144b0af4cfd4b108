mkdir -p gpurun_out
timeout 600 python tools/time_binsort_async.py bicycle
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/binasync_launches.csv python tools/time_binsort_async.py bicycle 1 > /dev/null 2>&1
