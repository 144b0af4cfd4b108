mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "records" > gpurun_out/t_rec.log 2>&1; echo "rc=$?" >> gpurun_out/t_rec.log
