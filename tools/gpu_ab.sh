mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"project_" -o gpurun_out/proj_src python tools/profile_batch.py bicycle 8 > gpurun_out/proj_ncu.log 2>&1
tail -1 gpurun_out/proj_ncu.log
