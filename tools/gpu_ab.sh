python -m pytest tests/test_gpu_parity.py -x -q -k "bin or bicycle or tiny" 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rect_diff" --csv python tools/time_binsort.py bicycle 1 2>/dev/null | grep -E "rect_diff" | head -3 | awk -F'","' '{print $5, $NF}' | cut -c1-30,80-
