mkdir -p gpurun_out
python -m pytest tests/test_gpu_loss.py -x -q 2>&1 | tail -3
python bench.py > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; tail -c 300 gpurun_out/bench_quick.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "e2e_with_loss", d.get("e2e_with_loss",{}).get("value"), "loss", d.get("loss_grad",{}).get("ms_per_view"), "clocks", d.get("clocks"))
PY
