#!/bin/bash
# GPU-side quick check (run under gpurun): GPU tests + one bench line summary
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest: $(tail -1 gpurun_out/pytest_gpu.log)"
python bench.py --no-cpu-baseline "$@" > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_check.json"))
e = d["e2e"]
print("bench:", d["value"], d["unit"], d["ms_per_step"], "ms/step, frac", d["roofline"]["frac"],
      "e2e", e["value"], "kernels", d.get("kernels"))
PY
