# bench the current library under each environment setting in $VARS (space-separated
# NAME=VALUE items, e.g. VARS="WSB_ROW_PF=0 WSB_ROW_PF=1"): step and kernel times
cd $GRAFT_REPO_ROOT
for V in $VARS; do
  env $V timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-cfg3 > gpurun_out/ev_$V.json 2> gpurun_out/ev_$V.err
  python - "$V" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ev_{v}.json").readline())
    print(v, d["ms_per_step"], {k: x["ms"] for k, x in d["kernels"].items()}, "e2e", d["e2e"]["ms_per_step"])
except Exception as e:
    print(v, "FAIL", e)
PY
done > gpurun_out/envvariants.txt 2>&1
