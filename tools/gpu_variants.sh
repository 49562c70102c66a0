# bench each variant library build/var*/libwsb.so (WSB_LIB) on one GPU: step and kernel
# times, plus an ncu launch list per variant (per-kernel durations)
cd $GRAFT_REPO_ROOT
for L in build/var*/libwsb.so; do
  v=$(basename $(dirname $L))
  WSB_LIB=$PWD/$L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-cfg3 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/var_{v}.json").readline())
    print(v, d["ms_per_step"], {k: x["ms"] for k, x in d["kernels"].items()})
except Exception as e:
    print(v, "FAIL", e)
PY
  if [ -n "$CFG3" ]; then
    WSB_LIB=$PWD/$L timeout 300 python tools/run_cfg3.py --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('  cfg3', d['ms_per_step'], d['kernel_ms'])"
  fi
  if [ -n "$LAUNCHES" ]; then
    WSB_LIB=$PWD/$L ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/var_$v.csv python tools/repro_grid.py 10000000 2048 32 > /dev/null 2>&1
    python tools/launch_summary.py gpurun_out/var_$v.csv | head -12
  fi
done > gpurun_out/variants.txt 2>&1
