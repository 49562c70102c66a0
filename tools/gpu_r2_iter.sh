# one iteration: GPU tests (subset or all), bench, cfg3 on one GPU, ncu of chosen kernels
cd $GRAFT_REPO_ROOT
TESTS=${TESTS:-tests}
timeout 1200 python -m pytest $TESTS -m gpu -q -p no:cacheprovider --timeout 600 -x -rf > gpurun_out/it_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/it_pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err
echo "bench rc=$?" >> gpurun_out/it_bench.err
if [ -n "$CFG3" ]; then timeout 300 python tools/run_cfg3.py --steps 5 > gpurun_out/it_cfg3.json 2> gpurun_out/it_cfg3.err; fi
if [ -n "$NCU" ]; then
python tools/repro_grid.py ${NCU_ARGS:-10000000 2048 32} > gpurun_out/it_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$NCU" -c ${NCU_C:-3} -o gpurun_out/it_prof python tools/repro_grid.py ${NCU_ARGS:-10000000 2048 32} > gpurun_out/it_ncu.log 2>&1
fi
