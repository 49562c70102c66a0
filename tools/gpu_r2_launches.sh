cd $GRAFT_REPO_ROOT
python tools/run_cfg3.py --steps 1 > gpurun_out/l3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python tools/run_cfg3.py --steps 1 > /dev/null 2>&1
python tools/repro_grid.py 10000000 2048 32 > gpurun_out/l2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/repro_grid.py 10000000 2048 32 > /dev/null 2>&1
