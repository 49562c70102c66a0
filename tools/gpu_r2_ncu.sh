cd $GRAFT_REPO_ROOT
python tools/repro_grid.py 10000000 2048 32 > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_grid_items|k_keys|k_radix_scatter" -c 4 -o gpurun_out/prof_r2a python tools/repro_grid.py 10000000 2048 32 > gpurun_out/ncu_r2a.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2a.csv python tools/repro_grid.py 10000000 2048 32 > /dev/null 2>&1
