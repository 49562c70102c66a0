#!/bin/bash
# GPU-side evidence capture for profiles/ (run under gpurun from the repo root):
#   1. the 1-GPU bench line (bench.py, default steps)
#   2. the ncu launch list of the same command (short run), cold-cache durations
#   3. one `ncu --set full` capture of the main kernels of one cfg2 step
# Each ncu pass runs only after its command has exited 0 without ncu.
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_raw.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_(grid_items|fft_rows|fft_cols|keys|count|radix_scatter|radix_hist|item_offsets)" \
    -c 12 -o gpurun_out/full python tools/profile_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1
# cfg3 (north-star mesh): launch list of one step
python tools/run_cfg3.py --steps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cfg3_raw.csv python tools/run_cfg3.py --steps 1 > /dev/null 2>&1
echo done
