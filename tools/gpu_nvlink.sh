#!/bin/bash
# NVLink evidence (gpurun --gpus 2 or 4): the push probe, then ncu with the
# NVLink byte counters on the same single-process run (k_push kernels)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/nvlink_push_probe.py > gpurun_out/nvlink_probe.json 2> gpurun_out/nvlink_probe.err
ncu --query-metrics 2>/dev/null | grep -i "nvl" > gpurun_out/nvlink_metrics.txt
M=nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum
echo "metrics: $M" > gpurun_out/nvlink_ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum,$M --clock-control none -k regex:k_push -c 6 --csv \
  python tools/nvlink_push_probe.py --reps 1 >> gpurun_out/nvlink_ncu.log 2>&1
