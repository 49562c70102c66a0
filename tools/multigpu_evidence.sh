#!/bin/bash
# Multi-GPU evidence (run under `gpurun --gpus 4` from the repo root):
# bench.py at N=2 and N=4 (cfg2 weak scaling) and the cfg3 north-star
# runner at 1, 2 and 4 GPUs (strong scaling). Output: gpurun_out/multigpu.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/multigpu.txt
run() {  # n, port, script args...
  n=$1; port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" --master-addr 127.0.0.1 \
    --master-port "$port" "$@" 2>> gpurun_out/multigpu.err | tail -1
}
{
  for d in planes slabs; do
    echo "# bench.py --gpus N --decomp $d (cfg2 weak scaling, 10M records per GPU), full JSON lines:"
    run 2 29611 bench.py --gpus 2 --no-cpu-baseline --decomp $d
    run 4 29612 bench.py --gpus 4 --no-cpu-baseline --decomp $d
  done
  echo "# tools/run_cfg3.py (cfg3 north star: 100M LOFAR-like tracks, 4096^2 x 64, strong scaling), 1/2/4 GPUs:"
  python tools/run_cfg3.py 2>> gpurun_out/multigpu.err | tail -1
  for d in planes slabs; do
    run 2 29613 tools/run_cfg3.py --decomp $d --check
    run 4 29614 tools/run_cfg3.py --decomp $d --check
  done
} > $out
cat $out | cut -c1-400
