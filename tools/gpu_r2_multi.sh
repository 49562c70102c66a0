#!/bin/bash
# Round-2 multi-GPU evidence (gpurun --gpus 4): the whole GPU test suite on a
# 4-GPU box (the real-NCCL equality test runs with 4 ranks), cfg2 weak scaling
# (bench.py at N=2,4; deterministic v-slabs and the w-plane mode) and cfg3
# (100M LOFAR-like, 4096^2 x 64) at 1/2/4 GPUs with the linearity check.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r2m_topo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rs \
  > gpurun_out/r2m_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2m_pytest_gpu.log
out=gpurun_out/r2m_multigpu.txt
run() {  # n, port, script args...
  n=$1; port=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" --master-addr 127.0.0.1 \
    --master-port "$port" "$@" 2>> gpurun_out/r2m_multigpu.err | tail -1
}
{
  for d in slabs planes; do
    echo "# bench.py --gpus N --decomp $d (cfg2 weak scaling, 10M records per GPU):"
    run 2 29611 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --decomp $d
    run 4 29612 bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline --decomp $d
  done
  echo "# tools/run_cfg3.py (cfg3: 100M LOFAR-like tracks, 4096^2 x 64, strong scaling) 1/2/4 GPUs:"
  timeout 600 python tools/run_cfg3.py --check 2>> gpurun_out/r2m_multigpu.err | tail -1
  for d in slabs planes; do
    run 2 29613 tools/run_cfg3.py --decomp $d --check
    run 4 29614 tools/run_cfg3.py --decomp $d --check
  done
} > $out
