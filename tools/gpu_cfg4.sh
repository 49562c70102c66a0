#!/bin/bash
# cfg4 (SKA-scale: 1B LOFAR-like records, 16384^2 x 32) on 4 GPUs of one box
# (gpurun --gpus 4): the v-slab decomposition with the distributed (slab
# transpose) FFT and the w-plane ranges, each with the linearity check.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/cfg4.txt
run() {  # port, args...
  port=$1; shift
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port "$port" tools/run_cfg3.py --records 1000000000 --mesh 16384 --planes 32 --cell 1e-5 \
    --steps 2 --check --label "cfg4 SKA-scale" "$@" 2>> gpurun_out/cfg4.err | tail -1
}
{
  echo "# cfg4: 1B LOFAR-like records, 16384^2 x 32, 4 GPUs, v-slabs (distributed FFT):"
  run 29621 --decomp slabs
  echo "# cfg4, 4 GPUs, w-plane ranges:"
  run 29622 --decomp planes
} > $out
