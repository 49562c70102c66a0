cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_scale.py -q -p no:cacheprovider -k bucketing > gpurun_out/dbg_bucket.log 2>&1
for a in "6500000 512 8" "7000000 512 8" "7500000 512 8"; do
  timeout 120 python tools/repro_grid.py $a >> gpurun_out/dbg.log 2>&1
done
