cd $GRAFT_REPO_ROOT
for a in "10000000 2048 32" "6500000 512 8"; do
  CUDA_LAUNCH_BLOCKING=1 WSB_LIB=$GRAFT_REPO_ROOT/paper_2504_00959_b200/libwsb_dbg.so timeout 300 python tools/repro_grid.py $a >> gpurun_out/dbg.log 2>&1
done
