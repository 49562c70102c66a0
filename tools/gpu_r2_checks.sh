#!/bin/bash
# Device bounds-check run (the substitute for compute-sanitizer, which is
# closed on this pool): build libwsb_dbg.so (WSB_DCHECK: printf + trap on an
# out-of-range index in K1/K2/radix) and run the GPU parity suites against it
# with synchronous launches.
cd "$(dirname "$0")/.."
python -m paper_2504_00959_b200.build --debug > gpurun_out/r2_dbg_build.log 2>&1
WSB_LIB=$PWD/paper_2504_00959_b200/libwsb_dbg.so CUDA_LAUNCH_BLOCKING=1 timeout 1500 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py tests/test_gpu_scale.py \
  tests/test_gpu_reference_suite.py -m gpu -q -p no:cacheprovider --timeout 900 -rs \
  > gpurun_out/r2_dbg_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_dbg_pytest.log
