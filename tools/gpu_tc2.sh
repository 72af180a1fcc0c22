#!/bin/bash
# TC pass iteration: fast parity, then the A/B table (+ ncu if asked).  gpurun -- 'bash tools/gpu_tc2.sh [ncu]'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_launch_configs.py tests/test_sampling.py -m gpu -x -q \
    -p no:cacheprovider > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fast.log
tail -4 gpurun_out/pytest_fast.log
grep -q "pytest rc=0" gpurun_out/pytest_fast.log && bash tools/ab_tc.sh $1
