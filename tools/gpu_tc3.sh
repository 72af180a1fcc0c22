#!/bin/bash
# TC pass iteration: fast parity, A/B table, per-pass times.  gpurun -- 'bash tools/gpu_tc3.sh [ncu]'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_launch_configs.py tests/test_sampling.py -m gpu -x -q \
    -p no:cacheprovider > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fast.log
tail -4 gpurun_out/pytest_fast.log
grep -q "pytest rc=0" gpurun_out/pytest_fast.log || exit 1
python tools/pass_times.py c2 0 256 > gpurun_out/pass_times_c2.txt 2>&1; cat gpurun_out/pass_times_c2.txt
python tools/pass_times.py c4 0 256 > gpurun_out/pass_times_c4.txt 2>&1; tail -3 gpurun_out/pass_times_c4.txt
bash tools/ab_tc.sh $1
