#!/bin/bash
# fast GPU check: parity + launch configs + sampling (+ optional extra pytest args)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_launch_configs.py tests/test_sampling.py -m gpu -x -q \
    -p no:cacheprovider "$@" > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fast.log
grep -v "^\.\.\.\.\." gpurun_out/pytest_fast.log | tail -30
