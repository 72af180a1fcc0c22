#!/bin/bash
# tensor-core pass bring-up: probe, fast parity, bench.  gpurun -- 'bash tools/gpu_tc.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tc_probe tools/tc_probe.cu > gpurun_out/probe.log 2>&1 && \
  timeout 120 /tmp/tc_probe >> gpurun_out/probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/probe.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_launch_configs.py tests/test_sampling.py -m gpu -x -q \
    -p no:cacheprovider > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fast.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
cat gpurun_out/probe.log; tail -15 gpurun_out/pytest_fast.log; tail -3 gpurun_out/bench.log
