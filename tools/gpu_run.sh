#!/bin/bash
# One gpurun call: GPU test suite (parity numbers to gpurun_out/parity.jsonl), a short
# bench, and one compute-sanitizer tool on small circuits.  Usage (from the repo root):
#   gpurun --timeout 2400 -- 'bash tools/gpu_run.sh [racecheck|memcheck|none]'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
STV_PARITY_LOG=gpurun_out/parity.jsonl timeout 1500 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider \
    > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tool=${1:-racecheck}
if [ "$tool" != none ]; then
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_small.py \
      > gpurun_out/sanitizer_$tool.log 2>&1; echo "sanitizer rc=$?" >> gpurun_out/sanitizer_$tool.log
  tail -5 gpurun_out/sanitizer_$tool.log
fi
grep -E "passed|failed|rc=" gpurun_out/pytest.log | tail -3; tail -2 gpurun_out/bench.log
