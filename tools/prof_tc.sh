#!/bin/bash
# one ncu --set full capture of a c2 tensor-core pass (after a plain run of the same command)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/tc
N="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$N > gpurun_out/tc/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tc_group_pass -s 33 -c 1 -o gpurun_out/tc/prof -f $N > gpurun_out/tc/ncu.log 2>&1
echo "ncu rc=$?"
