#!/bin/bash
# c3 (n=32) FMA group passes under ncu --set full: a QFT pass (launch 1) and the first tail pass (launch 5)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/c3
N="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$N > gpurun_out/c3/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_group_pass -s 28 -c 1 -o gpurun_out/c3/qft -f $N > gpurun_out/c3/ncu1.log 2>&1
$N > gpurun_out/c3/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_group_pass -s 32 -c 1 -o gpurun_out/c3/tail -f $N > gpurun_out/c3/ncu2.log 2>&1
tail -2 gpurun_out/c3/ncu1.log gpurun_out/c3/ncu2.log
