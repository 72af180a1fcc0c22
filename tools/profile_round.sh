#!/bin/bash
# One GPU call: plain bench, ncu launch list of the same bench command, and one
# ncu --set full capture of the dominant kernel (c2 pass 5).  Outputs under gpurun_out/.
set -x
TAG=${TAG:-r01}
timeout 400 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_group_pass --launch-skip 5 \
    --launch-count 1 -o gpurun_out/${TAG}_group_pass python tools/prof_pass.py --gates 723 --reps 1 \
    > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
