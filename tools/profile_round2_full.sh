#!/bin/bash
# One ncu --set full capture of a c2 tensor-core pass (after a plain run of the same command), with
# the raw and SASS-source pages exported for tools/ncu_srcmap.py.
#   gpurun --timeout 1200 -- 'bash tools/profile_round2_full.sh gpurun_out/r02'
cd "${GRAFT_REPO_ROOT:-.}"
O=${1:-gpurun_out/r02}
mkdir -p $O
N="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$N > $O/ncu_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_tc_group_pass -s 20 -c 1 \
      -o $O/tc_full -f $N > $O/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $O/ncu_full.log
ncu -i $O/tc_full.ncu-rep --page raw --csv > $O/tc_full_raw.csv 2>/dev/null
ncu -i $O/tc_full.ncu-rep --page source --csv --print-source sass > $O/tc_full_sass.csv 2>/dev/null
tail -2 $O/ncu_full.log
