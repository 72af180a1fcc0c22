#!/bin/bash
# A/B of the tensor-core group pass on c2 (one gpurun call): ms/circuit under several settings, then
# an ncu capture of one k_tc_group_pass launch.   gpurun -- 'bash tools/ab_tc.sh [ncu]'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0"
run() { echo "== $1"; env $2 $B $3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('ms', round(d['ms_per_step'],2), 'tile_launch_ms', round(r['avg_launch_ms'],3))
    elif 'rror' in l: print(l.strip())"; }
{
run tc X=1
run fma X=1 "--flags 256"
run tc_copy_only STV_TILE_DEBUG=1
run tc_compute_only STV_TILE_DEBUG=2
run tc_min400 STV_TC_MIN=400
run tc_min100 STV_TC_MIN=100
run tc_ns1 STV_TC_NS=1
} > gpurun_out/ab_tc.log 2>&1
cat gpurun_out/ab_tc.log
if [ "$1" = ncu ]; then
  $B > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_tc_group_pass -s 20 -c 1 \
      -o gpurun_out/tc_prof -f $B > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu.log
fi
