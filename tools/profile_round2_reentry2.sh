#!/bin/bash
# Re-entry evidence, second call: the default bench line (e2e planned from scratch), one
# ncu --set full capture of a c2 tensor-core pass at HEAD, then the full GPU suite.
#   gpurun --timeout 2400 -- 'bash tools/profile_round2_reentry2.sh gpurun_out/r02x'
cd "${GRAFT_REPO_ROOT:-.}"
O=${1:-gpurun_out/r02x}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "planner_options_tc" -p no:cacheprovider > $O/pytest_tc_options.log 2>&1
echo "pytest rc=$?" >> $O/pytest_tc_options.log
python bench.py --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
bash tools/profile_round2_full.sh $O > $O/full.log 2>&1
STV_PARITY_LOG=$O/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest_tc_options.log; tail -3 $O/pytest.log; tail -2 $O/full.log; head -c 400 $O/bench_c2.json
