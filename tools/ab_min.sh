#!/bin/bash
# sec/circuit of c3 and c2 for several tensor-core step thresholds (STV_TC_MIN) and the sink flag
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
for cfg in c3 c2 c4; do for m in 200 120 80; do
  echo "== $cfg STV_TC_MIN=$m"; STV_TC_MIN=$m python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('ms', round(d['ms_per_step'],2), 'tc_steps', d.get('tc_steps'))
    elif 'rror' in l: print(l.strip())"
done; done
echo "== c3 no sink"; python bench.py --config c3 --flags 1024 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | cut -c1-200
