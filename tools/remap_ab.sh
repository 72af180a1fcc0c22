#!/bin/bash
# remap pipelining on virtual shards: parity, then remap ms / GB/s with STV_REMAP_PIPE=1 vs 0
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_sampling.py -m gpu -q -x -k "virtual" -p no:cacheprovider 2>&1 | tail -1
for cfg in "c2 1" "c2 2" "c2 3" "c4 2"; do set -- $cfg; for p in 1 0; do
  echo "== $1 virtual_g=$2 pipe=$p"; STV_REMAP_PIPE=$p python bench.py --config $1 --virtual-g $2 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('ms', round(d['ms_per_step'],2), 'remap', d.get('remap'), 'passes', d.get('passes'))
    elif 'rror' in l: print(l.strip())"
done; done
