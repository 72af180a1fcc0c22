#!/bin/bash
# c3 sec/circuit under the FMA group-pass launch configurations (STV_GCFG 0..3)
cd "${GRAFT_REPO_ROOT:-.}"
for c in 0 1 2 3; do
  echo "== STV_GCFG=$c"; STV_GCFG=$c python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('ms', round(d['ms_per_step'],2))
    elif 'rror' in l: print(l.strip())"
done
