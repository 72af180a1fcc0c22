#!/bin/bash
# c3 timing against the per-pass diagonal-table budget STV_TAB_LIMIT (bytes; default 16384)
cd "${GRAFT_REPO_ROOT:-.}"
for t in 16384 20480 24576 32768; do echo "== STV_TAB_LIMIT=$t"; STV_TAB_LIMIT=$t python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('ms', round(d['ms_per_step'],2))
    elif 'rror' in l: print(l.strip())"; done
STV_TAB_LIMIT=24576 python tools/pass_times.py c3 0 2>&1 | tail -10
