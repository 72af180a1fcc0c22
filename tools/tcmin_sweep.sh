#!/bin/bash
# c2 / c4 timing against the M-step cost threshold STV_TC_MIN (FFMA2-equivalents per vector; default 200)
cd "${GRAFT_REPO_ROOT:-.}"
for cfg in c2 c4; do for m in 200 150 120 100 60; do echo "== $cfg STV_TC_MIN=$m"; STV_TC_MIN=$m python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('ms', round(d['ms_per_step'],2))
    elif 'rror' in l: print(l.strip())"; done; done
