#!/bin/bash
# c3 timing against the M-step cost threshold STV_TC_MIN (default 200)
cd "${GRAFT_REPO_ROOT:-.}"
for m in 200 100 60 30; do echo "== STV_TC_MIN=$m"; STV_TC_MIN=$m python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('ms', round(d['ms_per_step'],2), 'launch', round(d['roofline']['avg_launch_ms'],3), d['roofline'].get('kernel'))
    elif 'rror' in l: print(l.strip())"; done
STV_TC_MIN=60 python tools/pass_times.py c3 0 2>&1 | tail -12
