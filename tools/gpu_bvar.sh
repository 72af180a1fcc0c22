#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_launch_configs.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for cfg in c2 c4; do echo "== $cfg"; python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('ms', round(d['ms_per_step'],2), 'tc_steps', d.get('tc_steps'), 'launch', round(d['roofline']['avg_launch_ms'],3))
    elif 'rror' in l: print(l.strip())"; done
python tools/pass_times.py c2 0 256 2>&1 | tail -15
