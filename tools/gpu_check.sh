#!/bin/bash
# parity (fast GPU suites) + c2/c4 timings of the default path and of SV_OPT_TMA
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_launch_configs.py tests/test_sampling.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for fl in 0 2048; do for cfg in c2 c4; do echo "== $cfg flags=$fl"; python bench.py --config $cfg --flags $fl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('ms', round(d['ms_per_step'],2), 'launch', round(d['roofline']['avg_launch_ms'],3))
    elif 'rror' in l: print(l.strip())"; done; done
