#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_launch_configs.py tests/test_sampling.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for v in "STV_NO_TMA=0" "STV_NO_TMA=1" "STV_TMA_STORE=1"; do for cfg in c2 c4; do echo "== $cfg $v"; env $v python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('ms', round(d['ms_per_step'],2), 'launch', round(d['roofline']['avg_launch_ms'],3))
    elif 'rror' in l: print(l.strip())"; done; done
STV_TILE_DEBUG=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('copy only ms', d['ms_per_step'], d['roofline']['avg_launch_ms'])"
STV_TILE_DEBUG=1 STV_NO_TMA=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('copy only (cp.async) ms', d['ms_per_step'], d['roofline']['avg_launch_ms'])"
