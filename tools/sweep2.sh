#!/bin/bash
# tile shape sweep on full c2: "tile low budget [flags]"
IFS=, read -ra LIST <<< "${CFGS:-12 4 1000,12 2 1000,13 4 1000,12 4 300}"
for cfg in "${LIST[@]}"; do
set -- $cfg
EXTRA=""; [ -n "$4" ] && EXTRA="--flags $4"
python tools/prof_pass.py --gates 723 --reps 2 --tile-bits $1 --low-bits $2 --budget $3 $EXTRA 2>&1 | tail -1 | python -c "
import sys,json
l=sys.stdin.read().strip()
try:
  d=json.loads(l); a=d['args']; print('$cfg', 'passes',d['tile_passes'],'avg_ms %.2f run_ms %.1f'%(d['tile_ms_avg'],d['run_ms']))
except Exception: print('$cfg', l[-300:])
"
done
