#!/bin/bash
# planner/kernel parameter sweep on the full c2 circuit (one line per config)
BUDGETS=${BUDGETS:-"60 80 100 130 170 220"}
TILES=${TILES:-"12 13"}
EXTRA=${EXTRA:-""}
for tb in $TILES; do for bu in $BUDGETS; do
python tools/prof_pass.py --gates 723 --reps 2 --tile-bits $tb --budget $bu $EXTRA 2>&1 | tail -1
done; done | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except: print(l.strip()[:300]); continue
  a=d['args']; print(a['tile_bits'],a['budget'],'passes',d['tile_passes'],'ops',d['ops'],'avg_ms %.2f GBps %.0f run_ms %.1f'%(d['tile_ms_avg'],d['GBps'] or 0,d['run_ms']))
"
