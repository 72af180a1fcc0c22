#!/bin/bash
# pure data movement of the tile pass (ops skipped) vs run length
for lb in 3 5 7 9 11; do
STV_TILE_DEBUG=1 python tools/prof_pass.py --gates 723 --reps 1 --tile-bits 12 --low-bits $lb --budget 50 2>&1 | tail -1
done
