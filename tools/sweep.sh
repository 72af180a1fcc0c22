#!/bin/bash
# planner/kernel parameter sweep on the full c2 circuit (one line per config)
for tb in 12 13; do for lb in 5 7 9; do for bu in 50 80 120 200; do
python tools/prof_pass.py --gates 723 --reps 2 --tile-bits $tb --low-bits $lb --budget $bu 2>&1 | tail -1
done; done; done
