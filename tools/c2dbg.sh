# c2 per-pass times under STV_TILE_DEBUG 0/1/2 (normal / data movement only / compute only)
for d in 0 1 2; do
STV_TILE_DEBUG=$d ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2n_d$d.csv python tools/prof_cfg.py 2 > /dev/null 2>&1
done
