for d in 0 1 2; do
STV_TILE_DEBUG=$d ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3n_d$d.csv python tools/prof_cfg.py 3 > /dev/null 2>&1
done
