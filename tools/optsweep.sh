# planner-option sweep on c2 (default launch configuration)
run() { python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline "$@" 2>/dev/null | tail -1; }
run > gpurun_out/os_default.json
run --tile-bits 13 > gpurun_out/os_tb13.json
STV_GCFG=3 run --tile-bits 13 > gpurun_out/os_tb13_cfg3.json
run --tile-bits 11 > gpurun_out/os_tb11.json
run --budget 2000 > gpurun_out/os_b2000.json
run --budget 450 > gpurun_out/os_b450.json
