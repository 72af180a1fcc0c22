timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_group_pass --launch-skip 1 --launch-count 1 -o gpurun_out/c3p1 -f python tools/prof_cfg.py 3 > gpurun_out/c3p1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_group_pass --launch-skip 5 --launch-count 1 -o gpurun_out/c3p5 -f python tools/prof_cfg.py 3 > gpurun_out/c3p5.log 2>&1
