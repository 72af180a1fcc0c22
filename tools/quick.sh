# quick GPU check: c2 + c3 bench lines, gpu tests (not fullsize)
python bench.py --steps 5 --warmup 3 > gpurun_out/q_c2.json 2>gpurun_out/q_c2.err
python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/q_c3.json 2>&1
python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/q_tests.txt 2>&1; tail -2 gpurun_out/q_tests.txt
