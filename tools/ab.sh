# A/B: HEAD copy in _ab/ vs working tree, interleaved, c2 and c3; then the GPU tests
run() { python bench.py --e2e-steps 0 --no-cpu-baseline "$@" 2>/dev/null | tail -1; }
for r in 1 2; do
  (cd _ab && run --steps 5 --warmup 3 > ../gpurun_out/ab_A_c2_$r.json)
  run --steps 5 --warmup 3 > gpurun_out/ab_B_c2_$r.json
done
(cd _ab && run --config c3 --steps 3 --warmup 3 > ../gpurun_out/ab_A_c3.json)
run --config c3 --steps 3 --warmup 3 > gpurun_out/ab_B_c3.json
python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/ab_tests.txt 2>&1; tail -2 gpurun_out/ab_tests.txt
