# A/B: HEAD copy in _ab/ vs working tree on c2 (+ working tree with STV_GCFG=5)
run() { python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1; }
for r in 1 2; do
  (cd _ab && run > ../gpurun_out/ab_A_c2_$r.json)
  run > gpurun_out/ab_B_c2_$r.json
done
STV_GCFG=5 run > gpurun_out/ab_B5_c2.json
