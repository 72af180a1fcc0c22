# A/B: HEAD copy in _ab/ vs working tree, interleaved, c2 and c3
for r in 1 2; do
  (cd _ab && python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 > ../gpurun_out/ab_A_c2_$r.json)
  python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 > gpurun_out/ab_B_c2_$r.json
  (cd _ab && python bench.py --config c3 --steps 3 --warmup 3 2>/dev/null | tail -1 > ../gpurun_out/ab_A_c3_$r.json)
  python bench.py --config c3 --steps 3 --warmup 3 2>/dev/null | tail -1 > gpurun_out/ab_B_c3_$r.json
done
