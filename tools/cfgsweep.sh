# c2 / c3 under the STV_GCFG launch configurations
for r in 1 2; do
for c in 0 4 6; do
  STV_GCFG=$c python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 > gpurun_out/cfg${c}_c2_$r.json
done
done
for c in 0 4 6; do
  STV_GCFG=$c python bench.py --config c4 --steps 2 --warmup 3 2>/dev/null | tail -1 > gpurun_out/cfg${c}_c4.json
done
