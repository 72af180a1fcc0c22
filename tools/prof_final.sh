# final round profiles: bench (c2) + launch list + ncu full of pass 5, reference arm, other configs
TAG=${TAG:-r01j} bash tools/profile_round.sh
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG:-r01j}_bench_reference.json 2>/dev/null
for c in c1 c3 c4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/${TAG:-r01j}_bench_$c.json 2>/dev/null; done
bash tools/c2dbg.sh
