TAG=r01h bash tools/profile_round.sh
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01h_bench_reference.json 2>gpurun_out/r01h_ref.err
for c in c1 c3 c4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/r01h_bench_$c.json 2>gpurun_out/r01h_$c.err; done
