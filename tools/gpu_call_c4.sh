cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02b
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
free -g >> $O/gpu.txt; nproc >> $O/gpu.txt
timeout 300 python bench.py --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
echo "bench rc=$?" >> $O/bench_c2.err
timeout 2900 python tools/c4_full_oracle.py $O/c4_full_oracle.json 7 > $O/c4_oracle.log 2>&1
echo "c4 rc=$?" >> $O/c4_oracle.log
tail -2 $O/c4_oracle.log; head -c 600 $O/bench_c2.json
