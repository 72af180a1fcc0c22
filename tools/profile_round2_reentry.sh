#!/bin/bash
# Re-entry evidence at HEAD (one gpurun call, no A/B): full GPU test
# suite with parity numbers, bench lines c1-c4 and the reference arm, an ncu launch list of the
# default bench command, smoke.   gpurun --timeout 3000 -- 'bash tools/profile_round2_reentry.sh gpurun_out/r02y'
cd "${GRAFT_REPO_ROOT:-.}"
O=${1:-gpurun_out/r02y}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
B="python bench.py --steps 10 --warmup 3"
$B > $O/bench_c2.json 2> $O/bench_c2.err
$B --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
$B --config c1 --no-cpu-baseline --steps 50 > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
N="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$N > $O/ncu_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
      --log-file $O/launches.csv $N > $O/ncu_launches.log 2>&1
echo "ncu launches rc=$?" >> $O/ncu_launches.log
STV_PARITY_LOG=$O/parity.jsonl timeout 1800 python -m pytest tests -m gpu -q -s -p no:cacheprovider > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
for f in $O/bench_*.json; do echo $f; head -c 300 $f; echo; done
