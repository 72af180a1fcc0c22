#!/bin/bash
# Round-2 evidence run (one gpurun call): full GPU test suite with parity numbers, bench lines for
# every single-GPU config, the c2 k-sweep, per-pass times, an ncu launch list of the bench command
# (one ncu per call: the --set full capture of the tensor-core pass is tools/profile_round2_full.sh).
#   gpurun --timeout 3600 -- 'bash tools/profile_round2.sh gpurun_out/r02'
cd "${GRAFT_REPO_ROOT:-.}"
O=${1:-gpurun_out/r02}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
nproc > $O/host.txt; free -g >> $O/host.txt; lscpu | grep "Model name" >> $O/host.txt
STV_PARITY_LOG=$O/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
B="python bench.py --steps 10 --warmup 3"
$B > $O/bench_c2.json 2> $O/bench_c2.err
$B --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
$B --config c1 --no-cpu-baseline --steps 50 > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_c4.json 2> $O/bench_c4.err
$B --dtype c128 --no-cpu-baseline > $O/bench_c2_c128.json 2> $O/bench_c2_c128.err
$B --flags 256 --no-cpu-baseline > $O/bench_c2_fma.json 2> $O/bench_c2_fma.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
python tools/ksweep.py $O/ksweep.md > $O/ksweep.jsonl 2>&1
python tools/pass_times.py c2 0 256 > $O/pass_times_c2.txt 2>&1
python tools/pass_times.py c3 0 > $O/pass_times_c3.txt 2>&1
N="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$N > $O/ncu_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
      --log-file $O/launches.csv $N > $O/ncu_launches.log 2>&1
echo "ncu launches rc=$?" >> $O/ncu_launches.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
tail -3 $O/pytest.log; for f in $O/bench_*.json; do echo $f; head -c 300 $f; echo; done
