#!/bin/bash
# Variant bench lines at HEAD: c2 in complex128, c2 on the CUDA-core FMA pass (SV_OPT_NO_TC),
# c2 and c4 as virtual shards (remap path), the weak-ladder n = 34 circuit with g = 3.
#   gpurun --timeout 1200 -- 'bash tools/profile_round2_variants.sh gpurun_out/r02u'
cd "${GRAFT_REPO_ROOT:-.}"
O=${1:-gpurun_out/r02u}
mkdir -p $O
B="python bench.py --warmup 3 --no-cpu-baseline --e2e-steps 0"
$B --steps 5 --dtype c128 > $O/bench_c2_c128.json 2> $O/bench_c2_c128.err
$B --steps 5 --flags 256 > $O/bench_c2_fma.json 2> $O/bench_c2_fma.err
$B --steps 5 --virtual-g 3 > $O/bench_c2_g3.json 2> $O/bench_c2_g3.err
$B --steps 3 --config c4 --virtual-g 2 > $O/bench_c4_g2.json 2> $O/bench_c4_g2.err
$B --steps 3 --config 34 --virtual-g 3 > $O/bench_ladder34_g3.json 2> $O/bench_ladder34_g3.err
for f in $O/bench_*.json; do echo $f; python - "$f" <<'P'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(round(d["ms_per_step"], 2), "ms", "frac", round(d["roofline"]["frac"], 3), d["config"].get("gate_kernel"), "remap", json.dumps(d.get("remap"))[:300])
except Exception as e:
    print("ERR", e)
P
done
