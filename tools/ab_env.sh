#!/bin/bash
# A/B timings: bash tools/ab_env.sh "<cfg> [ENV=..] [--bench-arg ..]" ...
# each spec: a config, environment assignments, then bench.py arguments
cd "${GRAFT_REPO_ROOT:-.}"
for spec in "$@"; do
  set -- $spec
  cfg=$1; shift
  envs=(); args=()
  for a in "$@"; do if [[ $a == *=* && $a != --* ]]; then envs+=("$a"); else args+=("$a"); fi; done
  echo "== $cfg ${envs[*]} ${args[*]}"
  env "${envs[@]}" python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 "${args[@]}" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],3), 'launch', round(r['avg_launch_ms'],3), 'tc_steps', d.get('tc_steps'), 'passes', d.get('passes'))
    elif 'rror' in l or 'Traceback' in l: print(l.strip())"
done
