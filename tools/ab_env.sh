#!/bin/bash
# Same-box sweep of environment knobs (profiling only): for each "NAME=VALUE"
# (or "default") in $ENVS, one cfg2 device line ($CFG), two rounds.
mkdir -p gpurun_out
for r in 1 2; do for e in ${ENVS:-default}; do
  if [ "$e" = default ]; then envs=""; else envs="$e"; fi
  env $envs timeout 300 python bench.py --config ${CFG:-cfg2} --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abe.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/abe.json').read().strip().splitlines()[-1]);print('$e', $r, round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
