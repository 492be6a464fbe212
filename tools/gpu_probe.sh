#!/bin/bash
# quick probe: GPU tests, cfg2 + cfg5 bench lines (no CPU baseline, in-situ shares), cfg4 decode probe
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/probe_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/probe_tests.log
for c in cfg2 cfg5; do timeout 600 python bench.py --config $c --no-cpu-baseline --steps 8 --warmup 3 > gpurun_out/probe_$c.json 2>gpurun_out/probe_$c.err; echo "$c rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/probe_$c.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$c',round(d['value']),round(d['e2e']['value']),d['clocks'],r['kernel'],r['frac'],r['insitu_sm_share'])"; done
timeout 200 python tools/decode_probe.py cfg4 3 2>&1 | tail -1
