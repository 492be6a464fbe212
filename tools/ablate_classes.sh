#!/bin/bash
# Marginal pass-time cost of each kernel class in the timed mode: the cfg2
# pass with one class's launches skipped (AMUN_ABLATE_CLASSES bitmask;
# outputs are garbage, only ms_per_step is read).  Profiling only.
mkdir -p gpurun_out
for m in 0 0x80 0x4 0x40 0x20 0x10 0x1 0x84; do
  AMUN_ABLATE_CLASSES=$m timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/abl_$m.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('gpurun_out/abl_$m.json').read().strip().splitlines()[-1]);print('$m', d['ms_per_step'], d['clocks']['sm_mhz'])"
done
AMUN_DEBUG_SELECT=1 timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "select phases"
