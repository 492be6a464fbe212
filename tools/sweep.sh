#!/bin/bash
# bench sweep over env settings: tools/sweep.sh "ENV1=a ENV2=b" "ENV1=c" ...
mkdir -p gpurun_out
for cfg in "$@"; do
  line=$(env $cfg timeout 300 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | tail -1)
  python - "$cfg" "$line" <<'PY'
import json, sys
cfg, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    print(f"{cfg:40s} {d['value']:10.0f} wps  {d['ms_per_step']:8.1f} ms  eager/class {d['roofline']['kernel_ms_per_step']}")
except Exception as e:
    print(cfg, "FAILED", line[-300:])
PY
done
