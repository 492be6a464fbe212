mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_production_step.py -x -q -s > gpurun_out/prodstep.log 2>&1; echo "prodstep rc=$?"; grep -E "err|passed|failed" gpurun_out/prodstep.log | tail -6
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "not cfg2-64 and not cfg5-512" > gpurun_out/parity.log 2>&1; echo "parity rc=$?"; grep -E "token-identical|passed|failed|Error|assert" gpurun_out/parity.log | tail -15
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'] if d['e2e'] else None, d['ms_per_step'], d['roofline']['kernel_ms_per_step'])
P
