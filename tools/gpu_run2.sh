mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_production_step.py -x -q -s > gpurun_out/prodstep.log 2>&1; echo "prodstep rc=$?"; tail -12 gpurun_out/prodstep.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "not cfg2-64 and not cfg5-512" > gpurun_out/parity.log 2>&1; echo "parity rc=$?"; grep -E "token-identical|passed|failed|Error" gpurun_out/parity.log | tail -15
timeout 600 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench rc=$?"
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench_cfg4.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'] if d['e2e'] else None, d['ms_per_step'], d['roofline']['kernel_ms_per_step'])
P
