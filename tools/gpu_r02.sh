#!/bin/bash
# Round-2 GPU bundle: all -m gpu tests (-s to surface counts), smoke, default bench line,
# cfg4/cfg5/cfg1 bench lines, launch list of one 64-bucket pass.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; grep -E "token-identical|passed|failed|Error" gpurun_out/gputests.log | tail -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
for c in cfg4 cfg5 cfg1; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2>/dev/null; echo "$c rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c',d['value'],d.get('e2e',{}).get('value'))"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches64.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > /dev/null 2>&1; echo "ncu list rc=$?"
