#!/bin/bash
# Final build's bench lines (cfg2 default with the CPU baseline, cfg1/4/5), GPU tests,
# smoke, the ncu launch list of one 64-sentence bucket and an ncu --set full capture of
# the select kernel (outputs under gpurun_out/e_*).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/e_gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/e_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err; echo "bench rc=$?"
for c in cfg1 cfg4 cfg5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/e_bench_$c.json 2> gpurun_out/e_bench_$c.err; echo "$c rc=$?"; done
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/e_launches64.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"select_kernel|attn_sent" --launch-skip 30 --launch-count 2 \
  -o gpurun_out/e_sel python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > /dev/null 2>&1; echo "ncu sel rc=$?"
