#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/final_gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/final_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
for c in cfg1 cfg4 cfg5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/final_bench_$c.json 2>/dev/null; echo "$c rc=$?"; done
