#!/bin/bash
# Round profiling bundle (GPU box): parity tests, smoke, the default bench
# line, the ncu launch list of one realistic 64-sentence bucket, and one
# ncu --set full capture of each tensor-core kernel class.  Outputs under
# gpurun_out/ (copy the summaries worth keeping into profiles/).
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches64.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_sk|logits_pair" \
  --launch-skip 200 --launch-count 6 -o gpurun_out/full python bench.py --steps 1 --warmup 0 --no-e2e \
  --no-cpu-baseline --bucket 64 > /dev/null 2>&1; echo "ncu full rc=$?"
