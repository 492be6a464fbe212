#!/bin/bash
# Side benches on the current build: ensembles, shortlists (steady state), model load,
# scaling emulation, the ncu launch list of one 64-sentence bucket and a full ncu
# capture of every decoder-step class (outputs under gpurun_out/).
mkdir -p gpurun_out
timeout 600 python tools/ensemble_bench.py > gpurun_out/side_ensemble.txt 2>&1; echo "ens rc=$?"
timeout 600 python tools/shortlist_steady.py > gpurun_out/side_shortlist.txt 2>&1; echo "sl rc=$?"
timeout 300 python tools/load_probe.py > gpurun_out/side_load.txt 2>&1; echo "load rc=$?"
timeout 600 python tools/shard_probe.py > gpurun_out/side_shard.txt 2>&1; echo "shard rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/side_launches64.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"logits_pair|gemm_sk|attn_sent|select_kernel" --launch-skip 200 --launch-count 6 \
  -o gpurun_out/side_step python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > /dev/null 2>&1; echo "ncu full rc=$?"
