#!/bin/bash
# Round-2 measurement bundle: default bench line (cfg2), cfg1/4/5 lines, ensemble and shortlist
# benches, model-load probe, the ncu launch list of one 64-sentence bucket and one ncu --set full
# capture of every decoder-step kernel class.  Outputs under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
for c in cfg1 cfg4 cfg5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/final_bench_$c.json 2>/dev/null; echo "$c rc=$?"; done
timeout 600 python tools/ensemble_bench.py > gpurun_out/final_ensemble.txt 2>&1; echo "ens rc=$?"
SL_CFG=cfg1 timeout 300 python tools/shortlist_bench.py > gpurun_out/final_shortlist_cfg1.txt 2>&1
SL_CFG=cfg2 timeout 300 python tools/shortlist_bench.py > gpurun_out/final_shortlist_cfg2.txt 2>&1
timeout 300 python tools/load_probe.py > gpurun_out/final_load.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches64.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"logits_pair|gemm_sk|attn_sent|select_kernel" --launch-skip 200 --launch-count 8 \
  -o gpurun_out/final_step python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > /dev/null 2>&1; echo "ncu full rc=$?"
