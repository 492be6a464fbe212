#!/bin/bash
# ncu bundle for the projected-context build: full sections (with source) for
# every decoder-step kernel class of one realistic 64-sentence bucket
# (launches 200+ of one bucket decode), and the launch list of one cfg2 bench step.
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"logits_pair|gemm_sk|attn_sent|select_kernel" --launch-skip 200 --launch-count 7 \
  -o gpurun_out/r02b_step python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > gpurun_out/ncu_step.log 2>&1; echo "ncu step rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
