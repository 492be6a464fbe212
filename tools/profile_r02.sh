#!/bin/bash
# Round-2 ncu bundle (GPU box): full sections (with source) for every
# decoder-step kernel class of a realistic 64-sentence bucket (launches 200+
# of one bucket decode), the encode-ahead recurrence GEMMs, and the launch list.
# Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"logits_pair|gemm_sk|attn_sent|select_kernel" --launch-skip 200 --launch-count 8 \
  -o gpurun_out/r02_step python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > gpurun_out/ncu_step.log 2>&1; echo "ncu step rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:"gemm_sk|enc_mean|gather_split" --launch-skip 40 --launch-count 6 \
  -o gpurun_out/r02_enc python tools/decode_probe.py cfg2 1 > gpurun_out/ncu_enc.log 2>&1; echo "ncu enc rc=$?"
