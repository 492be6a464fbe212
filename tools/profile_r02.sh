#!/bin/bash
# Round-2 ncu bundle (GPU box): full sections for every decoder-step kernel
# class of one realistic 64-sentence bucket, the encode-ahead GEMMs, and the
# launch list of the bucket decode.  Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"logits_pair|gemm_sk|attn_sent|select_kernel" --launch-skip 200 --launch-count 14 \
  -o gpurun_out/r02_step python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > gpurun_out/ncu_step.log 2>&1; echo "ncu step rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:"EpiEncF|gather_split|enc_mean|gemm_simt" --launch-skip 0 --launch-count 16 \
  -o gpurun_out/r02_enc python tools/decode_probe.py cfg2 1 > gpurun_out/ncu_enc.log 2>&1; echo "ncu enc rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bucket64.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > /dev/null 2>&1; echo "ncu list rc=$?"
