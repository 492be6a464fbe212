#!/bin/bash
# Final round-2 measurement bundle on the current build (outputs under gpurun_out/d_*):
# GPU tests, smoke, bench lines for cfg2 (default, with the CPU baseline), cfg1/4/5,
# ensemble / shortlist side benches, the ncu launch list of one cfg2 bench step, one
# ncu --set full capture of every decoder-step kernel class (64-sentence bucket) and
# of the encode-ahead recurrence GEMMs.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader > gpurun_out/d_gpu.txt
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/d_gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/d_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err; echo "bench rc=$?"
for c in cfg1 cfg4 cfg5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/d_bench_$c.json 2> gpurun_out/d_bench_$c.err; echo "$c rc=$?"; done
timeout 300 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/d_bench_cfg1b.json 2> gpurun_out/d_bench_cfg1b.err; echo "cfg1b rc=$?"
timeout 600 python tools/ensemble_bench.py > gpurun_out/d_ensemble.txt 2>&1; echo "ens rc=$?"
SL_CFG=cfg1 timeout 300 python tools/shortlist_bench.py > gpurun_out/d_shortlist_cfg1.txt 2>&1; echo "sl1 rc=$?"
SL_CFG=cfg2 timeout 300 python tools/shortlist_bench.py > gpurun_out/d_shortlist_cfg2.txt 2>&1; echo "sl2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/d_ncu_launch.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"logits_pair|gemm_sk|attn_sent|select_kernel" --launch-skip 200 --launch-count 6 \
  -o gpurun_out/d_step python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --bucket 64 > gpurun_out/d_ncu_step.log 2>&1; echo "ncu step rc=$?"
timeout 600 ncu --set full --clock-control none \
  -k regex:"gemm_sk" --launch-skip 40 --launch-count 4 \
  -o gpurun_out/d_enc python tools/decode_probe.py cfg2 1 > gpurun_out/d_ncu_enc.log 2>&1; echo "ncu enc rc=$?"
