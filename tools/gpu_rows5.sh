for R in 320 768 512; do for kk in 5 12 1; do ./build/bench_logits_tc $R swap $kk | head -1; done; done
timeout 1200 python -m pytest tests -m gpu -q -s -x > gpurun_out/gputests_r5.log 2>&1; echo "tests rc=$?"; grep -E "token-identical|passed|failed|Error|assert" gpurun_out/gputests_r5.log | cut -c1-200 | tail -25
python tools/decode_probe.py cfg2 3 | tail -1
python tools/decode_probe.py cfg4 2 | tail -1
python tools/decode_probe.py cfg5 2 | tail -1
python tools/decode_probe.py cfg1 2 | tail -1
