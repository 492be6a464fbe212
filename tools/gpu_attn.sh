timeout 1200 python -m pytest tests -m gpu -q -s -x > gpurun_out/gputests_attn.log 2>&1; echo "tests rc=$?"; grep -E "token-identical|passed|failed|Error|assert" gpurun_out/gputests_attn.log | cut -c1-150 | tail -25
python tools/decode_probe.py cfg2 3 | tail -1
python tools/decode_probe.py cfg4 2 | tail -1
python tools/decode_probe.py cfg5 3 | tail -1
