timeout 1200 python -m pytest tests -m gpu -q -s -x > gpurun_out/gputests_thr.log 2>&1; echo "tests rc=$?"; grep -E "token-identical|passed|failed|Error|assert" gpurun_out/gputests_thr.log | cut -c1-150 | tail -25
python tools/decode_probe.py cfg2 3 | tail -1
python tools/decode_probe.py cfg5 3 | tail -1
python tools/decode_probe.py cfg1 3 | tail -1
SL_CFG=cfg2 python tools/shortlist_bench.py | tail -2
