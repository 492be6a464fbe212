timeout 1500 python -m pytest tests -m gpu -q -s -x 2>&1 | grep -E "identical|states at|passed|failed|Error|assert" | cut -c1-180
python tools/decode_probe.py cfg2 3 | tail -1
python tools/decode_probe.py cfg2 3 | tail -1
python tools/decode_probe.py cfg4 3 | tail -1
python tools/decode_probe.py cfg5 3 | tail -1
python tools/load_probe.py 2>&1 | tail -2
