timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
python tools/decode_probe.py cfg2 3 | tail -1
python tools/decode_probe.py cfg4 3 | tail -1
python tools/decode_probe.py cfg5 3 | tail -1
