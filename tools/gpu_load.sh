python tools/load_probe.py 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python tools/decode_probe.py cfg2 3 | tail -1
