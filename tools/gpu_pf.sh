python tools/decode_probe.py cfg2 3 | tail -1
python tools/decode_probe.py cfg2 3 | tail -1
python tools/decode_probe.py cfg4 3 | tail -1
