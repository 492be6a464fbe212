for T in 256 160 128; do echo "select threads $T"; AMUN_SELECT_THREADS=$T python tools/decode_probe.py cfg2 3 | tail -1; done
python tools/decode_probe.py cfg2 3 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
