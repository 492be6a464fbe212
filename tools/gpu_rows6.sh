python tools/decode_probe.py cfg5 4 | tail -2
AMUN_LOGIT_ROWS=1 python tools/decode_probe.py cfg5 4 | tail -2
python bench.py --config cfg5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(d['value'])"
