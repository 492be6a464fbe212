python tools/decode_probe.py cfg2 3 | tail -1
AMUN_ABLATE_CLASSES=1 python tools/decode_probe.py cfg2 3 | tail -1
python bench.py --config cfg4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);r=d['roofline'];print('cfg4',d['value'],r['insitu_sm_share'],r['kernel'],r['frac'])"
python bench.py --config cfg5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);r=d['roofline'];print('cfg5',d['value'],r['insitu_sm_share'],r['kernel'],r['frac'])"
