AMUN_LOGIT_ROWS=0 python tools/decode_probe.py cfg2 3 | tail -1
AMUN_LOGIT_ROWS_CTAS=48 python tools/decode_probe.py cfg2 3 | tail -1
for c in 1 2; do for n in 48 72; do echo "cmax $c ctas $n"; AMUN_LOGIT_ROWS_CMAX=$c AMUN_LOGIT_ROWS_CTAS=$n python tools/decode_probe.py cfg2 3 | tail -1; done; done
for v in 0 1; do AMUN_LOGIT_ROWS=$v AMUN_LOGIT_ROWS_CTAS=48 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);r=d['roofline'];print('rows=$v',d['value'],r['kernel_ms_per_step'],r['tensor_core_classes']['logits'])"; done
