run() { echo -n "$* : "; env "$@" python tools/decode_probe.py cfg2 3 | tail -1 | sed 's/.*device//'; }
run AMUN_LANES=24
run AMUN_LANES=20
run AMUN_LANES=28
run AMUN_LANES=32
run AMUN_LOGIT_PAIRS=32
run AMUN_LOGIT_PAIRS=48
run AMUN_LANES=24
