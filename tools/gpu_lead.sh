for L in 0 256 512 1024; do echo "lead $L"; AMUN_ENC_LEAD=$L python tools/decode_probe.py cfg2 3 | tail -1; done
AMUN_DEBUG_SCHED=1 python tools/decode_probe.py cfg2 2 2>&1 | grep sched | tail -1
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
