for H in 0 1 2 4; do echo "prio $H"; AMUN_PRIO_BUCKETS=$H AMUN_DEBUG_SCHED=1 python tools/decode_probe.py cfg2 3 2>&1 | grep -E "sched|rep 2" | tail -2; done
