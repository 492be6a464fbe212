python tools/decode_probe.py cfg2 3 | tail -1
AMUN_DISPATCH=mix python tools/decode_probe.py cfg2 3 | tail -1
AMUN_DISPATCH=mix AMUN_AHEAD_CTAS=296 python tools/decode_probe.py cfg2 3 | tail -1
AMUN_AHEAD_CTAS=296 python tools/decode_probe.py cfg2 3 | tail -1
AMUN_DEBUG_SCHED=1 python tools/decode_probe.py cfg2 1 2>&1 | tail -30
