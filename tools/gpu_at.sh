for T in 512 256; do echo "attn threads $T"; AMUN_ATTN_THREADS=$T python tools/decode_probe.py cfg2 3 | tail -1; AMUN_ATTN_THREADS=$T python tools/decode_probe.py cfg5 3 | tail -1; done
