for n in 32 64 128; do echo "split ctas $n"; AMUN_AHEAD_SPLIT_CTAS=$n python tools/enc_only.py 3 | tail -1; AMUN_AHEAD_SPLIT_CTAS=$n python tools/decode_probe.py cfg2 3 | tail -1; done
