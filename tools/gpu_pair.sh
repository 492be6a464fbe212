for kk in 12 5; do ./build/bench_logits_tc 768 rows $kk | head -1; AMUN_LOGIT_ROWS_PAIR=0 ./build/bench_logits_tc 768 rows $kk | head -1; ./build/bench_logits_tc 512 rows $kk | head -1; AMUN_LOGIT_ROWS_PAIR=0 ./build/bench_logits_tc 512 rows $kk | head -1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x -k "pair_and_cluster or extra or (fullset and cfg4)" 2>&1 | grep -E "identical|passed|failed|Error|assert" | cut -c1-200
python tools/decode_probe.py cfg4 3 | tail -1
AMUN_LOGIT_ROWS_PAIR=0 python tools/decode_probe.py cfg4 3 | tail -1
