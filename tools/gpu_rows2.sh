for R in 320 768 512 5; do for kk in 5 12 1; do ./build/bench_logits_tc $R rows $kk | head -1; done; done
./build/bench_logits_tc 320 rows 5
