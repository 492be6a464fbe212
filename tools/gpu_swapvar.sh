for b in build/bench_swap_s3_e3 build/bench_swap_s2_e4; do echo $b; for R in 320 768 512; do for kk in 5 1; do $b $R swap $kk | head -1; done; done; done
