for b in build/bench_rows_s3_e4 build/bench_rows_s4_e2 ; do echo $b; for R in 320 768 512 5; do for kk in 5 12 1; do $b $R rows $kk | head -1; done; done; $b 320 rows 5 | tail -6; done
