for U in 160 96 128 192; do echo "unit rows $U"; for R in 320 512 768; do ./build/bench_swap_u$U $R swap 5 | head -1; done; done
