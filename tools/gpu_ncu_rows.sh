mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:logits_rows --launch-skip 3 --launch-count 1 -o gpurun_out/rows320 ./build/bench_logits_tc 320 rows 5 > gpurun_out/ncu_rows.log 2>&1; echo rc=$?
