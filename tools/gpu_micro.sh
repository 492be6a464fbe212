mkdir -p gpurun_out
for R in 320 160; do ./build/bench_logits_tc $R; done > gpurun_out/micro_logits.txt 2>&1
./build/bench_sk > gpurun_out/micro_sk.txt 2>&1
cat gpurun_out/micro_logits.txt; tail -40 gpurun_out/micro_sk.txt
