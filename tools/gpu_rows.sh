mkdir -p gpurun_out
( for R in 320 768 512 5; do for kk in 5 12 1; do ./build/bench_logits_tc $R rows $kk | head -1; ./build/bench_logits_tc $R swap $kk | head -1; done; done ) > gpurun_out/micro_rows.txt 2>&1
cat gpurun_out/micro_rows.txt
timeout 1200 python -m pytest tests -m gpu -q -s -x > gpurun_out/gputests_rows.log 2>&1; echo "tests rc=$?"; grep -E "token-identical|passed|failed|Error|assert" gpurun_out/gputests_rows.log | tail -25
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_rows.json 2>gpurun_out/bench_rows.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_rows.json'));print(d['value'],d['e2e']['value'],d['roofline']['kernel_ms_per_step'])"
for c in cfg4 cfg5 cfg1; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_rows_$c.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_rows_$c.json'));print('$c',d['value'],d.get('e2e',{}).get('value'))"; done
