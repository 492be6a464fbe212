python tools/decode_probe.py cfg2 3 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
python bench.py --no-cpu-baseline > gpurun_out/bench_insitu.json 2>gpurun_out/bench_insitu.err; echo rc=$?
