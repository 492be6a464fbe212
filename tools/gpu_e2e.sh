timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err; echo rc=$?
python tools/e2e_breakdown.py 2>&1 | tail -12
