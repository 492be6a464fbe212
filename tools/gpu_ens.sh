mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x -k "ensemble" > gpurun_out/ens.log 2>&1; echo "ens rc=$?"; grep -E "token-identical|passed|failed|Error|assert" gpurun_out/ens.log | tail -15
timeout 600 python tools/ensemble_bench.py > gpurun_out/ens_bench.txt 2>&1; echo "bench rc=$?"; cat gpurun_out/ens_bench.txt | tail -8
