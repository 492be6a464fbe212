mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_production_step.py -x -q -s > gpurun_out/prodstep.log 2>&1; echo "prodstep rc=$?"; grep -E "err|passed|failed" gpurun_out/prodstep.log | tail -6
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x -k "not cfg2-64 and not cfg5-512" > gpurun_out/parity.log 2>&1; echo "parity rc=$?"; grep -E "token-identical|passed|failed|Error|assert" gpurun_out/parity.log | tail -15
AMUN_DEBUG_SCHED=1 python tools/decode_probe.py cfg2 3 2>&1 | tail -3
AMUN_ABLATE_CLASSES=1 python tools/decode_probe.py cfg2 3 2>&1 | tail -1
