mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/gputests_full.log 2>&1; echo "gpu tests rc=$?"; grep -E "token-identical|early-stopping|passed|failed|Error" gpurun_out/gputests_full.log | tail -24
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
SL_CFG=cfg1 timeout 300 python tools/shortlist_bench.py 2>&1 | tail -3
SL_CFG=cfg2 timeout 300 python tools/shortlist_bench.py 2>&1 | tail -2
