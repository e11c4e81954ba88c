# Parity tests + per-kernel timing on the two BASELINE configs (bring-up loop).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 100 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 || { echo SMOKE FAILED; tail -5 gpurun_out/smoke.log; exit 1; }
timeout 240 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 150 python tools/quick_timing.py hyv110k > gpurun_out/quick_hyv.log 2>&1; echo "exit $?" >> gpurun_out/quick_hyv.log
timeout 150 python tools/quick_timing.py cogx45k > gpurun_out/quick_cogx.log 2>&1; echo "exit $?" >> gpurun_out/quick_cogx.log
tail -15 gpurun_out/pytest_gpu.log; cat gpurun_out/quick_hyv.log gpurun_out/quick_cogx.log | grep -v "per-head\|head recall"
