# One GPU call: parity tests, smoke, quick per-kernel timing, bench line.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python tools/quick_timing.py hyv110k > gpurun_out/quick_hyv.log 2>&1; echo "exit $?" >> gpurun_out/quick_hyv.log
timeout 600 python tools/quick_timing.py cogx45k > gpurun_out/quick_cogx.log 2>&1; echo "exit $?" >> gpurun_out/quick_cogx.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "exit $?" >> gpurun_out/bench.log
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/quick_hyv.log gpurun_out/quick_cogx.log; tail -3 gpurun_out/bench.log
