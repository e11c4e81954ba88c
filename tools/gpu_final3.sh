# Final evidence of the round: GPU tests, smoke, bench (HYV default, CogX, reference arm), ncu launch
# list + --set full captures (HYV), clocks recorded by bench.py.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "exit $?" >> gpurun_out/bench.log
timeout 900 python bench.py > gpurun_out/bench2.log 2>&1; echo "exit $?" >> gpurun_out/bench2.log
timeout 900 python bench.py --config cogx45k --no-cpu-baseline > gpurun_out/bench_cogx.log 2>&1; echo "exit $?" >> gpurun_out/bench_cogx.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "exit $?" >> gpurun_out/bench_ref.log
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
bash tools/gpu_prof.sh > gpurun_out/prof.log 2>&1
echo done
