# Round evidence: GPU tests, smoke, bench (default + reference arm), CogX-45K bench line, ncu launch
# lists and --set full captures for HYV-110K and CogX-45K, sanitizer on the d=64 path.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "exit $?" >> gpurun_out/bench.log
timeout 900 python bench.py --config cogx45k --no-cpu-baseline > gpurun_out/bench_cogx.log 2>&1; echo "exit $?" >> gpurun_out/bench_cogx.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "exit $?" >> gpurun_out/bench_ref.log
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/bench.log | cut -c1-400; tail -2 gpurun_out/bench_cogx.log | cut -c1-400
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_memcheck_d64.txt 2>&1; tail -1 gpurun_out/sanitizer_memcheck_d64.txt
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_synccheck_d64.txt 2>&1; tail -1 gpurun_out/sanitizer_synccheck_d64.txt
bash tools/gpu_prof.sh > gpurun_out/prof.log 2>&1
CFG=cogx45k bash tools/gpu_prof.sh > gpurun_out/prof_cogx.log 2>&1
tail -3 gpurun_out/prof.log gpurun_out/prof_cogx.log
