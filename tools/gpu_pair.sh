# Bring-up of the CTA-pair kernel: short timeouts, first the smallest dense case.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "test_dense_attn_lse" > gpurun_out/pair_dense.log 2>&1; echo "exit $?" >> gpurun_out/pair_dense.log
tail -30 gpurun_out/pair_dense.log
grep -q "exit 0" gpurun_out/pair_dense.log || exit 1
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
timeout 200 python tools/quick_timing.py hyv110k > gpurun_out/quick_hyv.log 2>&1; echo "exit $?" >> gpurun_out/quick_hyv.log
ADASPA_NO_PAIR=1 timeout 200 python tools/quick_timing.py hyv110k > gpurun_out/quick_hyv_nopair.log 2>&1; echo "exit $?" >> gpurun_out/quick_hyv_nopair.log
grep -v "per-head\|head recall" gpurun_out/quick_hyv.log gpurun_out/quick_hyv_nopair.log
