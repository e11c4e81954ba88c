# Bring-up of the CTA-pair kernel (ADASPA_PAIR=1): short timeouts, smallest dense case first.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export ADASPA_PAIR=1
timeout 60 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "test_dense_attn_lse" > gpurun_out/pair_dense.log 2>&1; echo "exit $?" >> gpurun_out/pair_dense.log
tail -30 gpurun_out/pair_dense.log
grep -q "exit 0" gpurun_out/pair_dense.log || exit 1
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_pair.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_pair.log
tail -30 gpurun_out/pytest_gpu_pair.log
for W in hyv110k; do
  timeout 150 python tools/quick_timing.py $W 2>&1 | grep -E "^K1|^K4|^K2" | sed "s/^/pair $W /"
  ADASPA_PAIR=0 timeout 150 python tools/quick_timing.py $W 2>&1 | grep -E "^K1|^K4" | sed "s/^/one $W /"
done
