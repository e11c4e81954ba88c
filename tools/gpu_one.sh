# attn_one.cu (ADASPA_ONE=1) bring-up: dense parity + edge tests under the opt-in, then K1 timing
# with and without it.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
ADASPA_ONE=1 timeout 200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_rescale.py -x -q -p no:cacheprovider -k "dense or edge or rescale or end_to_end or hot_path" > gpurun_out/pytest_one.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_one.log
tail -25 gpurun_out/pytest_one.log
ADASPA_ONE=1 timeout 120 python tools/quick_timing.py hyv110k 2>&1 | grep -v "per-head\|head recall" | head -6
timeout 120 python tools/quick_timing.py hyv110k 2>&1 | grep "K1"
