cd "$GRAFT_REPO_ROOT" || exit 1
export ADASPA_PAIR=1
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k hyv110k 2>&1 | grep -E "Error|assert|error|FAIL|passed|failed" | head -20
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider 2>&1 | tail -5
ADASPA_LIB=build/lib_trace_a4.so timeout 120 python tools/trace_pair.py 2>&1 | tail -22
