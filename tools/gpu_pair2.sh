cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export ADASPA_PAIR=1
timeout 60 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "test_dense_attn_lse" 2>&1 | tail -3
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 150 python tools/quick_timing.py hyv110k 2>&1 | grep -E "^K1|^K4" | sed "s/^/pair /"
ADASPA_LIB=build/lib_trace.so timeout 120 python tools/trace_pair.py 2>&1 | tail -22
