cd "$GRAFT_REPO_ROOT" || exit 1
export ADASPA_PAIR=1
timeout 400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 150 python tools/quick_timing.py hyv110k 2>&1 | grep -E "^K1|^K4" | sed "s/^/pair /"
ADASPA_LIB=build/lib_trace.so timeout 120 python tools/trace_pair.py 2>&1 | tail -23
