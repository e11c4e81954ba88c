cd "$GRAFT_REPO_ROOT" || exit 1
export ADASPA_PAIR=1
timeout 120 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "test_block_sparse_attn and tiny-over2" 2>&1 | tail -2
timeout 400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 150 python tools/quick_timing.py hyv110k 2>&1 | grep -E "^K1|^K4" | sed "s/^/pair /"
