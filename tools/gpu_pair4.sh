cd "$GRAFT_REPO_ROOT" || exit 1
export ADASPA_PAIR=1
for K in "test_dense_token" "test_block_sparse_attn and tiny-over0" "test_block_sparse_attn and tiny_tf-over1" "test_block_sparse_attn and tiny-over2" "test_block_sparse_attn and tiny_tf-over3" "test_block_sparse_attn and tiny-over4" "test_block_sparse_attn and tiny_tf-over5" "test_end_to_end" "test_run_sparse_host"; do
  echo "=== $K"
  timeout 60 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$K" 2>&1 | grep -E "passed|failed|Error|assert|error|Timeout" | head -4
  echo "rc $?"
done
