cd "$GRAFT_REPO_ROOT" || exit 1
timeout 200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "search or end_to_end or smoke" 2>&1 | tail -2
for M in 4 0 8 3; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared \
    -DADASPA_SEARCH_POLY_MOD=$M paper_2502_21079_b200/csrc/*.cu -o /tmp/lib_s$M.so > /dev/null 2>&1 || { echo build fail; exit 1; }
  echo "== search poly mod $M"
  ADASPA_LIB=/tmp/lib_s$M.so timeout 120 python tools/quick_timing.py hyv110k 2>&1 | grep -E "K2"
  ADASPA_LIB=/tmp/lib_s$M.so timeout 120 python tools/quick_timing.py cogx45k 2>&1 | grep -E "K2"
done
