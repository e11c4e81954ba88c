cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for A in ${ABL:-0 1 2 3}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared \
    -DADASPA_TRACE -DADASPA_ABLATE=$A paper_2502_21079_b200/csrc/*.cu -o /tmp/lib_a$A.so > /dev/null 2>&1 || { echo build fail; exit 1; }
  echo "=== ablate $A"
  ADASPA_LIB=/tmp/lib_a$A.so timeout 120 python tools/trace_probe.py hyv110k dense 2>&1 | head -22
  ADASPA_LIB=/tmp/lib_a$A.so timeout 120 python tools/quick_timing.py hyv110k 2>&1 | grep -E "K1"
done
