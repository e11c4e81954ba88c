# Build exp-path variants of the trace library and trace/time each (K1 dense, HYV-110K).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for V in ${VARIANTS:-"4 1" "0 1" "0 0" "8 1" "8 0" "4 0"}; do :; done
for V in "4 1" "0 1" "0 0" "8 1" "8 0" "4 0"; do
  set -- $V
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared \
    -DADASPA_TRACE -DADASPA_EXP_POLY_MOD=$1 -DADASPA_EXP_PACKED=$2 paper_2502_21079_b200/csrc/*.cu -o /tmp/lib_$1_$2.so > /dev/null 2>&1 || { echo build fail; exit 1; }
  ADASPA_LIB=/tmp/lib_$1_$2.so timeout 120 python tools/trace_probe.py hyv110k dense > gpurun_out/var_$1_$2.txt 2>&1
  ADASPA_LIB=/tmp/lib_$1_$2.so timeout 120 python tools/quick_timing.py hyv110k 2>&1 | grep -E "K1|K4" >> gpurun_out/var_$1_$2.txt
done
for f in gpurun_out/var_*.txt; do echo "=== $f"; head -7 $f; grep -E "K1|K4" $f; done
