cd "$GRAFT_REPO_ROOT" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared -DADASPA_TRACE paper_2502_21079_b200/csrc/*.cu -o /tmp/libadaspa_trace.so || exit 1
ADASPA_LIB=/tmp/libadaspa_trace.so timeout 120 python tools/trace_probe.py hyv110k dense
ADASPA_LIB=/tmp/libadaspa_trace.so timeout 120 python tools/trace_probe.py hyv110k sparse
