# 16-row-warp softmax: parity, then K1/K4 timing with exp-offload variants (HYV-110K, CogX-45K).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
for V in p0 p2 p4 p8; do
  L=build/lib_$V.so; [ $V = p0 ] && L=paper_2502_21079_b200/libadaspa.so
  for W in hyv110k cogx45k; do
    ADASPA_LIB=$L timeout 150 python tools/quick_timing.py $W 2>&1 | grep -E "^K1|^K4|^K2" | sed "s/^/$V $W /"
  done
done
