# ncu --set full of K1 (dense) and K2 (search) at one config (source-level stalls).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CFG=${CFG:-hyv110k}
TAG=${TAG:-v2}
for K in K1 K2 K4; do
  case $K in K1) pat=attn_fwd_kernel; skip=0;; K2) pat=search_kernel; skip=0;; K4) pat=attn_fwd_kernel; skip=1;; esac
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$pat" -s $skip -c 1 \
    -o gpurun_out/prof_${CFG}_${K}_${TAG} -f python tools/prof_one.py $CFG 1 > gpurun_out/prof_${CFG}_${K}_${TAG}.log 2>&1
  echo "$K exit $?"
done
