cd "$GRAFT_REPO_ROOT" || exit 1
export ADASPA_PAIR=1
for V in default pm00 pm92 pmAA; do
  L=build/lib_$V.so; [ $V = default ] && L=paper_2502_21079_b200/libadaspa.so
  ADASPA_LIB=$L timeout 150 python tools/quick_timing.py hyv110k 2>&1 | grep -E "^K1|^K4" | sed "s/^/$V /"
done
