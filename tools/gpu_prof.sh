# ncu evidence: launch list of a short bench run, then one --set full capture per hot kernel.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CFG=${CFG:-hyv110k}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}.csv \
  python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_${CFG}.log 2>&1
echo "launches exit $?"
for K in "attn_fwd_kernel<128, false, false>:K1" "search_kernel:K2" "select_rows_kernel:K3" "attn_fwd_kernel<128, false, true>:K4"; do
  pat="${K%%:*}"; tag="${K##*:}"
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:${pat%%<*}" \
    $( [ "$tag" = K1 ] && echo "-s 0" ) $( [ "$tag" = K4 ] && echo "-s 1" ) -c 1 \
    -o gpurun_out/prof_${CFG}_${tag} -f python tools/prof_one.py $CFG 1 > gpurun_out/prof_${CFG}_${tag}.log 2>&1
  echo "$tag exit $?"
done
ls -la gpurun_out
