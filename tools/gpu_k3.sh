cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
  -k regex:"select|sparse_stream|sparse_order" --csv python tools/prof_one.py ${CFG:-hyv110k} 1 > gpurun_out/k3_${CFG:-hyv110k}.csv 2> gpurun_out/k3_err.txt
python - <<'PY'
import csv, os
f = "gpurun_out/k3_%s.csv" % os.environ.get("CFG", "hyv110k")
rows = [r for r in csv.reader(open(f)) if len(r) > 10]
h = rows[0]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
for r in rows[1:]:
    print(f"{r[ik][:40]:40s} {r[im]:60s} {r[iv]}")
PY
