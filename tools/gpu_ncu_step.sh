#!/bin/bash
# ncu --set full captures of every kernel of one bench step (tools/prof_step.py) on a config;
# reports land in gpurun_out/<tag>_<kernel>.ncu-rep.  Usage: tools/gpu_ncu_step.sh TAG [config]
tag=$1; cfg=${2:-hyv110k}
N="ncu --set full --import-source on --clock-control none"
$N -k regex:attn_fwd_kernel -c 3 -o gpurun_out/${tag}_attn -f python tools/prof_step.py $cfg > gpurun_out/${tag}_ncu_attn.log 2>&1
$N -k regex:"block_mass|search_kernel|select_rows_kernel" -c 3 -o gpurun_out/${tag}_other -f python tools/prof_step.py $cfg > gpurun_out/${tag}_ncu_other.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv python tools/prof_step.py $cfg 2 > /dev/null 2>&1
# export on the box (the .ncu-rep files are large): raw metrics and details per kernel, source-level
# SASS stalls of the attention kernels; the reports themselves are removed
for r in gpurun_out/${tag}_attn gpurun_out/${tag}_other; do
  ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
  ncu -i $r.ncu-rep --page details --csv > $r.details.csv 2>/dev/null
done
ncu -i gpurun_out/${tag}_attn.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_attn.source.csv 2>/dev/null
gzip -f gpurun_out/${tag}_attn.source.csv
rm -f gpurun_out/${tag}_*.ncu-rep
