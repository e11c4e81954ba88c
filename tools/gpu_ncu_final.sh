#!/bin/bash
# The evidence set of a round's final state on one gpurun box: the GPU test suite, the bench lines
# (HYV-110K default, CogX-45K, reference arm), an ncu launch list of one bench step, and `ncu --set
# full` captures of every kernel of the step, one kernel per report (the fused search's dense pass
# with 2-head passes: ncu's replay saves and restores what a launch writes, 0.8 GB of block LSEs then).
# Usage: tools/gpu_ncu_final.sh TAG
tag=$1
python -m pytest tests -m gpu -q --durations=8 > gpurun_out/${tag}_pytest_gpu.txt 2>&1
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
python bench.py --config cogx45k > gpurun_out/${tag}_bench_cogx45k.json 2>> gpurun_out/${tag}_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2>> gpurun_out/${tag}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python tools/prof_step.py hyv110k 2 > /dev/null 2>&1
N="ncu --set full --import-source on --clock-control none"
$N -k regex:attn_fwd_kernel -c 1 -o gpurun_out/${tag}_k1 -f python tools/prof_step.py hyv110k 1 > gpurun_out/${tag}_ncu.log 2>&1
$N -k regex:attn_fwd_kernel --launch-skip 2 -c 1 -o gpurun_out/${tag}_k4 -f python tools/prof_step.py hyv110k 1 >> gpurun_out/${tag}_ncu.log 2>&1
$N -k regex:attn_fwd_kernel --launch-skip 1 -c 1 -o gpurun_out/${tag}_fs -f python tools/prof_step.py hyv110k 1 2 >> gpurun_out/${tag}_ncu.log 2>&1
$N -k regex:"block_mass|search_kernel|select_rows" -c 3 -o gpurun_out/${tag}_other -f python tools/prof_step.py hyv110k 1 >> gpurun_out/${tag}_ncu.log 2>&1
$N -k regex:"select_(rows|head|scan|write)" -c 4 -o gpurun_out/${tag}_k3 -f python tools/k3_bench.py hyv110k 1 >> gpurun_out/${tag}_ncu.log 2>&1
for r in k1 k4 fs other k3; do
  ncu -i gpurun_out/${tag}_${r}.ncu-rep --page raw --csv > gpurun_out/${tag}_${r}.raw.csv 2>/dev/null
done
ncu -i gpurun_out/${tag}_k1.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_k1.source.csv 2>/dev/null
gzip -f gpurun_out/${tag}_k1.source.csv
rm -f gpurun_out/${tag}_*.ncu-rep
tail -2 gpurun_out/${tag}_pytest_gpu.txt
