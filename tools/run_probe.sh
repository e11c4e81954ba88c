set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for w in select dense search sparse; do
  timeout 120 python tools/gpu_probe.py $w tiny 2>&1 | tail -15
  echo "exit $?"
done
timeout 120 python tools/gpu_probe.py dense tiny "dict(f=5,h=9,w=11,n_text=37,head_dim=128,block=128)" 2>&1 | tail -8
timeout 120 python tools/gpu_probe.py search tiny "dict(f=5,h=9,w=11,n_text=37,head_dim=128,block=128)" 2>&1 | tail -8
timeout 120 python tools/gpu_probe.py sparse tiny "dict(f=5,h=9,w=11,n_text=37,head_dim=128,block=128)" 2>&1 | tail -8
