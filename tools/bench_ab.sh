for r in 1 2 3; do
for lib in lib_rt0 lib_cur; do
ADASPA_LIB=variants/$lib.so python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-variants > gpurun_out/r02ab_$lib.$r.json 2>/dev/null
python -c "
import json
d=json.loads(open('gpurun_out/r02ab_$lib.$r.json').read().strip().splitlines()[-1])
k=d['kernels']
print('$lib', $r, 'K4', k['K4_block_sparse_attn']['ms'], 'K1', k['K1_dense_attn_lse']['ms'], 'FS', k['K1K2K3_search_step']['ms'], 'K2', k['K2_lse_cached_search']['ms'], d['clocks']['sm_mhz'])
"
done; done
