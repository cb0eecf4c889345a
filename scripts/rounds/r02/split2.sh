cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 0 15 24 32 48 64; do
  SAB_KV_SPLIT=$c timeout 200 python bench.py --workload C2 --shard-of 8 --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin > /tmp/s.json 2>&1
  python3 -c "
import json
l=[x for x in open('/tmp/s.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('split=$c', 'NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f split=%s' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['config'].get('kv_split')))
" | tee -a gpurun_out/r02_split_sweep.txt
done
SAB_KV_SPLIT=15 timeout 300 ncu --set full --clock-control none -k regex:k2_attention -s 3 -c 1 -o gpurun_out/r02_split15 python bench.py --workload C2 --shard-of 8 --steps 2 --warmup 2 --e2e-steps 1 --no-cpu-baseline --no-secondary --no-dropin > /dev/null 2>&1
SAB_KV_SPLIT=0 timeout 300 ncu --set full --clock-control none -k regex:k2_attention -s 3 -c 1 -o gpurun_out/r02_split0 python bench.py --workload C2 --shard-of 8 --steps 2 --warmup 2 --e2e-steps 1 --no-cpu-baseline --no-secondary --no-dropin > /dev/null 2>&1
ls gpurun_out
