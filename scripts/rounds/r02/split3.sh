cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_split.py -m gpu -q -x > gpurun_out/r02_split6_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_split6_pytest.log
tail -3 gpurun_out/r02_split6_pytest.log
for c in 0 auto 32 64; do
  if [ $c = auto ]; then unset SAB_KV_SPLIT; else export SAB_KV_SPLIT=$c; fi
  timeout 200 python bench.py --workload C2 --shard-of 8 --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin > /tmp/s.json 2>&1
  python3 -c "
import json
l=[x for x in open('/tmp/s.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('split=$c', 'NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f split=%s' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['config'].get('kv_split')))
" | tee -a gpurun_out/r02_split_sweep6.txt
done
unset SAB_KV_SPLIT
for sh in 4 2; do
  timeout 200 python bench.py --workload C2 --shard-of $sh --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin > /tmp/s.json 2>&1
  python3 -c "
import json
l=[x for x in open('/tmp/s.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('shard-of $sh', 'NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f split=%s' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['config'].get('kv_split')))
" | tee -a gpurun_out/r02_split_sweep6.txt
done
