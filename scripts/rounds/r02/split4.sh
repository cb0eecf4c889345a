cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2410_02367_b200/libsageattn_b200.so /tmp/orig.so
for v in libsageattn_b200 sk_nomerge sk_nopart; do
 cp paper_2410_02367_b200/$v.so /tmp/v.so; cp /tmp/v.so paper_2410_02367_b200/libsageattn_b200.so
 for c in 0 8 15 64; do
  export SAB_KV_SPLIT=$c
  timeout 200 python bench.py --workload C2 --shard-of 8 --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin > /tmp/s.json 2>&1
  python3 -c "
import json
l=[x for x in open('/tmp/s.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$v split=$c', 'NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step']))
" | tee -a gpurun_out/r02_split_sweep4.txt
 done
done
cp /tmp/orig.so paper_2410_02367_b200/libsageattn_b200.so
