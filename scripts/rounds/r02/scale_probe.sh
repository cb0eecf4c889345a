cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in "C4-128-16384-nc" "C3" "C5"; do
 for sh in 8 4; do for pers in unset 0; do
  if [ $pers = unset ]; then unset SAB_K2_PERSIST; else export SAB_K2_PERSIST=$pers; fi
  timeout 400 python bench.py --workload $w --shard-of $sh --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-secondary --no-dropin > /tmp/s.json 2>&1
  python3 -c "
import json
l=[x for x in open('/tmp/s.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$w shard-of $sh persist=$pers', 'NA' if d is None else '%.1f ms=%.4f k2=%.1f k2ms=%.4f k1ms=%.4f mhz=%s %s split=%s' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['clocks']['sm_mhz'], d['config'].get('k2_launch'), d['config'].get('kv_split')))
" | tee -a gpurun_out/r02_scale_probe.txt
 done; done
done
unset SAB_K2_PERSIST
