# K2 L2 raster-group budget sweep (SAB_L2_GROUP_MB) on a few workloads.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for mb in ${MBS:-8 24 48 96 200}; do for w in ${WORKLOADS:-C2 C4-128-16384-nc}; do
  SAB_L2_GROUP_MB=$mb timeout 120 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 1 --no-cpu-baseline > /tmp/b.log 2>&1
  echo "$mb $w $(python3 -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('NA' if d is None else 'k2=%.1f k2ms=%.4f mhz=%s' % (d['roofline']['achieved'], d['roofline']['ms_per_launch'], d['clocks']['sm_mhz']))
")" | tee -a gpurun_out/${TAG:-l2}_sweep.txt
done; done
