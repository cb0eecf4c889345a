# Drop-in e2e (sageattn::sage_attention on fp32 Tensor4f): O storage advised onto huge pages or not.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat /sys/kernel/mm/transparent_hugepage/enabled > gpurun_out/thp_ab.txt
for rep in 1 2; do for t in 1 0; do
  SAB_DROPIN_THP=$t timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-secondary > /tmp/b.log 2>&1
  echo "THP=$t rc=$? $(python3 -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('NA' if d is None else 'dropin %.2f TOPS %.4f s/call; e2e %.1f' % (d['e2e_dropin']['value'], d['e2e_dropin']['seconds_per_call'], d['e2e']['value']))
")" | tee -a gpurun_out/thp_ab.txt
done; done
