# A/B of the host-path (e2e) chunking across library variants.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp paper_2410_02367_b200/libsageattn_b200.so /tmp/lib_orig.so
for v in $VARIANTS; do
  cp paper_2410_02367_b200/$v.so paper_2410_02367_b200/libsageattn_b200.so
  for w in ${WORKLOADS:-C2}; do
    timeout 200 python bench.py --workload $w --steps 5 --warmup 3 --e2e-steps 5 --no-cpu-baseline > /tmp/b.log 2>&1
    echo "$v $w $(python3 -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('NA' if d is None else 'e2e=%.1f value=%.1f' % (d['e2e']['value'], d['value']))
")" | tee -a gpurun_out/${TAG:-e2e}_ab.txt
  done
done
cp /tmp/lib_orig.so paper_2410_02367_b200/libsageattn_b200.so
