cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/r02_dropin_threads.txt
for t in 8 16 32 64; do
  SAB_HOST_COPY_THREADS=$t timeout 300 python bench.py --workload C4-128-16384-nc --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-secondary > /tmp/b.log 2>&1
  echo "threads=$t $(python3 -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[0]) if l else {}
print(d.get('e2e',{}).get('value'), d.get('e2e_dropin'))
")" >> gpurun_out/r02_dropin_threads.txt
done
