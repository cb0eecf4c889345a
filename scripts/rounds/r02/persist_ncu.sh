cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2410_02367_b200/libsageattn_b200.so /tmp/orig.so
for v in v_head v_new; do
  cp paper_2410_02367_b200/$v.so paper_2410_02367_b200/libsageattn_b200.so
  SAB_K2_PERSIST=0 timeout 600 ncu --set full --clock-control none -k regex:k2_attention -s 2 -c 1 -o gpurun_out/r02_pncu_$v python bench.py --workload C2 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-secondary --no-dropin > /dev/null 2>&1
  SAB_K2_PERSIST=0 timeout 200 python bench.py --workload C2 --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin 2>&1 | python3 -c "
import json,sys
l=[x for x in sys.stdin if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$v C2 persist0', 'NA' if d is None else '%.1f k2=%.1f' % (d['value'], d['roofline']['achieved']))
"
  timeout 200 python bench.py --workload C2 --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin 2>&1 | python3 -c "
import json,sys
l=[x for x in sys.stdin if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$v C2 persist-default', 'NA' if d is None else '%.1f k2=%.1f' % (d['value'], d['roofline']['achieved']))
"
done
cp /tmp/orig.so paper_2410_02367_b200/libsageattn_b200.so
