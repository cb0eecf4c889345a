# Locate the C2 --shard-of 8 segfault; fused-K1 lag sweep; C4 / C3 shard proxies.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {  # label, env, bench args
  local label="$1" envs="$2"; shift 2
  env $envs timeout 180 python -X faulthandler bench.py "$@" --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline > /tmp/b.log 2>&1
  local rc=$?
  echo "$label $* rc=$rc $(python3 -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f k1frac=%.3f mhz=%s e2e=%.1f' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['roofline_k1']['frac'], d['clocks']['sm_mhz'], d['e2e']['value']))
")" | tee -a gpurun_out/shard_dbg.txt
  if [ $rc -ne 0 ]; then tail -30 /tmp/b.log > gpurun_out/shard_dbg_${label}.log; fi
}
run base "SAB_K1_FUSED=0" --workload C2 --shard-of 8
run streams1 "SAB_K1_FUSED=0 SAB_HOST_STREAMS=1" --workload C2 --shard-of 8
run noramp "SAB_K1_FUSED=0 SAB_HOST_RAMP=0 SAB_HOST_STREAMS=1" --workload C2 --shard-of 8
run nopersist "SAB_K1_FUSED=0 SAB_K2_PERSIST=0" --workload C2 --shard-of 8
run shard4 "SAB_K1_FUSED=0" --workload C2 --shard-of 4
for lag in 300 600 1500; do
  run lag$lag "SAB_K1_FUSED=1 SAB_K1_LAG_PCT=$lag" --workload C4-128-16384-nc
  run lag$lag "SAB_K1_FUSED=1 SAB_K1_LAG_PCT=$lag" --workload C4-128-1024-c
done
run c4s8 "SAB_K1_FUSED=0" --workload C4-128-16384-nc --shard-of 8
run c3s8 "SAB_K1_FUSED=0" --workload C3 --shard-of 8
