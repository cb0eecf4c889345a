# Shard proxies (rank 0's K3 shard of an N-GPU strong-scaling run on one GPU) with the
# two-launch K1 and with k1_fused; the drop-in e2e now uses the shard's own unit count.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {  # label, env, bench args
  local label="$1" envs="$2"; shift 2
  env $envs timeout 240 python -X faulthandler bench.py "$@" --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline > /tmp/b.log 2>&1
  local rc=$?
  cp /tmp/b.log gpurun_out/shard2_${label}_$(echo "$*" | tr ' -' '__').log
  echo "$label $* rc=$rc $(python3 -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f k1frac=%.3f mhz=%s e2e=%.1f' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['roofline_k1']['frac'], d['clocks']['sm_mhz'], d['e2e']['value']))
")" | tee -a gpurun_out/shard2.txt
}
for g in 8 4 2; do
  run base "SAB_K1_FUSED=0" --workload C2 --shard-of $g
  run fused "SAB_K1_FUSED=1" --workload C2 --shard-of $g
done
run base "SAB_K1_FUSED=0" --workload C4-128-16384-nc --shard-of 8
run base "SAB_K1_FUSED=0" --workload C4-128-16384-nc --shard-of 4
run base "SAB_K1_FUSED=0" --workload C3 --shard-of 8
run fused "SAB_K1_FUSED=1" --workload C3 --shard-of 8
run base "SAB_K1_FUSED=0" --workload C5 --shard-of 8
run fused "SAB_K1_FUSED=1" --workload C5 --shard-of 8
run base "SAB_K1_FUSED=0" --workload C4-128-1024-c --shard-of 8
run fused "SAB_K1_FUSED=1" --workload C4-128-1024-c --shard-of 8
