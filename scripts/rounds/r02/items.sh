cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_items_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_items_pytest.log
tail -n 3 gpurun_out/r02_items_pytest.log
for sh in 8 4 2; do for alt in 0 1; do
  SAB_K1_ALT=$alt timeout 200 python bench.py --workload C2 --shard-of $sh --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin 2>/dev/null | python3 -c "
import json,sys
l=[x for x in sys.stdin if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('shard $sh alt=$alt', 'NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step']))
" | tee -a gpurun_out/r02_items_ab.txt
done; done
cp paper_2410_02367_b200/libsageattn_b200.so /tmp/orig.so
cp paper_2410_02367_b200/libsab_trace.so paper_2410_02367_b200/libsageattn_b200.so
for spec in "C4-128-1024-nc 5" "C4-128-1024-c 5" "C4-64-1024-nc 5"; do
  set -- $spec
  timeout 120 python scripts/trace_k2.py $1 $2 gpurun_out/r02_items_$1.npy > /dev/null 2>&1
  echo "== $spec"; python scripts/trace_items.py gpurun_out/r02_items_$1.npy
done > gpurun_out/r02_items.txt 2>&1
cp /tmp/orig.so paper_2410_02367_b200/libsageattn_b200.so
cat gpurun_out/r02_items.txt
