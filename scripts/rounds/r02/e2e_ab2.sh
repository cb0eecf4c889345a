cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in C4-128-16384-nc C2 C3 C4-128-1024-c; do
  for cfg in "SAB_HOST_RAMP=0" "SAB_HOST_RAMP=1" "SAB_HOST_CHUNK_UNITS=8" "SAB_HOST_CHUNK_UNITS=16" "SAB_HOST_RAMP=1 SAB_HOST_STREAMS=1"; do
    echo "$cfg $(env $cfg timeout 300 python scripts/rounds/r02/e2e_probe.py $w 4 2>&1 | tail -1)" | tee -a gpurun_out/r02_e2e_ab2.txt
  done
done
timeout 600 python -m pytest tests -q -x -m gpu -k "host or dropin or capi or dist or shard" > gpurun_out/r02_e2e_tests.log 2>&1; echo rc=$? >> gpurun_out/r02_e2e_tests.log
