# Host-buffer path: one vs two compute streams, chunk sizes; raw copy ceilings.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in C4-128-16384-nc C2 C3; do
  for cfg in "SAB_HOST_STREAMS=1" "SAB_HOST_STREAMS=2" "SAB_HOST_CHUNK_UNITS=2" "SAB_HOST_CHUNK_UNITS=4" "SAB_HOST_CHUNK_UNITS=8"; do
    echo "$cfg $(env $cfg timeout 300 python scripts/rounds/r02/e2e_probe.py $w 4 2>&1 | tail -1)" | tee -a gpurun_out/r02_e2e_ab.txt
  done
done
