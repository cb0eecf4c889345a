cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in "C2 --shard-of 8" "C2" "C4-128-1024-c"; do echo "== $w"; timeout 120 python scripts/timeline.py $w; done > gpurun_out/r02_timeline.txt 2>&1
cat gpurun_out/r02_timeline.txt
