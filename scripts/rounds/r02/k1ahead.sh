cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARIANTS="k1a0 k1a296 k1a592 k1a1184 k1a0 k1a592" WORKLOADS="C2 C4-128-16384-nc C4-128-1024-c C3" TAG=r02_k1ahead BENCH_ARGS="--no-secondary --no-dropin" bash scripts/ab.sh 2>/dev/null
