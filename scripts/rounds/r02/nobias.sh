cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARIANTS="libsageattn_b200 v_nobias libsageattn_b200 v_nobias" WORKLOADS="C4-128-16384-nc C2 C4-64-16384-nc" TAG=r02_nobias BENCH_ARGS="--no-secondary --no-dropin" bash scripts/ab.sh 2>/dev/null
