cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARIANTS="libsageattn_b200 sk_nokv sk_nobias sk_noexp sk_all" WORKLOADS="C4-128-16384-nc C4-64-16384-nc" TAG=r02_exp2 BENCH_ARGS="--no-secondary --no-dropin" bash scripts/ab.sh 2>/dev/null
