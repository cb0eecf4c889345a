cd $GRAFT_REPO_ROOT
export VARIANTS="v_p2 v_p3 v_p4 v_p4r0 v_p3r4 v_p2 v_p3 v_p4 v_p4r0 v_p3r4" WORKLOADS="C3 C4-64-4096-c"
TAG=r02_poly64 BENCH_ARGS="--no-secondary --no-dropin" bash scripts/ab.sh
