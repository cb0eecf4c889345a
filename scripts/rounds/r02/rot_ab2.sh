cd $GRAFT_REPO_ROOT
export VARIANTS="v_r0 v_rd v_ra v_rb v_rc v_r0 v_rd v_ra v_rb v_rc" WORKLOADS="C3 C2 C4-64-4096-c"
TAG=r02_rot2 BENCH_ARGS="--no-secondary --no-dropin" bash scripts/ab.sh
