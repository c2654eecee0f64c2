# A/B of the Dijkstra-loop unroll + source profile at iteration 10
cd $GRAFT_REPO_ROOT
VAR=QAP_LAP_UNROLL VALS="2 1 2 1" K="lap_kernel or config4_n30_full or phase" bash scripts/gpu_ab2.sh un
bash scripts/gpu_src.sh s10 10
