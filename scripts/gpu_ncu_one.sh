# usage: bash scripts/gpu_ncu_one.sh <tag> <kernel-regex> <skip> [N] [T] [lapcfg]
# Runs with QAP_FLAG_NO_GRAPH (4): ncu cannot replay the graph-captured k_lap node
# (LaunchFailed under ncu only); the kernels and launch configurations are identical.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/$1 python scripts/profile_one.py ${4:-30} ${5:-2} ${6:-0} 4 > gpurun_out/$1.txt 2>&1
tail -3 gpurun_out/$1.txt
