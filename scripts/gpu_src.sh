# usage: bash scripts/gpu_src.sh <tag> : ncu source counters (instructions per source line) of the
# level-2 LAP kernel at iteration 1, N = 30
cd $GRAFT_REPO_ROOT
TAG=${1:-s}
mkdir -p gpurun_out
timeout 900 ncu --section SourceCounters --section InstructionStats --clock-control none --import-source on -k regex:k_lap -s 2 -c 1 -o gpurun_out/${TAG}_lap2 python scripts/profile_one.py 30 1 0 0 > gpurun_out/${TAG}_ncu_lap2.txt 2>&1
ls -la gpurun_out/ | grep ${TAG}_
