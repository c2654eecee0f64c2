# usage: bash scripts/gpu_src.sh <tag> [T] : ncu source counters (instructions per source line) of
# the level-2 LAP kernel at iteration T (default 1), N = 30
cd $GRAFT_REPO_ROOT
TAG=${1:-s}
T=${2:-1}
S=$((2 + 3 * (T - 1)))
mkdir -p gpurun_out
timeout 900 ncu --section SourceCounters --section InstructionStats --clock-control none --import-source on -k regex:k_lap -s $S -c 1 -o gpurun_out/${TAG}_lap2 python scripts/profile_one.py 30 $T 0 0 > gpurun_out/${TAG}_ncu_lap2.txt 2>&1
ls -la gpurun_out/ | grep ${TAG}_
