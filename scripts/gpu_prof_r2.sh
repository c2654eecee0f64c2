# usage: bash scripts/gpu_prof_r2.sh <tag> : ncu --set full (source counters) of the level-2 LAP
# kernel at iteration 1 and of the transfer, N = 30
cd $GRAFT_REPO_ROOT
TAG=${1:-p}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lap -s 2 -c 1 -o gpurun_out/${TAG}_lap2 python scripts/profile_one.py 30 1 0 0 > gpurun_out/${TAG}_ncu_lap2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_transfer -s 1 -c 1 -o gpurun_out/${TAG}_transfer python scripts/profile_one.py 30 2 0 0 > gpurun_out/${TAG}_ncu_transfer.txt 2>&1
ls -la gpurun_out/ | grep ${TAG}
