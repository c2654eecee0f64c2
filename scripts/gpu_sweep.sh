cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/sweep_lap.py ${2:-30} > gpurun_out/${1}_sweep.txt 2>&1
cat gpurun_out/${1}_sweep.txt
