# usage: bash scripts/gpu_profile.sh <tag>
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_one.py 30 3 > gpurun_out/${TAG}_launches_stdout.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lap -s 2 -c 1 -o gpurun_out/${TAG}_lap2 python scripts/profile_one.py 30 1 8 > gpurun_out/${TAG}_ncu_lap2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_transfer -s 1 -c 1 -o gpurun_out/${TAG}_transfer python scripts/profile_one.py 30 2 > gpurun_out/${TAG}_ncu_transfer.txt 2>&1
ls -la gpurun_out
