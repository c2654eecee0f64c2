# usage: bash scripts/gpu_round_profile.sh <tag> : bench + launch list of the bench command + ncu --set full of lap2 and transfer
cd $GRAFT_REPO_ROOT
TAG=${1:-r}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_launches_stdout.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lap -s 2 -c 1 -o gpurun_out/${TAG}_lap2 python scripts/profile_one.py 30 1 0 4 > gpurun_out/${TAG}_ncu_lap2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_transfer -s 1 -c 1 -o gpurun_out/${TAG}_transfer python scripts/profile_one.py 30 2 0 4 > gpurun_out/${TAG}_ncu_transfer.txt 2>&1
tail -n 2 gpurun_out/${TAG}_bench.txt | cut -c1-400
