# usage: bash scripts/gpu_all.sh <tag> : smoke, gpu tests, sweep, bench, ncu of lap2 + transfer
cd $GRAFT_REPO_ROOT
TAG=${1:-r}
mkdir -p gpurun_out
bash scripts/gpu_check.sh $TAG > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lap -s 2 -c 1 -o gpurun_out/${TAG}_lap2 python scripts/profile_one.py 30 1 > gpurun_out/${TAG}_ncu_lap2.txt 2>&1
tail -n 3 gpurun_out/${TAG}_smoke.txt gpurun_out/${TAG}_pytest.txt gpurun_out/${TAG}_sweep.txt
