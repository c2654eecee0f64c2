# usage: bash scripts/gpu_x3.sh <tag> : class-layout tests, bench, ncu of the level-2 LAP kernel
cd $GRAFT_REPO_ROOT
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_xlayout.py tests/test_gpu_transfer.py -x -q -p no:cacheprovider --timeout 600 > gpurun_out/${TAG}_xtest.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_xtest.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lap -s 2 -c 1 -o gpurun_out/${TAG}_lap2 python scripts/profile_one.py 30 1 0 4 > gpurun_out/${TAG}_lap2.txt 2>&1
tail -n 3 gpurun_out/${TAG}_xtest.txt
