# usage: bash scripts/gpu_x4.sh <tag> : class-layout tests + bench (+ ncu of the transfer)
cd $GRAFT_REPO_ROOT
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_xlayout.py -x -q -p no:cacheprovider --timeout 600 > gpurun_out/${TAG}_xtest.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_xtest.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_transfer -s 1 -c 1 -o gpurun_out/${TAG}_transfer python scripts/profile_one.py 30 2 0 4 > gpurun_out/${TAG}_transfer.txt 2>&1
tail -n 2 gpurun_out/${TAG}_xtest.txt
