# usage: bash scripts/gpu_x5.sh <tag> : fused-kernel tests + bench both ways
cd $GRAFT_REPO_ROOT
TAG=${1:-x}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_xlayout.py -x -q -p no:cacheprovider --timeout 300 -k fused > gpurun_out/${TAG}_xtest.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_xtest.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb --fused > gpurun_out/${TAG}_benchf.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_benchf.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
tail -n 2 gpurun_out/${TAG}_xtest.txt
