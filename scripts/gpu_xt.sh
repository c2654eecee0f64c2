# usage: bash scripts/gpu_xt.sh <tag> : class-layout + transfer GPU tests
cd $GRAFT_REPO_ROOT
TAG=${1:-xt}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_xlayout.py tests/test_gpu_transfer.py -x -q -p no:cacheprovider --timeout 600 > gpurun_out/${TAG}_xtest.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_xtest.txt
tail -n 3 gpurun_out/${TAG}_xtest.txt
