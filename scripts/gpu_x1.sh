# usage: bash scripts/gpu_x1.sh <tag> : class-layout tests, parity/transfer suites, short bench
cd $GRAFT_REPO_ROOT
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_xlayout.py -x -q -p no:cacheprovider --timeout 600 > gpurun_out/${TAG}_xtest.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_xtest.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
tail -3 gpurun_out/${TAG}_xtest.txt; tail -2 gpurun_out/${TAG}_pytest.txt; tail -2 gpurun_out/${TAG}_bench.txt | cut -c1-300
